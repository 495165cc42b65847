"""B200-native DGC chunk-partitioned DGNN training step.

Drop-in for the hot path of the reference package ``dynpart`` (DGC,
arXiv 2309.03523): the plan (partition -> assignment -> fusion) is consumed
unchanged; the simulated epoch (sim.simulate_epoch / run_epochs) is replaced
by a real fwd+bwd+exchange+update step on sm_100a kernels (csrc/, C ABI in
include/dgc_b200.h). Names mirror the reference API.
"""
from .plan import (PlanArrays, PlanGraphMismatch, from_dynpart, from_reference_artifacts,
                   load_plan_npz, single_device)
from .stale import EpochLossTrace, StaleConfig, StaleMode, threshold
from .model import DGNNConfig, init_params, synthetic_inputs

__version__ = "0.1.0"


def __getattr__(name):
    # GPU-facing pieces load the native library lazily (fail loudly if absent)
    if name in ("DGNNTrainer", "EpochReport", "run_epochs", "simulate_epoch", "StaleState",
                "reference_billed_messages"):
        from . import trainer
        return getattr(trainer, name)
    if name in ("GruCell", "PackedBatch", "pack_sequences", "gru_forward_masked"):
        from . import fusion
        return getattr(fusion, name)
    if name in ("build_layout",):
        from . import layout
        return layout.build_layout
    raise AttributeError(name)
