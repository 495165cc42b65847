"""End-to-end parity of the B200 training step against the fp64 oracle on the
frozen reference plans: loss, every gradient, and the staleness schedule,
over several epochs, for GRU (T-GCN) and LSTM (MPNN-LSTM) models, D = 1/2/4
(virtual devices on one GPU; same kernels and exchange logic as NCCL)."""
import numpy as np
import pytest
import torch

from oracle.dgnn import OracleConfig, OracleDGNN
from oracle.layout import build_layouts

pytestmark = pytest.mark.gpu


def run_pair(pa, cfg_kw, stale_mode="off", epochs=3, fraction=0.5, seed=0, precision="fp32"):
    from paper_2309_03523_b200 import DGNNConfig, StaleConfig
    from paper_2309_03523_b200.trainer import DGNNTrainer
    from paper_2309_03523_b200.model import init_params, synthetic_inputs
    cfg = DGNNConfig(optimizer="sgd", lr=0.05, precision=precision, **cfg_kw)
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, seed)
    params = init_params(cfg, seed)
    scfg = {"off": StaleConfig.off(), "relax": StaleConfig.adaptive(),
            "tighten": StaleConfig.adaptive(True), "static": StaleConfig.static(fraction)}[stale_mode]
    tr = DGNNTrainer(pa, cfg, scfg, seed=seed, features=X, labels=y, params=params)
    lays = build_layouts(pa.n_instances, pa.inst_entity, pa.inst_t, pa.spatial_edges,
                         pa.temporal_links, pa.structure_device, pa.chunk_of, pa.n_devices,
                         pa.group_device, pa.group_ptr, pa.group_chunks)
    ocfg = OracleConfig(F=cfg.F, H=cfg.H, C=cfg.C, rnn=cfg.rnn, n_rnn=cfg.n_rnn,
                        stale_mode={"relax": "adaptive-relax", "tighten": "adaptive-tighten"}.get(
                            stale_mode, stale_mode), static_fraction=fraction,
                        optimizer="sgd", lr=0.05, momentum=0.9)
    orc = OracleDGNN(lays, X, y, params, ocfg)
    out = []
    for r in range(1, epochs + 1):
        rep = tr.run_epoch()
        forced = None
        if tr.shards[0].stale_on:
            # replay the GPU's decisions; the oracle logs every key where its
            # own fp64 decision differs (checked against the tie band below)
            forced = {f"s{l}": [sh.scache[l].send.cpu().numpy().astype(bool) for sh in tr.shards]
                      for l in range(2)}
            forced.update({f"t{k}": [sh.tcache[k].send.cpu().numpy().astype(bool)
                                     for sh in tr.shards] for k in range(cfg.n_rnn)})
        # replay the GPU's ReLU decisions too (near-ties logged in orc.relu_log,
        # checked against the precision's tie band by check_epochs)
        o = orc.epoch(r, forced, forced_relu=oracle_relu_masks(tr, lays))
        out.append((rep, o, tr.grads(0)))
    orc.precision = precision
    return out, tr, orc


def oracle_relu_masks(tr, lays):
    """The GPU's ReLU decisions of this epoch in the oracle layouts' row order
    (GPU layouts may carry snapshot padding rows: EvolveGCN segments)."""
    out = {0: [], 1: []}
    for i, lay in enumerate(lays):
        gl = tr.layouts[i].own_gid
        pos = np.full(max(int(gl.max(initial=-1)) + 1, 1), -1, np.int64)
        pos[gl[gl >= 0]] = np.flatnonzero(gl >= 0)
        rows = pos[np.asarray(lay.own_gid)]
        assert (rows >= 0).all()
        for l, m in tr.relu_masks(i).items():
            out[l].append(m[rows])
    return out


# ReLU tie band (|z| / max|z| of the layer) per precision; see test_gpu_c2_parity.py
RELU_BAND = {"fp32": 5e-7, "tf32": 2e-3}


def check_relu_ties(orc):
    for e in orc.relu_log:
        assert abs(e["z"]) <= RELU_BAND[orc.precision] * e["scale"], e


def check_epochs(out, rtol=1e-4, orc=None):
    if orc is not None:
        check_relu_ties(orc)
    for rep, o, grads in out:
        assert rep.loss == pytest.approx(o["loss"], rel=rtol)
        for k, g in grads.items():
            ref = o["grads"][k]
            err = np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-30)
            assert err <= rtol, f"epoch {rep.epoch} grad {k}: {err:.2e}"


@pytest.mark.parametrize("name,cfg_kw", [
    ("t2", dict(F=16, H=16, C=16, rnn="gru", n_rnn=1)),
    ("t4", dict(F=16, H=16, C=16, rnn="lstm", n_rnn=2)),
    ("c1", dict(F=16, H=16, C=16, rnn="gru", n_rnn=1)),
])
def test_trainer_matches_oracle_stale_off(artifacts_dir, name, cfg_kw):
    from paper_2309_03523_b200 import load_plan_npz
    pa = load_plan_npz(artifacts_dir / name / "plan.npz")
    out, _, orc = run_pair(pa, cfg_kw, "off", epochs=3)
    check_epochs(out, orc=orc)


def test_trainer_single_device_wide(artifacts_dir):
    from paper_2309_03523_b200 import load_plan_npz, single_device
    pa = single_device(load_plan_npz(artifacts_dir / "t2" / "plan.npz"))
    out, _, orc = run_pair(pa, dict(F=32, H=64, C=16, rnn="lstm", n_rnn=2), "off", epochs=2)
    check_epochs(out, orc=orc)


def subsample_plan(pa, t_max):
    """The plan restricted to snapshots 1..t_max (same devices, chunks and
    instance order; spatial edges are snapshot-local, temporal links kept when
    both ends are)."""
    from paper_2309_03523_b200.plan import PlanArrays
    keep = pa.inst_t <= t_max
    new = np.full(pa.n_instances, -1, np.int64)
    new[keep] = np.arange(int(keep.sum()))
    se = pa.spatial_edges[keep[pa.spatial_edges].all(axis=1)]
    tl = pa.temporal_links[keep[pa.temporal_links].all(axis=1)]
    return PlanArrays(T=t_max, feature_dim=pa.feature_dim, inst_entity=pa.inst_entity[keep],
                      inst_t=pa.inst_t[keep], spatial_edges=new[se].astype(np.int32),
                      temporal_links=new[tl].astype(np.int32),
                      structure_device=pa.structure_device[keep], chunk_of=pa.chunk_of[keep],
                      n_devices=pa.n_devices, profile=dict(pa.profile), meta=dict(pa.meta))


@pytest.mark.parametrize("plan,cfg_kw,mode", [
    ("t2", dict(F=16, H=16, C=16, rnn="gru", n_rnn=1), "relax"),
    ("t2", dict(F=16, H=16, C=16, rnn="gru", n_rnn=1), "tighten"),
    ("t2", dict(F=16, H=16, C=16, rnn="gru", n_rnn=1), "static"),
    # LSTM temporal carries (h|c, width 2H) through their own caches, D = 4
    ("t4", dict(F=16, H=16, C=16, rnn="lstm", n_rnn=2), "relax"),
    ("t4", dict(F=16, H=64, C=16, rnn="lstm", n_rnn=2), "static"),
    # the C4 sweep's plan (1M x 64, GCN+GRU, D = 8), snapshots 1-6 (40k instances)
    ("c4d8-sub", dict(F=16, H=16, C=16, rnn="gru", n_rnn=1), "relax"),
])
def test_trainer_stale_schedule_matches_oracle(artifacts_dir, plan, cfg_kw, mode):
    from paper_2309_03523_b200 import load_plan_npz
    pa = load_plan_npz(artifacts_dir / plan.split("-")[0] / "plan.npz")
    if plan.endswith("-sub"):
        pa = subsample_plan(pa, 6)
    out, tr, orc = run_pair(pa, cfg_kw, mode, epochs=4, fraction=0.3)
    check_epochs(out, rtol=1e-4, orc=orc)
    for rep, o, _ in out:
        for key, th in o["theta"].items():
            if key in rep.stale_detail["theta"]:
                assert rep.stale_detail["theta"][key] == pytest.approx(th, rel=1e-4, abs=2e-6)
    # staleness schedule: the GPU's send sets equal the oracle's fp64 decisions
    # except keys inside the fp32 tie band. The fp32 distance
    # of two nearly equal rows carries the rows' absolute rounding (~1e-7 of
    # their norm each), so the band is |dist - theta| <= 1e-6 * max(1, ||row||);
    # when the rows barely move (layer-0 embeddings, dist ~ 1e-5) that band is a
    # few 1e-3 of theta and holds a few tenths of a percent of the keys.
    n_keys = sum(len(sh.key_rows) for sh in tr.shards) * 2 * len(out)
    for t_ in orc.tie_log:
        assert abs(t_["dist"] - t_["theta"]) <= 1e-6 * max(1.0, t_["norm"]), t_
    assert len(orc.tie_log) <= max(2, n_keys // 100), len(orc.tie_log)
    assert out[-1][0].stale_reduction_pct > 0.0
    print(f"\n{plan} {mode}: {len(orc.tie_log)} tie-band keys; stale reduction "
          + ", ".join(f"{rep.stale_reduction_pct:.1f}%" for rep, _, _ in out))


@pytest.mark.parametrize("name,H", [("t4", 64), ("t2", 128), ("t2-single", 128)])
def test_trainer_tf32_tensor_core_path(artifacts_dir, name, H):
    """TF32 perf mode (tcgen05 GEMMs + tensor-core LSTM recurrence, TF32-rounded
    operands) against the fp64 oracle: loss and EVERY gradient within the
    north star's 2e-2 (max-normalised), with the GPU's ReLU decisions replayed
    and every disagreement inside the TF32 tie band (test_gpu_c2_parity.py)."""
    from paper_2309_03523_b200 import load_plan_npz, single_device
    pa = load_plan_npz(artifacts_dir / name.split("-")[0] / "plan.npz")
    if name.endswith("-single"):  # one device: layer 1 runs aggregate-first
        pa = single_device(pa)
    out, tr, orc = run_pair(pa, dict(F=32, H=H, C=16, rnn="lstm", n_rnn=2), "off", epochs=2,
                            precision="tf32")
    assert tr.shards[0].tc_rnn
    assert tr.shards[0].agg_first == name.endswith("-single")
    check_epochs(out, rtol=2e-2, orc=orc)


def test_trainer_aggregate_first_fp32(artifacts_dir, monkeypatch):
    """Layer 1 as relu((A X) W1 + b1) (the single-device TF32 default, forced
    here in fp32 mode) against the oracle's relu(A (X W1) + b1): the
    reassociated sum differs in rounding only, so with the ReLU decisions
    replayed (near-ties inside the fp32 band) loss and every gradient are
    within 1e-4."""
    monkeypatch.setenv("DGC_AGG_FIRST", "1")
    from paper_2309_03523_b200 import load_plan_npz, single_device
    pa = single_device(load_plan_npz(artifacts_dir / "t2" / "plan.npz"))
    out, tr, orc = run_pair(pa, dict(F=32, H=64, C=16, rnn="lstm", n_rnn=2), "off", epochs=2)
    assert tr.shards[0].agg_first
    check_epochs(out, rtol=1e-4, orc=orc)


@pytest.mark.parametrize("precision,tol,single", [("fp32", 1e-4, False), ("tf32", 2e-2, False),
                                                  ("tf32", 2e-2, True)])
def test_trainer_evolvegcn_matches_oracle(artifacts_dir, precision, tol, single):
    """C3 model (EvolveGCN-O weight evolution + per-snapshot GCN on snapshot-
    segmented layouts) on the reference's 2-device EvolveGCN plan vs the oracle."""
    from paper_2309_03523_b200 import DGNNConfig, load_plan_npz, single_device
    from paper_2309_03523_b200.model import init_params, synthetic_inputs
    from paper_2309_03523_b200.trainer import DGNNTrainer
    pa = load_plan_npz(artifacts_dir / "e2" / "plan.npz")
    if single:  # one device: layer 1 aggregate-first on the per-snapshot weights
        pa = single_device(pa)
    T = int(pa.inst_t.max())
    cfg = DGNNConfig(F=32, H=32, C=8, model="evolve", n_rnn=0, T=T, optimizer="sgd", lr=0.05,
                     precision=precision)
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    params = init_params(cfg, 0)
    tr = DGNNTrainer(pa, cfg, None, features=X, labels=y, params=params)
    assert tr.shards[0].agg_first == single
    lays = build_layouts(pa.n_instances, pa.inst_entity, pa.inst_t, pa.spatial_edges,
                         pa.temporal_links, pa.structure_device, pa.chunk_of, pa.n_devices,
                         pa.group_device, pa.group_ptr, pa.group_chunks)
    ocfg = OracleConfig(F=32, H=32, C=8, model="evolve", T=T, n_rnn=0, optimizer="sgd", lr=0.05)
    orc = OracleDGNN(lays, X, y, params, ocfg, inst_t=pa.inst_t)
    orc.precision = precision
    worst = {}
    for r in (1, 2, 3):
        rep = tr.run_epoch()
        o = orc.epoch(r, forced_relu=oracle_relu_masks(tr, lays))
        assert rep.loss == pytest.approx(o["loss"], rel=tol)
        for k, g in tr.grads(0).items():
            ref = o["grads"][k]
            err = np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-30)
            worst[k] = max(worst.get(k, 0.0), err)
    print(f"\nevolve {precision} single={single}: "
          + ", ".join(f"{k}={v:.1e}" for k, v in worst.items()))
    check_relu_ties(orc)
    bad = {k: v for k, v in worst.items() if not v <= tol}
    assert not bad, bad


@pytest.mark.parametrize("H,precision,devices", [(128, "tf32", 1), (16, "fp32", 1), (16, "fp32", 4)])
def test_cuda_graph_epochs_equal_eager(H, precision, devices):
    """A single-device epoch captured once as a CUDA graph and replayed gives
    bitwise the same losses and parameters as eager epochs (same kernels, every
    reduction in fixed order; the Adam step count lives in device memory)."""
    from pathlib import Path
    from paper_2309_03523_b200 import DGNNConfig, load_plan_npz, single_device
    from paper_2309_03523_b200.trainer import DGNNTrainer
    from paper_2309_03523_b200.model import init_params, synthetic_inputs
    root = Path(__file__).resolve().parents[1]
    pa = load_plan_npz(root / "artifacts" / "t4" / "plan.npz")  # D = 4
    if devices == 1:
        pa = single_device(pa)
    cfg = DGNNConfig(F=H, H=H, C=16, rnn="lstm", n_rnn=2, optimizer="adam", lr=1e-3,
                     precision=precision)
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    params = init_params(cfg, 0)
    runs = []
    for graph in (False, True):
        tr = DGNNTrainer(pa, cfg, None, features=X, labels=y, params=params, cuda_graph=graph)
        losses = [tr.run_epoch().loss for _ in range(4)]
        assert bool(tr._graphs) == graph
        runs.append((losses, tr.params(0)))
    (l0, p0), (l1, p1) = runs
    assert l0 == l1
    for k in p0:
        assert np.array_equal(p0[k], p1[k]), k


@pytest.mark.parametrize("graph", [False, True])
def test_staged_inputs_equal_resident(graph):
    """Epochs fed through the double-buffered input pipeline (stage_inputs /
    run_epoch(next_inputs=...)) equal epochs on resident inputs, bitwise."""
    from pathlib import Path
    from paper_2309_03523_b200 import DGNNConfig, load_plan_npz, single_device
    from paper_2309_03523_b200.trainer import DGNNTrainer
    from paper_2309_03523_b200.model import init_params, synthetic_inputs
    root = Path(__file__).resolve().parents[1]
    pa = single_device(load_plan_npz(root / "artifacts" / "t4" / "plan.npz"))
    cfg = DGNNConfig(F=128, H=128, C=16, rnn="lstm", n_rnn=2, optimizer="adam", lr=1e-3,
                     precision="tf32")
    X, y = synthetic_inputs(pa.n_instances, cfg.F, cfg.C, 0)
    params = init_params(cfg, 0)
    a = DGNNTrainer(pa, cfg, None, features=X, labels=y, params=params, cuda_graph=graph)
    la = [a.run_epoch().loss for _ in range(3)]
    b = DGNNTrainer(pa, cfg, None, features=np.zeros_like(X), labels=np.zeros_like(y),
                    params=params, cuda_graph=graph)
    xs, ys = b.host_inputs(X, y)
    b.stage_inputs(xs, ys)
    lb = [b.run_epoch(next_inputs=(xs, ys)).loss for _ in range(3)]
    assert la == lb
    pa_, pb_ = a.params(0), b.params(0)
    for k in pa_:
        assert np.array_equal(pa_[k], pb_[k]), k
    # software-pipelined submission (epoch i+1 queued before epoch i is read)
    c = DGNNTrainer(pa, cfg, None, features=np.zeros_like(X), labels=np.zeros_like(y),
                    params=params, cuda_graph=graph)
    c.stage_inputs(xs, ys)
    pend = [c.submit_epoch(next_inputs=(xs, ys)) for _ in range(3)]
    lc = [p.result().loss for p in pend]
    assert la == lc
    pc_ = c.params(0)
    for k in pa_:
        assert np.array_equal(pa_[k], pc_[k]), k


@pytest.mark.parametrize("plan,rnn,n_rnn", [("t4", "lstm", 2), ("c1", "gru", 1)])
def test_simulate_epoch_report_fields(artifacts_dir, plan, rnn, n_rnn):
    """simulate_epoch (sim.py:423-432 signature) threaded through one StaleState
    for 3 adaptive-relax epochs: the device-accumulated billing equals the
    host restatement of the reference accounting (sim.py:464-469) for the
    GPU's own send masks, per-device times are measured (one per device,
    compute <= wall) and lambda = max/min of the walls (assign.py:98-104)."""
    from paper_2309_03523_b200 import DGNNConfig, StaleConfig, load_plan_npz
    from paper_2309_03523_b200.trainer import StaleState, reference_billed_messages, simulate_epoch
    pa = load_plan_npz(artifacts_dir / plan / "plan.npz")
    cfg = DGNNConfig(F=16, H=16, C=16, rnn=rnn, n_rnn=n_rnn, optimizer="adam", lr=1e-2)
    scfg = StaleConfig.adaptive()
    state = StaleState(pa, None, pa.profile, pa.n_devices, scfg, cfg=cfg)
    tr = state.trainer
    prof = pa.profile
    per_msg = prof.get("blocks", 1) * prof["embedding_dim"] * prof["bytes_per_scalar"]
    for r in (1, 2, 3):
        rep = simulate_epoch(pa, None, pa.profile, pa.n_devices, scfg, r, None, state)
        sp = [[sh.scache[l].send.cpu().numpy().astype(bool) for sh in tr.shards] for l in range(2)]
        tm = [[sh.tcache[k].send.cpu().numpy().astype(bool) for sh in tr.shards]
              for k in range(n_rnn)]
        n_sp, n_tm = reference_billed_messages(tr.layouts, sp, tm)
        assert rep.spatial_traffic_bytes == n_sp * per_msg
        assert rep.temporal_traffic_bytes == n_tm * per_msg
        assert rep.stale_sent_bytes == (n_sp + n_tm) * per_msg
        assert len(rep.per_device_wall_ms) == len(rep.per_device_compute_ms) == pa.n_devices
        assert all(0 < c <= w for c, w in zip(rep.per_device_compute_ms, rep.per_device_wall_ms))
        assert rep.load_divergence == pytest.approx(max(rep.per_device_wall_ms)
                                                    / min(rep.per_device_wall_ms))
        assert rep.exchanged_rows > 0 and rep.exchanged_bytes > 0
        if r >= 2:
            assert rep.stale_theta > 0 and rep.stale_d > 0
    assert rep.stale_avoided_bytes > 0
    with pytest.raises(ValueError):
        simulate_epoch(pa, None, pa.profile, pa.n_devices, scfg, 7, None, state)
