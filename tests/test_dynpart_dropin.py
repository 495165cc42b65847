"""The drop-in boundary against the LIVE reference package (CPU; skipped when
/root/reference is absent, e.g. on the GPU box): a plan built by the
unmodified dynpart.sim.build_plan goes through from_dynpart unchanged, and the
B200 step's billing of send masks equals the reference's own accounting
(sim.py:445-470) -- with staleness off against simulate_epoch's report, and
with the reference's own adaptive stale decisions over several epochs."""
import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path("/root/reference/pkg/src")
if not REF.exists():
    pytest.skip("reference package not present", allow_module_level=True)
if str(REF) not in sys.path:
    sys.path.insert(0, str(REF))

dynpart = pytest.importorskip("dynpart")
from dynpart import graphstore, sim, stale  # noqa: E402
from dynpart.costmodel import ModelProfile  # noqa: E402

from paper_2309_03523_b200.layout import build_layout  # noqa: E402
from paper_2309_03523_b200.plan import PlanGraphMismatch, from_dynpart  # noqa: E402


def _graph(N=3000, T=8, seed=0):
    E = 4 * N
    spec = graphstore.SyntheticSpec(
        total_vertices=N, total_edges=E, T=T, edges_per_snapshot_mean=E / T,
        edges_per_snapshot_stddev=E / T,
        presence_length_distribution=graphstore.LengthDistribution.bimodal(1, T // 4, T // 2, T, 0.2),
        rng_seed=seed, feature_dim=16, edge_attachment="preferential")
    return graphstore.generate(spec)


@pytest.fixture(scope="module", params=[(1, 2, 1), (1, 2, 2)], ids=["gcn+gru", "gcn+lstm"])
def live(request):
    g = _graph()
    profile = ModelProfile(*request.param, "previous-only", 16, 4)
    cluster = sim.ClusterSpec(n_devices=4)
    plan = sim.build_plan(g, "pgc", profile, cluster)
    pa = from_dynpart(g, plan)
    lays = [build_layout(pa, d) for d in range(pa.n_devices)]
    return g, plan, profile, cluster, pa, lays


def _billing(pa, lays, profile, sp_masks, tm_masks):
    """The trainer's billing (trainer.reference_billed_messages x per-message
    bytes of one layer) for global per-instance masks per layer."""
    from paper_2309_03523_b200.trainer import reference_billed_messages
    sp = [[m[lay.own_gid[lay.key_rows]] for lay in lays] for m in sp_masks]
    tm = [[m[lay.own_gid[lay.tkey_rows]] for lay in lays] for m in tm_masks]
    n_sp, n_tm = reference_billed_messages(lays, sp, tm)
    per_msg = profile.blocks * profile.embedding_dim * profile.bytes_per_scalar
    return n_sp * per_msg, n_tm * per_msg


def test_from_dynpart_is_the_plan(live):
    g, plan, profile, cluster, pa, lays = live
    np.testing.assert_array_equal(pa.structure_device, plan.structure_device)
    assert pa.meta["method"] == "pgc" and pa.n_devices == 4
    assert pa.profile == profile.to_dict()
    for d, lay in enumerate(lays):  # rows = the device's instances, fusion-group order
        assert set(lay.own_gid.tolist()) == set(np.flatnonzero(plan.structure_device == d).tolist())


def test_billing_equals_simulate_epoch_stale_off(live):
    g, plan, profile, cluster, pa, lays = live
    rep = sim.simulate_epoch(g, plan, profile, cluster)
    n_rnn = profile.temporal_msgs_per_block
    ones = np.ones(pa.n_instances, bool)
    sp, tm = _billing(pa, lays, profile, [ones, ones], [ones] * n_rnn)
    assert sp == rep.spatial_traffic_bytes
    assert tm == rep.temporal_traffic_bytes
    # padding / loading fields as the trainer reports them
    assert sum(l.padding for l in lays) == rep.padding_slots
    assert sum(l.naive_padding for l in lays) == rep.naive_padding_slots
    assert sum(l.loaded_rows for l in lays) * g.feature_dim * profile.bytes_per_scalar == rep.loading_bytes


def test_billing_equals_reference_stale_decisions(live, monkeypatch):
    """Replay the reference's own adaptive-relax decisions (one send mask per
    source instance, sim.py:450-463) through the trainer's billing: every
    epoch's spatial/temporal/stale bytes equal the reference report's."""
    g, plan, profile, cluster, pa, lays = live
    decisions = []
    orig = sim.filter_transmissions

    def spy(current, cache, theta):
        dec = orig(current, cache, theta)
        decisions.append(set(int(k) for k in dec.send))
        return dec
    monkeypatch.setattr(sim, "filter_transmissions", spy)
    reps = sim.run_epochs(g, plan, profile, cluster, 4, stale.StaleConfig.adaptive())
    assert len(decisions) == 4
    n_rnn = profile.temporal_msgs_per_block
    for rep, sent in zip(reps, decisions):
        m = np.zeros(pa.n_instances, bool)
        m[list(sent)] = True
        sp, tm = _billing(pa, lays, profile, [m, m], [m] * n_rnn)
        assert sp == rep.spatial_traffic_bytes, rep.epoch
        assert tm == rep.temporal_traffic_bytes, rep.epoch
        assert sp + tm == rep.stale_sent_bytes
    assert reps[-1].stale_avoided_bytes > 0


def test_billing_random_per_layer_masks(live):
    """Per-layer caches: each GCN / RNN layer bills its own
    mask at one layer's share of a reference message."""
    g, plan, profile, cluster, pa, lays = live
    rng = np.random.default_rng(5)
    msgs = plan.messages
    cut = msgs.cut_mask(plan.structure_device, None)
    n_rnn = profile.temporal_msgs_per_block
    sp_m = [rng.random(pa.n_instances) < 0.5 for _ in range(2)]
    tm_m = [rng.random(pa.n_instances) < 0.5 for _ in range(n_rnn)]
    exp_sp = sum(int(msgs.nbytes[cut & msgs.is_spatial & m[msgs.src]].sum()) // 2 for m in sp_m)
    exp_tm = sum(int(msgs.nbytes[cut & ~msgs.is_spatial & m[msgs.src]].sum()) // n_rnn
                 for m in tm_m)
    assert _billing(pa, lays, profile, sp_m, tm_m) == (exp_sp, exp_tm)


def test_simulate_epoch_guards(live):
    """The reference's plan/graph and plan/cluster guards (sim.py:433-437)
    fire before any device work."""
    from paper_2309_03523_b200.trainer import simulate_epoch
    g, plan, profile, cluster, pa, lays = live
    with pytest.raises(PlanGraphMismatch):
        simulate_epoch(g, plan, profile, sim.ClusterSpec(n_devices=2))
    other = _graph(N=2000, seed=1)
    with pytest.raises(PlanGraphMismatch):
        simulate_epoch(other, plan, profile, cluster)


def test_from_dynpart_rejects_pss_ts():
    g = _graph(N=1500)
    profile = ModelProfile.recurrent(16)
    plan = sim.build_plan(g, "pss-ts", profile, sim.ClusterSpec(n_devices=2))
    with pytest.raises(ValueError, match="pss-ts"):
        from_dynpart(g, plan)
    plan = sim.build_plan(g, "pts", profile, sim.ClusterSpec(n_devices=2))
    assert from_dynpart(g, plan).meta["method"] == "pts"


def test_for_profile_rejects_all_snapshots_fanout():
    from paper_2309_03523_b200 import DGNNConfig
    prof = ModelProfile(1, 2, 1, "all-snapshots", 16, 4).to_dict()
    with pytest.raises(ValueError, match="previous-only"):
        DGNNConfig.for_profile(prof, F=16)
