"""Self-pinning of the fp64 DGNN oracle (the reference has no GCN/LSTM/loss/
backward to pin against): finite differences and
partitioned == unpartitioned structure encoder."""
import json

import numpy as np
import pytest

from oracle.dgnn import OracleConfig, OracleDGNN, param_names, GATES
from oracle.layout import build_layouts


def load_plan(path):
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def layouts_for(z, meta, n_dev=None, fused=True):
    D = meta["n_devices"] if n_dev is None else n_dev
    sdev = z["structure_device"] if n_dev is None else np.zeros_like(z["structure_device"])
    kw = {}
    if fused and n_dev is None:
        kw = dict(group_device=z["group_device"], group_ptr=z["group_ptr"], group_chunks=z["group_chunks"])
    return build_layouts(len(z["inst_entity"]), z["inst_entity"], z["inst_t"], z["spatial_edges"],
                         z["temporal_links"], sdev, z["chunk_of"], D, **kw)


def init_params(cfg, seed=0):
    rng = np.random.default_rng(seed)
    G = GATES[cfg.rnn]
    u = lambda fan, shape: rng.uniform(-1 / np.sqrt(fan), 1 / np.sqrt(fan), size=shape)
    p = {"W1": u(cfg.F, (cfg.F, cfg.H)), "b1": u(cfg.H, cfg.H),
         "W2": u(cfg.H, (cfg.H, cfg.H)), "b2": u(cfg.H, cfg.H)}
    for k in range(cfg.n_rnn):
        p[f"Wx{k}"] = u(cfg.H, (cfg.H, G * cfg.H))
        p[f"U{k}"] = u(cfg.H, (cfg.H, G * cfg.H))
        p[f"br{k}"] = u(cfg.H, G * cfg.H)
    p["Wo"] = u(cfg.H, (cfg.H, cfg.C))
    p["bo"] = u(cfg.H, cfg.C)
    return p


@pytest.fixture(scope="module")
def t2(artifacts_dir):
    return load_plan(artifacts_dir / "t2" / "plan.npz")


@pytest.mark.parametrize("rnn,n_rnn", [("gru", 1), ("lstm", 2)])
def test_oracle_gradients_finite_difference(t2, rnn, n_rnn):
    z, meta = t2
    lays = layouts_for(z, meta)
    cfg = OracleConfig(F=6, H=5, C=4, rnn=rnn, n_rnn=n_rnn, lr=0.0)
    n = len(z["inst_entity"])
    rng = np.random.default_rng(3)
    X = rng.normal(size=(n, cfg.F))
    y = rng.integers(0, cfg.C, size=n)
    p0 = init_params(cfg)
    base = OracleDGNN(lays, X, y, p0, cfg).epoch(1)
    for trial in range(3):
        v = {k: rng.normal(size=np.shape(a)) for k, a in p0.items()}
        eps = 1e-6
        lp = OracleDGNN(lays, X, y, {k: p0[k] + eps * v[k] for k in p0}, cfg).epoch(1)["loss"]
        lm = OracleDGNN(lays, X, y, {k: p0[k] - eps * v[k] for k in p0}, cfg).epoch(1)["loss"]
        fd = (lp - lm) / (2 * eps)
        an = sum(float((base["grads"][k] * v[k]).sum()) for k in p0)
        assert fd == pytest.approx(an, rel=1e-6, abs=1e-10)


def test_partitioned_structure_encoder_equals_unpartitioned(t2):
    z, meta = t2
    cfg = OracleConfig(F=6, H=5, C=4, rnn="gru", n_rnn=1)
    n = len(z["inst_entity"])
    rng = np.random.default_rng(4)
    X = rng.normal(size=(n, cfg.F))
    y = rng.integers(0, cfg.C, size=n)
    p0 = init_params(cfg)
    part = layouts_for(z, meta)
    one = layouts_for(z, meta, n_dev=1)
    a = OracleDGNN(part, X, y, p0, cfg).epoch(1)
    b = OracleDGNN(one, X, y, p0, cfg).epoch(1)
    full = np.zeros((n, cfg.H))
    for lay, h in zip(part, a["h_gcn"][1]):
        full[lay.own_gid] = h
    ref = np.zeros((n, cfg.H))
    ref[one[0].own_gid] = b["h_gcn"][1][0]
    np.testing.assert_allclose(full, ref, rtol=1e-12, atol=1e-12)
    # W1/W2 gradients of the structure encoder agree up to the RNN carry cut:
    # with zero carries the only difference is the temporal carry, which the
    # partitioned epoch-1 model replaces by zero (Appendix B.2(a)).
    assert np.isfinite(a["loss"]) and np.isfinite(b["loss"])


def test_stale_schedule_first_epoch_sends_all(t2):
    z, meta = t2
    cfg = OracleConfig(F=6, H=5, C=4, rnn="gru", n_rnn=1, stale_mode="adaptive-relax")
    n = len(z["inst_entity"])
    rng = np.random.default_rng(5)
    X = rng.normal(size=(n, cfg.F))
    y = rng.integers(0, cfg.C, size=n)
    o = OracleDGNN(layouts_for(z, meta), X, y, init_params(cfg), cfg)
    e1 = o.epoch(1)
    assert all(s.all() for s in e1["send"]["s0"])
    e2 = o.epoch(2)
    e3 = o.epoch(3)
    for e in (e2, e3):
        assert e["theta"]["s0"] <= e["d_r"]["s0"] + 1e-15
        assert e["d_r"]["s0"] > 0


def test_oracle_evolvegcn_gradients_finite_difference(artifacts_dir):
    """EvolveGCN-O oracle (C3 model): directional finite differences through the
    weight evolution, the per-snapshot GCN and the partitioned exchange."""
    from paper_2309_03523_b200.model import DGNNConfig, init_params as pinit
    z, meta = load_plan(artifacts_dir / "e2" / "plan.npz")
    lays = layouts_for(z, meta)
    T = int(meta["T"])
    cfg = OracleConfig(F=6, H=5, C=4, model="evolve", T=T, n_rnn=0, lr=0.0)
    pc = DGNNConfig(F=6, H=5, C=4, model="evolve", n_rnn=0, T=T)
    n = len(z["inst_entity"])
    rng = np.random.default_rng(7)
    X = rng.normal(size=(n, cfg.F))
    y = rng.integers(0, cfg.C, size=n)
    p0 = {k: v.astype(np.float64) for k, v in pinit(pc, 1).items()}
    base = OracleDGNN(lays, X, y, p0, cfg, inst_t=z["inst_t"]).epoch(1)
    for trial in range(3):
        v = {k: rng.normal(size=np.shape(a)) for k, a in p0.items()}
        eps = 1e-6
        lp = OracleDGNN(lays, X, y, {k: p0[k] + eps * v[k] for k in p0}, cfg, inst_t=z["inst_t"]).epoch(1)["loss"]
        lm = OracleDGNN(lays, X, y, {k: p0[k] - eps * v[k] for k in p0}, cfg, inst_t=z["inst_t"]).epoch(1)["loss"]
        fd = (lp - lm) / (2 * eps)
        an = sum(float((base["grads"][k] * v[k]).sum()) for k in p0)
        assert fd == pytest.approx(an, rel=1e-6, abs=1e-10)
