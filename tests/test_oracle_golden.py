"""Pin the CPU oracle (oracle/reference_path.py) against golden vectors the
unmodified reference produced (tools/make_golden.py)."""
import numpy as np
import pytest

from oracle import reference_path as rp


def test_pack_sequences_matches_reference(golden_dir):
    z = np.load(golden_dir / "packing.npz")
    ptr, meta = z["len_ptr"], z["meta"]
    roff = 0
    for i in range(len(meta)):
        lengths = z["lengths"][ptr[i]:ptr[i + 1]].tolist()
        R, L, pad, naive = meta[i]
        slots, mask, padding = rp.pack_sequences(lengths)
        assert slots.shape[:2] == (R, L)
        np.testing.assert_array_equal(slots.reshape(-1, 2), z["rows"][roff:roff + R * L])
        np.testing.assert_array_equal(mask.reshape(-1), z["mask"][roff:roff + R * L])
        assert padding == pad
        assert rp.packed_padding(lengths) == (pad, naive)
        roff += R * L


def test_spec_packing_examples():
    # [4,2,2] -> 2 rows of 4, padding 0 (naive 4)
    slots, mask, pad = rp.pack_sequences([4, 2, 2])
    assert slots.shape[:2] == (2, 4) and pad == 0
    np.testing.assert_array_equal(mask, [[0, 1, 1, 1], [0, 1, 0, 1]])
    assert rp.packed_padding([4, 2, 2]) == (0, 4)


def test_gru_forward_masked_matches_reference(golden_dir):
    z = np.load(golden_dir / "gru.npz")
    for ci in range(4):
        p = f"c{ci}_"
        cell = {k: z[p + k] for k in ("w_update", "u_update", "b_update", "w_reset", "u_reset",
                                      "b_reset", "w_cand", "u_cand", "b_cand")}
        h = rp.gru_forward_masked(cell, z[p + "lengths"].tolist(), z[p + "x"])
        np.testing.assert_allclose(h, z[p + "h"], rtol=0, atol=1e-12)


def test_threshold_known_answers(golden_dir):
    z = np.load(golden_dir / "stale.npz")
    assert rp.threshold([2.0, 1.0], 3, 1.0, "adaptive-tighten") == pytest.approx(float(z["thr_tighten"]), abs=0)
    assert rp.threshold([2.0, 1.0], 3, 1.0, "adaptive-relax") == pytest.approx(float(z["thr_relax"]), abs=0)
    assert rp.threshold([2.0, 2.0], 3, 4.0, "adaptive-relax") == 2.0
    assert rp.threshold([2.0], 2, 5.0, "off") == 0.0


@pytest.mark.parametrize("mode,cfg", [("off", ("off", 0.5)), ("static3", ("static", 0.3)),
                                      ("tighten", ("adaptive-tighten", 0.5)),
                                      ("relax", ("adaptive-relax", 0.5))])
def test_filter_transmissions_matches_reference(golden_dir, mode, cfg):
    z = np.load(golden_dir / "stale.npz")
    emb, send, theta, drs = z[mode + "_emb"], z[mode + "_send"], z[mode + "_theta"], z[mode + "_dr"]
    n, dim = emb.shape[1:]
    cache = np.zeros((n, dim))
    cached = np.zeros(n, bool)
    losses = []
    for r in range(1, emb.shape[0] + 1):
        keys = np.arange(n)[(np.arange(n) + r) % 4 != 0]
        th = 0.0
        if r >= 2:
            d_r = rp.max_cache_gap(emb[r - 1][keys], cache[keys], cached[keys])
            assert d_r == pytest.approx(drs[r - 1], rel=1e-12)
            th = rp.threshold(losses, r, d_r, *cfg)
        assert th == pytest.approx(theta[r - 1], rel=1e-12, abs=0)
        c, cc = cache[keys], cached[keys]
        s, _, _ = rp.filter_transmissions(emb[r - 1][keys], c, cc, th)
        cache[keys], cached[keys] = c, cc
        got = np.zeros(n, np.uint8)
        got[keys[s]] = 1
        np.testing.assert_array_equal(got, send[r - 1])
        losses.append(2.0 * 0.9 ** (r - 1))


def test_device_sequences_and_billing_match_reference(golden_dir, artifacts_dir):
    z = np.load(golden_dir / "sim_c1.npz")
    pz = np.load(artifacts_dir / "c1" / "plan.npz")
    sdev = pz["structure_device"].astype(np.int64)
    runs = rp.device_sequences(pz["inst_entity"], pz["inst_t"], sdev, 4)
    lens = [len(r) for dev in runs for r in dev]
    np.testing.assert_array_equal(lens, z["run_len"])
    np.testing.assert_array_equal(np.cumsum([0] + [len(d) for d in runs]), z["run_ptr"])
    pad = naive = 0
    for dev in runs:
        a, b = rp.packed_padding([len(r) for r in dev])
        pad, naive = pad + a, naive + b
    assert pad == z["rep_padding_slots"][0] and naive == z["rep_naive_padding_slots"][0]
    import json
    meta = json.loads(bytes(pz["meta"]).decode())
    src, dst, nb, is_sp = rp.messages(pz["spatial_edges"], pz["temporal_links"], meta["profile"])
    np.testing.assert_array_equal(src, z["msg_src"])
    np.testing.assert_array_equal(dst, z["msg_dst"])
    np.testing.assert_array_equal(nb, z["msg_nbytes"])
    sp_b, tm_b, tot, av = rp.billed_bytes(src, dst, nb, is_sp, sdev)
    assert tot == z["rep_stale_sent_bytes"][0]  # epoch 1 sends every cut message
    assert av == 0
