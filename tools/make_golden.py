"""Generate golden vectors for the hot path by running the UNMODIFIED
reference (``dynpart``, /root/reference, read-only) in the build container.

The fixtures pin the CPU oracle (oracle/) and the GPU parity tests; neither the
tests nor the product ever import the reference on the GPU box.

Usage: PYTHONPATH=/root/reference/pkg/src python tools/make_golden.py
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from dynpart import fusion, sim, stale
from dynpart.costmodel import MessageSet, ModelProfile

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "tests" / "golden"


def _save(name: str, **arrays) -> None:
    np.savez_compressed(OUT / f"{name}.npz", **arrays)


def golden_packing() -> None:
    """pack_sequences / packed_padding (fusion.py:249-325) on SPEC examples
     plus seeded random length lists."""
    cases = [[4, 2, 2], [5, 3, 3], [7], [1, 1, 1, 1], [3, 3, 2, 2, 1, 5, 4]]
    rng = np.random.default_rng(1)
    for n in (10, 57, 300):
        cases.append(rng.integers(1, 33, size=n).tolist())
    ptr, lens, rows_all, mask_all, meta = [0], [], [], [], []
    for lengths in cases:
        b = fusion.pack_sequences([(i, l) for i, l in enumerate(lengths)])
        rows = np.full((b.n_rows, b.row_length, 2), -1, dtype=np.int32)
        for r, row in enumerate(b.rows):
            for p, slot in enumerate(row):
                if slot is not None:
                    rows[r, p] = slot
        packed, naive = fusion.packed_padding(lengths)
        assert packed == b.padding_count
        lens.extend(lengths)
        ptr.append(len(lens))
        rows_all.append(rows.reshape(-1, 2))
        mask_all.append(b.mask.reshape(-1))
        meta.append([b.n_rows, b.row_length, b.padding_count, naive])
    _save("packing", len_ptr=np.asarray(ptr), lengths=np.asarray(lens, dtype=np.int32),
          rows=np.concatenate(rows_all), mask=np.concatenate(mask_all),
          meta=np.asarray(meta, dtype=np.int64))


def golden_gru() -> None:
    """gru_forward_masked / gru_forward (fusion.py:334-469) on seeded cells."""
    out = {}
    for ci, (n_in, hid, nseq, maxlen, seed) in enumerate(
            [(4, 4, 5, 6, 0), (16, 16, 40, 7, 1), (8, 32, 25, 12, 2), (24, 16, 60, 32, 3)]):
        cell = fusion.GruCell.random(n_in, hid, seed=seed)
        rng = np.random.default_rng(100 + seed)
        lengths = rng.integers(1, maxlen + 1, size=nseq)
        seqs = [(e, int(l)) for e, l in enumerate(lengths)]
        batch = fusion.pack_sequences(seqs)
        inputs = {e: rng.normal(size=(l, n_in)) for e, l in seqs}
        res = fusion.gru_forward_masked(cell, batch, inputs)
        unf = {e: fusion.gru_forward(cell, inputs[e]) for e, _ in seqs}
        maxdiff = max(float(np.abs(res[e] - unf[e]).max()) for e, _ in seqs)
        assert maxdiff < 1e-12, maxdiff
        p = f"c{ci}_"
        for k in ("w_update", "u_update", "b_update", "w_reset", "u_reset", "b_reset",
                  "w_cand", "u_cand", "b_cand"):
            out[p + k] = getattr(cell, k)
        out[p + "lengths"] = lengths.astype(np.int32)
        out[p + "x"] = np.concatenate([inputs[e] for e, _ in seqs])
        out[p + "h"] = np.concatenate([res[e] for e, _ in seqs])
    _save("gru", **out)


def golden_stale() -> None:
    """threshold / filter_transmissions / max_cache_gap (stale.py:97-212) over
    a DriftStream (stale.py:269-294), every mode, 6 epochs."""
    n, dim = 400, 16
    spec = stale.DriftSpec(dim=dim)
    out = {}
    modes = {"off": stale.StaleConfig.off(), "static3": stale.StaleConfig.static(0.3),
             "tighten": stale.StaleConfig.adaptive(True), "relax": stale.StaleConfig.adaptive()}
    for mname, cfg in modes.items():
        stream = stale.DriftStream(list(range(n)), spec, seed=7)
        cache = stale.EmbeddingCache()
        trace = stale.EpochLossTrace()
        embs, sends, thetas, drs = [], [], [], []
        for r in range(1, 7):
            emb = stream.epoch(r)
            # a 3/4 subset of keys is boundary each epoch (reference sends per key)
            keys = np.arange(n)[(np.arange(n) + r) % 4 != 0]
            current = {int(k): emb[k] for k in keys}
            theta = 0.0
            d_r = 0.0
            if r >= 2:
                d_r = stale.max_cache_gap(cache, current)
                theta = stale.threshold(trace, r, d_r, cfg)
            dec = stale.filter_transmissions(current, cache, theta)
            assert dec.d_r == d_r or r == 1
            mask = np.zeros(n, dtype=np.uint8)
            mask[dec.send] = 1
            embs.append(emb)
            sends.append(mask)
            thetas.append(theta)
            drs.append(d_r)
            trace.append(2.0 * 0.9 ** (r - 1))
        out[mname + "_emb"] = np.stack(embs)
        out[mname + "_send"] = np.stack(sends)
        out[mname + "_theta"] = np.asarray(thetas)
        out[mname + "_dr"] = np.asarray(drs)
    # threshold known answers
    tr = stale.EpochLossTrace([2.0, 1.0])
    out["thr_tighten"] = np.asarray(stale.threshold(tr, 3, 1.0, stale.StaleConfig.adaptive(True)))
    out["thr_relax"] = np.asarray(stale.threshold(tr, 3, 1.0, stale.StaleConfig.adaptive()))
    _save("stale", **out)


def golden_sim() -> None:
    """Epoch accounting of simulate_epoch/run_epochs (sim.py:401-599) on the
    frozen c1 plan: per-device runs, padding, cut bytes, stale billing."""
    from dynpart.graphstore import load_graph
    from dynpart.partition import chunk_graph_from_json
    from dynpart.assign import Assignment
    from dynpart.fusion import FusionPlan

    d = ROOT / "artifacts" / "c1"
    g = load_graph(str(d / "graph.dg"))
    cg, profile = chunk_graph_from_json(json.loads((d / "chunks.json").read_text()))
    z = np.load(d / "plan.npz")
    sdev = z["structure_device"].astype(np.int64)
    runs = sim._device_sequences(g, sdev, 4)
    msgs = MessageSet(g, profile)
    cut = msgs.cut_mask(sdev)
    asg = Assignment.from_dict(json.loads((d / "assignment.json").read_text()))
    fus = FusionPlan.from_dict(json.loads((d / "fusion.json").read_text()))
    plan = sim.Plan("pgc", cg, asg, fus, sdev, None, {}, msgs, 4)
    cluster = sim.ClusterSpec(n_devices=4)
    reps = sim.run_epochs(g, plan, profile, cluster, 4, stale.StaleConfig.adaptive(),
                          stale.DriftSpec(dim=16), seed=0)
    out = dict(
        run_ptr=np.cumsum([0] + [len(r) for r in runs]),
        run_len=np.asarray([l for r in runs for l in r], dtype=np.int32),
        cut=cut, msg_src=msgs.src, msg_dst=msgs.dst, msg_nbytes=msgs.nbytes,
        msg_spatial=msgs.is_spatial,
    )
    for k in ("spatial_traffic_bytes", "temporal_traffic_bytes", "loading_bytes",
              "padding_slots", "naive_padding_slots", "stale_sent_bytes",
              "stale_avoided_bytes", "stale_theta", "stale_d"):
        out["rep_" + k] = np.asarray([getattr(r, k) for r in reps])
    _save("sim_c1", **out)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    golden_packing()
    golden_gru()
    golden_stale()
    golden_sim()
    print("golden fixtures written to", OUT)
