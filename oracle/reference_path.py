"""numpy restatement of the reference functions on the hot path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Pinned against the
golden vectors in tests/golden/ that tools/make_golden.py produced by running
the unmodified reference.
"""
from __future__ import annotations

import math

import numpy as np


# -- temporal fusion: fusion.py:249-325 ------------------------------------------

def ffd_place(lengths):
    """fusion.py:249-275 ``_ffd_place``: exact first-fit-decreasing with the
    scan restart only when the length value drops."""
    row_length = max(lengths) if len(lengths) else 0
    order = sorted(range(len(lengths)), key=lambda i: (-lengths[i], i))
    row_of = [0] * len(lengths)
    used: list[int] = []
    start = 0
    prev = None
    for i in order:
        ln = lengths[i]
        if ln != prev:
            start = 0
            prev = ln
        r = start
        while r < len(used) and used[r] + ln > row_length:
            r += 1
        start = r
        if r == len(used):
            used.append(0)
        used[r] += ln
        row_of[i] = r
    return row_of, used


def pack_sequences(lengths):
    """fusion.py:278-313 ``pack_sequences`` keyed by sequence index.

    Returns (slots int32[R, L, 2] = (seq, pos) or -1, mask uint8[R, L], padding).
    """
    if len(lengths) == 0:
        return np.zeros((0, 0, 2), np.int32), np.zeros((0, 0), np.uint8), 0
    if min(lengths) < 1:
        raise ValueError("sequence length must be >= 1")
    L = max(lengths)
    row_of, used = ffd_place(list(lengths))
    slots = np.full((len(used), L, 2), -1, dtype=np.int32)
    fill = [0] * len(used)
    for i in sorted(range(len(lengths)), key=lambda k: (-lengths[k], k)):
        r = row_of[i]
        for p in range(lengths[i]):
            slots[r, fill[r] + p] = (i, p)
        fill[r] += lengths[i]
    mask = np.zeros((len(used), L), dtype=np.uint8)
    a, b = slots[:, :-1], slots[:, 1:]
    cont = (a[..., 0] >= 0) & (b[..., 0] == a[..., 0]) & (b[..., 1] == a[..., 1] + 1)
    mask[:, 1:] = cont
    padding = sum(L - u for u in used)
    return slots, mask, padding


def packed_padding(lengths):
    """fusion.py:316-325."""
    if len(lengths) == 0:
        return 0, 0
    L = max(lengths)
    _, used = ffd_place(list(lengths))
    return len(used) * L - sum(lengths), len(lengths) * L - sum(lengths)


# -- reference-form GRU: fusion.py:341-469 ---------------------------------------

def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def gru_step(x, h, wr, ur, br, wz, uz, bz, wc, uc, bc):
    """fusion.py:409-413 ``GruCell.step`` (reset applied before U_c)."""
    r = sigmoid(x @ wr + h @ ur + br)
    z = sigmoid(x @ wz + h @ uz + bz)
    c = np.tanh(x @ wc + (r * h) @ uc + bc)
    return (1.0 - z) * c + z * h


def gru_forward_masked(cell: dict, lengths, xs):
    """fusion.py:428-469 ``gru_forward_masked`` on sequences keyed by index.

    ``cell`` holds the GruCell fields by name; ``xs`` is the concatenation of
    all sequences' (len, in) inputs. Returns the concatenated (len, H) states.
    """
    slots, mask, _ = pack_sequences(list(lengths))
    offs = np.concatenate([[0], np.cumsum(lengths)])
    R, L = mask.shape
    H = cell["w_update"].shape[1]
    X = np.zeros((R, L, xs.shape[1]))
    valid = slots[..., 0] >= 0
    gidx = np.where(valid, offs[np.maximum(slots[..., 0], 0)] + slots[..., 1], 0)
    X[valid] = xs[gidx[valid]]
    h = np.zeros((R, H))
    out = np.zeros((len(xs), H))
    args = [cell[k] for k in ("w_reset", "u_reset", "b_reset", "w_update", "u_update",
                              "b_update", "w_cand", "u_cand", "b_cand")]
    for p in range(L):
        h = h * mask[:, p:p + 1]
        h = gru_step(X[:, p], h, *args)
        out[gidx[valid[:, p], p]] = h[valid[:, p]]
    return out


# -- adaptive stale aggregation: stale.py:72-212 --------------------------------

def progress(losses, r):
    """stale.py:85-94 ``EpochLossTrace.progress``."""
    if r < 2:
        raise ValueError("progress is defined from epoch 2 on")
    l1 = losses[0]
    return (l1 - losses[r - 2]) / l1


def threshold(losses, r, d_r, mode: str, static_fraction: float = 0.5) -> float:
    """stale.py:97-108 ``threshold`` (modes: off/static/adaptive-tighten/adaptive-relax)."""
    if d_r < 0:
        raise ValueError("d_r must be >= 0")
    if mode == "off":
        return 0.0
    if mode == "static":
        return static_fraction * d_r
    p = progress(losses, r)
    if mode == "adaptive-tighten":
        return d_r / (1.0 + math.exp(p))
    return d_r / (1.0 + math.exp(-p))


def filter_transmissions(current: np.ndarray, cache: np.ndarray, cached: np.ndarray,
                         theta: float, dist_dtype=np.float64):
    """stale.py:154-176 ``filter_transmissions`` over dense key arrays.

    ``current``/``cache`` are (K, H); ``cached`` marks keys with a cached copy.
    Send iff uncached or ||cur - cached||_2 > theta (strict); sent keys refresh
    the cache in place. Returns (send mask, d_r, dist). ``dist_dtype`` float32
    reproduces the GPU's fp32 sequential distance (the tie-band caveat of
    SURVEY.md §7 (ii)).
    """
    diff = (current.astype(dist_dtype) - cache.astype(dist_dtype))
    if dist_dtype == np.float32:
        acc = np.zeros(len(diff), dtype=np.float32)
        for j in range(diff.shape[1]):  # fixed sequential order, fp32 (= K5)
            acc = (acc + diff[:, j] * diff[:, j]).astype(np.float32)
        dist = np.sqrt(acc).astype(np.float64)
    else:
        dist = np.sqrt((diff * diff).sum(axis=1))
    d_r = float(dist[cached].max()) if cached.any() else 0.0
    send = (~cached) | (dist > theta)
    cache[send] = current[send]
    cached |= send
    return send, d_r, dist


def max_cache_gap(current, cache, cached) -> float:
    """stale.py:205-212."""
    if not cached.any():
        return 0.0
    d = current[cached] - cache[cached]
    return float(np.sqrt((d * d).sum(axis=1)).max())


# -- epoch accounting: sim.py:401-420, costmodel.py:106-165 -----------------------

def device_sequences(inst_entity, inst_t, tdev, n_dev):
    """sim.py:401-420 ``_device_sequences``: per device, lengths of maximal
    same-device runs of each entity's presence chain, entities ascending.
    Also returns the runs as lists of global instance indices."""
    order = np.lexsort((inst_t, inst_entity))
    runs = [[] for _ in range(n_dev)]
    cur = []
    prev_e = None
    prev_d = None
    for i in order.tolist():
        e, d = int(inst_entity[i]), int(tdev[i])
        if e != prev_e or d != prev_d:
            if cur:
                runs[prev_d].append(cur)
            cur = []
        cur.append(i)
        prev_e, prev_d = e, d
    if cur:
        runs[prev_d].append(cur)
    return runs


def messages(spatial_edges, temporal_links, profile: dict):
    """costmodel.py:95-158 ``MessageSet`` for previous-only fanout."""
    H, s = profile["embedding_dim"], profile["bytes_per_scalar"]
    ts = profile["blocks"] * profile["spatial_msgs_per_block"] * H * s
    tt = profile["blocks"] * profile["temporal_msgs_per_block"] * H * s
    se = np.asarray(spatial_edges, dtype=np.int64).reshape(-1, 2)
    tl = np.asarray(temporal_links, dtype=np.int64).reshape(-1, 2)
    src = np.concatenate([se[:, 0], se[:, 1], tl[:, 0]])
    dst = np.concatenate([se[:, 1], se[:, 0], tl[:, 1]])
    nbytes = np.concatenate([np.full(2 * len(se), ts, np.int64), np.full(len(tl), tt, np.int64)])
    is_sp = np.concatenate([np.ones(2 * len(se), bool), np.zeros(len(tl), bool)])
    return src, dst, nbytes, is_sp


def billed_bytes(src, dst, nbytes, is_sp, sdev, send_mask=None):
    """sim.py:445,464-470: billed = cut & send[src]; returns (spatial, temporal,
    sent_total, avoided)."""
    cut = sdev[src] != sdev[dst]
    billed = cut if send_mask is None else cut & send_mask[src]
    sp = int(nbytes[billed & is_sp].sum())
    tm = int(nbytes[billed & ~is_sp].sum())
    avoided = int(nbytes[cut & ~billed].sum())
    return sp, tm, sp + tm, avoided
