"""Plan -> per-device layout, restated in plain Python.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). An independent
restatement of the product's native builder
(paper_2309_03523_b200/csrc/layout.cpp); tests/test_layout.py compares the two
array by array. Every ordering rule comes from the reference:
  rows by fusion group (fusion.py:200-203), ascending global index inside a
  group (partition.py:303-304); runs exactly as sim.py:401-420; packing
  fusion.py:278-313 keyed by run index; exchange lists from the cut messages
  of costmodel.py:106-165.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .reference_path import device_sequences, pack_sequences


@dataclass
class OracleLayout:
    device: int
    n_devices: int
    own_gid: np.ndarray
    halo_gid: np.ndarray
    group_ptr: np.ndarray
    row_ptr: np.ndarray
    col: np.ndarray
    dinv: np.ndarray
    t_row_ptr: np.ndarray
    t_col: np.ndarray
    key_rows: np.ndarray          # spatial stale keys (local own rows)
    send_ptr: np.ndarray          # per peer, positions into key_rows
    send_pos: np.ndarray
    recv_ptr: np.ndarray          # per peer, local halo ids (>= n_own)
    recv_slot: np.ndarray
    run_ptr: np.ndarray
    run_rows: np.ndarray          # local own rows, time order per run
    run_pred_gid: np.ndarray      # -1 or global index of the remote predecessor
    run_carry: np.ndarray         # carry slot of the run or -1
    n_rows: int
    row_len: int
    slot_row: np.ndarray          # (R*L,) local own row or -1
    slot_mask: np.ndarray         # (R*L,) uint8 carry mask (reference form)
    slot_carry: np.ndarray        # (R*L,) carry slot at remote-pred run starts else -1
    tkey_rows: np.ndarray         # temporal carry keys (own rows with remote successor)
    tsend_ptr: np.ndarray
    tsend_pos: np.ndarray
    trecv_ptr: np.ndarray
    trecv_carry: np.ndarray       # carry slots, ordered by predecessor gid
    padding: int
    naive_padding: int
    extra: dict = field(default_factory=dict)

    @property
    def n_own(self):
        return len(self.own_gid)

    @property
    def n_halo(self):
        return len(self.halo_gid)

    @property
    def n_carry(self):
        return int((self.run_carry >= 0).sum())


def own_row_order(structure_device, chunk_of, group_device, group_ptr, group_chunks, d):
    """Rows of device d: fusion groups in FusionPlan order, ascending global
    index inside each group; without a fusion plan one segment per chunk in
    ascending chunk id."""
    gids = np.flatnonzero(structure_device == d)
    if group_device is None or len(group_device) == 0:
        seg_of = chunk_of[gids]
    else:
        gidx = np.flatnonzero(group_device == d)
        chunk_seg = {}
        for s, gi in enumerate(gidx):
            for c in group_chunks[group_ptr[gi]:group_ptr[gi + 1]]:
                chunk_seg[int(c)] = s
        seg_of = np.asarray([chunk_seg[int(c)] for c in chunk_of[gids]], dtype=np.int64)
    order = np.lexsort((gids, seg_of))
    rows = gids[order]
    seg_sorted = seg_of[order]
    segs, starts = np.unique(seg_sorted, return_index=True)
    group_ptr_out = np.concatenate([starts, [len(rows)]]).astype(np.int64)
    return rows, group_ptr_out


def build_layouts(n_inst, inst_entity, inst_t, spatial_edges, temporal_links,
                  structure_device, chunk_of, n_devices,
                  group_device=None, group_ptr=None, group_chunks=None):
    se = np.asarray(spatial_edges, dtype=np.int64).reshape(-1, 2)
    tl = np.asarray(temporal_links, dtype=np.int64).reshape(-1, 2)
    sdev = np.asarray(structure_device, dtype=np.int64)
    deg = np.bincount(se.reshape(-1), minlength=n_inst)
    dinv_g = 1.0 / np.sqrt(deg + 1.0)
    nbrs = [[] for _ in range(n_inst)]
    for u, v in se.tolist():
        nbrs[u].append(v)
        nbrs[v].append(u)
    succ = np.full(n_inst, -1, np.int64)
    pred = np.full(n_inst, -1, np.int64)
    succ[tl[:, 0]] = tl[:, 1]
    pred[tl[:, 1]] = tl[:, 0]
    runs_all = device_sequences(inst_entity, inst_t, sdev, n_devices)

    out = []
    for d in range(n_devices):
        own, gptr = own_row_order(sdev, chunk_of, group_device, group_ptr, group_chunks, d)
        n_own = len(own)
        halo = sorted({v for u in own.tolist() for v in nbrs[u] if sdev[v] != d})
        halo = np.asarray(halo, dtype=np.int64)
        local = {int(g): i for i, g in enumerate(own)}
        for j, g in enumerate(halo.tolist()):
            local[g] = n_own + j
        row_ptr = [0]
        col = []
        for u in own.tolist():
            cs = sorted(nbrs[u] + [u])
            col.extend(local[c] for c in cs)
            row_ptr.append(len(col))
        gid_of_local = np.concatenate([own, halo])
        # transposed CSR: for each local column, the own rows pointing at it
        tcols = [[] for _ in range(len(gid_of_local))]
        for i, u in enumerate(own.tolist()):
            for c in col[row_ptr[i]:row_ptr[i + 1]]:
                tcols[c].append(i)
        t_row_ptr = [0]
        t_col = []
        for c in range(len(gid_of_local)):
            lst = sorted(tcols[c], key=lambda i: own[i])
            t_col.extend(lst)
            t_row_ptr.append(len(t_col))
        # spatial exchange lists
        key_set = sorted({u for u in own.tolist() if any(sdev[v] != d for v in nbrs[u])})
        key_pos = {g: k for k, g in enumerate(key_set)}
        send_ptr, send_pos, recv_ptr, recv_slot = [0], [], [0], []
        for p in range(n_devices):
            if p != d:
                srows = sorted({u for u in own.tolist() if any(sdev[v] == p for v in nbrs[u])})
                send_pos.extend(key_pos[g] for g in srows)
                recv_slot.extend(local[g] for g in halo.tolist() if sdev[g] == p)
            send_ptr.append(len(send_pos))
            recv_ptr.append(len(recv_slot))
        # time-encoder runs (sim.py:401-420) keyed by run index
        runs = runs_all[d]
        run_ptr = np.cumsum([0] + [len(r) for r in runs]).astype(np.int64)
        run_rows = np.asarray([local[g] for r in runs for g in r], dtype=np.int64)
        run_pred = np.asarray([pred[r[0]] if pred[r[0]] >= 0 and sdev[pred[r[0]]] != d else -1
                               for r in runs], dtype=np.int64)
        run_carry = np.full(len(runs), -1, np.int64)
        run_carry[run_pred >= 0] = np.arange(int((run_pred >= 0).sum()))
        lengths = [len(r) for r in runs]
        slots, mask, padding = pack_sequences(lengths)
        R, L = mask.shape
        slot_row = np.full((R, L), -1, np.int64)
        slot_carry = np.full((R, L), -1, np.int64)
        valid = slots[..., 0] >= 0
        rr = slots[..., 0][valid]
        pp = slots[..., 1][valid]
        slot_row[valid] = run_rows[run_ptr[rr] + pp]
        sc = np.where(pp == 0, run_carry[rr], -1)
        slot_carry[valid] = sc
        naive = sum(max(lengths) - l for l in lengths) if lengths else 0
        # temporal carry keys / lists
        tkeys = sorted(g for g in own.tolist() if succ[g] >= 0 and sdev[succ[g]] != d)
        tpos = {g: k for k, g in enumerate(tkeys)}
        carry_of_pred = {int(run_pred[k]): int(run_carry[k]) for k in range(len(runs))
                         if run_pred[k] >= 0}
        tsend_ptr, tsend_pos, trecv_ptr, trecv_carry = [0], [], [0], []
        for p in range(n_devices):
            if p != d:
                tsend_pos.extend(tpos[g] for g in tkeys if sdev[succ[g]] == p)
                preds = sorted(g for g in carry_of_pred if sdev[g] == p)
                trecv_carry.extend(carry_of_pred[g] for g in preds)
            tsend_ptr.append(len(tsend_pos))
            trecv_ptr.append(len(trecv_carry))
        a = lambda x: np.asarray(x, dtype=np.int64)
        out.append(OracleLayout(
            device=d, n_devices=n_devices, own_gid=own, halo_gid=halo, group_ptr=gptr,
            row_ptr=a(row_ptr), col=a(col), dinv=dinv_g[gid_of_local],
            t_row_ptr=a(t_row_ptr), t_col=a(t_col),
            key_rows=a([local[g] for g in key_set]), send_ptr=a(send_ptr), send_pos=a(send_pos),
            recv_ptr=a(recv_ptr), recv_slot=a(recv_slot),
            run_ptr=run_ptr, run_rows=run_rows, run_pred_gid=run_pred, run_carry=run_carry,
            n_rows=R, row_len=L, slot_row=slot_row.reshape(-1), slot_mask=mask.reshape(-1),
            slot_carry=slot_carry.reshape(-1),
            tkey_rows=a([local[g] for g in tkeys]), tsend_ptr=a(tsend_ptr), tsend_pos=a(tsend_pos),
            trecv_ptr=a(trecv_ptr), trecv_carry=a(trecv_carry),
            padding=int(padding), naive_padding=int(naive)))
    return out
