"""Temporal fusion on the GPU, mirroring the reference API (fusion.py:223-469):
PackedBatch / pack_sequences (native FFD, dgc_pack_sequences), GruCell and
gru_forward_masked running the masked recurrence as K2 (x W + b on tcgen05)
followed by K3 (dgc_rnn_fwd). Results match the reference's float64 kernel
within the fp32 tolerance (tests/test_gpu_kernels.py)."""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Mapping, Sequence

import numpy as np
import torch

from . import ops
from .layout import pack_sequences_native


@dataclass
class PackedBatch:
    """fusion.py:229-246: rows[r][p] = (entity, pos) or None, carry mask."""
    rows: list
    row_length: int
    mask: np.ndarray
    padding_count: int
    sequences: list

    @property
    def n_rows(self) -> int:
        return len(self.rows)


def pack_sequences(sequences: Sequence[tuple[int, int]]) -> PackedBatch:
    """fusion.py:278-313 (duplicate entities rejected, lengths >= 1)."""
    seqs = list(sequences)
    if len({e for e, _ in seqs}) != len(seqs):
        raise ValueError("duplicate entity in sequence list")
    for e, length in seqs:
        if length < 1:
            raise ValueError(f"sequence length must be >= 1, got {length} for {e}")
    if not seqs:
        return PackedBatch([], 0, np.zeros((0, 0), np.uint8), 0, [])
    seq, pos, mask, pad = pack_sequences_native([l for _, l in seqs])
    rows = [[(seqs[s][0], int(p)) if s >= 0 else None for s, p in zip(rs, ps)]
            for rs, ps in zip(seq.tolist(), pos.tolist())]
    return PackedBatch(rows, seq.shape[1], mask, int(pad), seqs)


@dataclass
class GruCell:
    """Same fields as the reference GruCell (fusion.py:341-361)."""
    w_update: np.ndarray
    u_update: np.ndarray
    b_update: np.ndarray
    w_reset: np.ndarray
    u_reset: np.ndarray
    b_reset: np.ndarray
    w_cand: np.ndarray
    u_cand: np.ndarray
    b_cand: np.ndarray

    @classmethod
    def coerce(cls, cell) -> "GruCell":
        return cls(*(np.asarray(getattr(cell, k), np.float64) for k in cls.__dataclass_fields__))

    @property
    def input_size(self):
        return self.w_update.shape[0]

    @property
    def hidden_size(self):
        return self.w_update.shape[1]

    def packed(self):
        """(Wx [in, 3H], U [H, 3H], b [3H]) in the kernel's (r, z, c) order."""
        Wx = np.concatenate([self.w_reset, self.w_update, self.w_cand], axis=1)
        U = np.concatenate([self.u_reset, self.u_update, self.u_cand], axis=1)
        b = np.concatenate([self.b_reset, self.b_update, self.b_cand])
        return Wx, U, b


def gru_forward_masked(cell, batch: PackedBatch, inputs: Mapping[int, np.ndarray],
                       precision: int = 3, device="cuda") -> dict:
    """GPU gru_forward_masked (fusion.py:428-469): same inputs/outputs."""
    cell = GruCell.coerce(cell)
    n_in, H = cell.input_size, cell.hidden_size
    for e, length in batch.sequences:
        feats = inputs.get(e)
        if feats is None or np.shape(feats) != (length, n_in):
            raise ValueError(f"inputs for entity {e} must have shape ({length}, {n_in})")
    if not batch.rows:
        return {}
    offs, o = {}, 0
    for e, length in batch.sequences:
        offs[e] = o
        o += length
    R, L = batch.n_rows, batch.row_length
    slot_row = np.full(R * L, -1, np.int32)
    for r, row in enumerate(batch.rows):
        for p, slot in enumerate(row):
            if slot is not None:
                slot_row[r * L + p] = offs[slot[0]] + slot[1]
    X = np.concatenate([np.asarray(inputs[e], np.float32) for e, _ in batch.sequences])
    Wx, U, b = cell.packed()
    dev = torch.device(device)
    f32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float32), device=dev)
    n = X.shape[0]
    gx = torch.empty((n, 3 * H), dtype=torch.float32, device=dev)
    Xd, Wd, Ud, bd = f32(X), f32(Wx), f32(U), f32(b)
    ops.gemm(Xd, Wd, gx, n, 3 * H, n_in, precision=precision, bias=bd)
    h = torch.empty((n, H), dtype=torch.float32, device=dev)
    save = torch.empty((n, ops.rnn_save_floats(0, H)), dtype=torch.float32, device=dev)
    sr = torch.as_tensor(slot_row, device=dev)
    sm = torch.as_tensor(np.ascontiguousarray(batch.mask.reshape(-1), np.uint8), device=dev)
    sc = torch.full((R * L,), -1, dtype=torch.int32, device=dev)
    carry = torch.zeros((1, H), dtype=torch.float32, device=dev)
    ops.rnn_fwd(0, gx, Ud, sr, sm, sc, carry, R, L, H, H, h, None, save)
    hh = h.cpu().numpy().astype(np.float64)
    return {e: hh[offs[e]:offs[e] + length] for e, length in batch.sequences}
