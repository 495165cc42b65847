"""The B200 chunk-partitioned DGNN training step behind the reference's
trainer API (simulate_epoch / run_epochs, sim.py:423-599).

One ``Shard`` = one device's share of the reference plan (its fusion groups,
SURVEY.md §8(b)). ``Shard.step`` is a generator that yields at every
collective; a ``Runner`` services the yields either with torch.distributed
NCCL (one process per GPU, the production path) or by direct device copies
among all shards of one process (``LocalRunner``: D virtual devices on one
GPU, used for parity tests and single-GPU runs of multi-device plans). The
arithmetic is identical in both.

Per epoch and shard:
  GCN layer l: Y = H_{l-1} W_l (K2) -> [K5 stale filter, MAX all-reduce of D_r,
    K6 pack, all-to-allv, unpack into halo rows] -> H_l = relu(A_hat Y + b) (K1)
  RNN layer k: gx = x Wx + b (K2) -> masked GRU/LSTM over packed runs (K3/K4)
    -> carry exchange for the next epoch (K5/K6)
  readout + CE (K2, K8) -> backward (K2/K3/K4/K1 transposed, reverse all-to-allv
  of fresh halo gradients) -> SUM all-reduce of the flat gradient (K7) ->
  Adam/SGD.
"""
from __future__ import annotations

import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import ops
from .layout import DeviceLayout, build_layout
from .model import DGNNConfig, flat_offsets, init_params, synthetic_inputs
from .plan import PlanArrays
from .stale import (EmbeddingCacheGPU, EpochLossTrace, StaleConfig, StaleMode, cache_gap_gpu,
                    filter_transmissions_gpu, threshold)


def k_segment_items(seg, T: int, fp32_chain: bool, n_sms: int = 148):
    """Work items (first k-block, k-blocks) of the K-segmented per-snapshot
    weight-gradient GEMM dW_t = X_t^T dY_t, seg = row offsets of the T snapshot
    segments (multiples of 32). fp32 (3xTF32) mode caps every TMEM chain at 16
    k-blocks; TF32 mode splits each snapshot's K evenly so the items form a
    whole number of waves (2 x n_sms when T <= 2 n_sms), the parts per snapshot
    by largest remainder. Returns (items, item_ptr) with item_ptr[t] the first
    item of snapshot t."""
    seg = np.asarray(seg, dtype=np.int64)
    total_kb = max(1, int(seg[T] // 32))
    kbs = [int(seg[t + 1] // 32 - seg[t] // 32) for t in range(T)]
    target = 2 * n_sms if T <= 2 * n_sms else -(-T // n_sms) * n_sms
    share = [k * target / total_kb for k in kbs]
    parts = [max(1, int(x)) if k else 0 for x, k in zip(share, kbs)]
    order = sorted(range(T), key=lambda t: -(share[t] - int(share[t])))
    for t in order:
        if sum(parts) >= target:
            break
        if kbs[t] > parts[t]:
            parts[t] += 1
    items, item_ptr = [], [0]
    for t in range(T):
        kb0, kb1 = int(seg[t] // 32), int(seg[t + 1] // 32)
        chunk = 16 if fp32_chain else max(1, -(-(kb1 - kb0) // max(1, parts[t])))
        for a in range(kb0, kb1, chunk):
            items.append((a, min(chunk, kb1 - a)))
        item_ptr.append(len(items))
    return items, item_ptr


@dataclass
class EpochReport:
    """Fields of the reference EpochReport (sim.py:259-303), filled with
    measured times and the reference-billed bytes of the actual send masks;
    the extra fields are additive."""
    method: str
    epoch: int
    per_device_compute_ms: list
    per_device_wall_ms: list
    spatial_traffic_bytes: int
    temporal_traffic_bytes: int
    shuffle_bytes: int
    loading_bytes: int
    padding_slots: int
    naive_padding_slots: int
    load_divergence: float
    wall_ms: float
    stale_theta: float = 0.0
    stale_d: float = 0.0
    stale_sent_bytes: int = 0
    stale_avoided_bytes: int = 0
    stale_reduction_pct: float = 0.0
    loss: float = 0.0
    exchanged_rows: int = 0
    exchanged_bytes: int = 0
    stale_detail: dict = field(default_factory=dict)

    @property
    def traffic_bytes(self) -> int:
        return self.spatial_traffic_bytes + self.temporal_traffic_bytes + self.shuffle_bytes

    def to_dict(self) -> dict:
        d = dict(self.__dict__)
        d["traffic_bytes"] = self.traffic_bytes
        return d


def _dev_i32(a, device):
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=device)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class ExchangePlan:
    """Index arrays and persistent buffers of one boundary exchange (one GCN
    layer's halo rows, or one RNN layer's carries) for the one-buffer data
    plane (csrc/exchange.cu): the per-peer send lists concatenated peer-major
    ("entries"), the per-peer receive lists, and a key -> entries CSR in
    ascending peer order for the fixed-order gradient return."""

    def __init__(self, D, send_ptr, send_pos, recv_ptr, recv_slot, width, dev, n_keys,
                 backward=True):
        send_ptr = np.asarray(send_ptr, np.int64)
        recv_ptr = np.asarray(recv_ptr, np.int64)
        n_ent = int(send_ptr[-1])
        n_recv = int(recv_ptr[-1])
        self.n_ent, self.n_recv = n_ent, n_recv
        peer_of = np.repeat(np.arange(D), np.diff(send_ptr))
        self.ent_key = _dev_i32(np.asarray(send_pos)[:n_ent], dev)
        self.ent_ptr = _dev_i32(send_ptr, dev)
        self.ent_idx = _dev_i32(np.arange(n_ent) - send_ptr[peer_of], dev)
        self.rlist = _dev_i32(np.asarray(recv_slot)[:n_recv], dev)
        self.rlist_ptr = _dev_i32(recv_ptr, dev)
        self.send_static = [int(x) for x in np.diff(send_ptr)]
        self.recv_static = [int(x) for x in np.diff(recv_ptr)]
        self.sent_host, self.recv_host = list(self.send_static), list(self.recv_static)
        order = np.argsort(np.asarray(send_pos)[:n_ent], kind="stable")  # (key, peer) order
        keys_sorted = np.asarray(send_pos)[:n_ent][order]
        self.kent = _dev_i32(order, dev)
        self.kent_ptr = _dev_i32(np.searchsorted(keys_sorted, np.arange(n_keys + 1)), dev)
        i32 = dict(dtype=torch.int32, device=dev)
        f32 = dict(dtype=torch.float32, device=dev)
        self.ent_slot = torch.zeros(max(1, n_ent), **i32)
        self.counts = torch.as_tensor(np.asarray(self.send_static, np.int32), device=dev)
        self.rcounts = torch.as_tensor(np.asarray(self.recv_static, np.int32), device=dev)
        self.sendbuf = torch.zeros(max(1, n_ent) * (width + 4), **f32)
        self.recvbuf = torch.zeros(max(1, n_recv) * (width + 4), **f32)
        if backward:
            self.backsend = torch.zeros(max(1, n_recv) * width, **f32)
            self.backrecv = torch.zeros(max(1, n_ent) * width, **f32)


class Shard:
    """One device's state: layout tensors, activations, caches, parameters."""

    def __init__(self, pa: PlanArrays, lay: DeviceLayout, cfg: DGNNConfig, params: dict,
                 X: np.ndarray, y: np.ndarray, stale: StaleConfig, n_total: int, device):
        self.pa, self.lay, self.cfg, self.stale = pa, lay, cfg, stale
        self.d, self.D = lay.device, lay.n_devices
        self.device = device
        self.n_total = n_total
        dev = device
        n, nh, H, F = lay.n_own, lay.n_halo, cfg.H, cfg.F
        self.n, self.nh, self.nloc = n, nh, n + nh
        self.prec = 3 if cfg.precision == "fp32" else 1
        # structure-encoder GEMMs: their outputs feed the ReLU masks, whose
        # flips dominate TF32 gradient error; DGC_GCN_PREC=3 keeps them 3xTF32
        self.prec_gcn = int(os.environ.get("DGC_GCN_PREC", self.prec))
        # layout on device
        self.row_ptr = _dev_i32(lay.row_ptr, dev)
        self.col = _dev_i32(lay.col, dev)
        self.t_row_ptr = _dev_i32(lay.t_row_ptr, dev)
        self.t_col = _dev_i32(lay.t_col, dev)
        self.dinv = torch.as_tensor(lay.dinv.astype(np.float32), device=dev)
        self.slot_row = _dev_i32(lay.slot_row, dev)
        self.slot_mask = torch.as_tensor(lay.slot_mask.astype(np.uint8), device=dev)
        self.slot_carry = _dev_i32(lay.slot_carry, dev)
        self.R, self.L = lay.n_rows, lay.row_len
        # instances at the last slot of their run: the only c rows the cluster LSTM writes
        if self.R and self.L:
            sr2 = np.asarray(lay.slot_row).reshape(self.R, self.L)
            nxt = np.zeros((self.R, self.L), np.uint8)
            nxt[:, :-1] = np.asarray(lay.slot_mask).reshape(self.R, self.L)[:, 1:]
            self.n_run_ends = int(((sr2 >= 0) & (nxt == 0)).sum())
        else:
            self.n_run_ends = 0
        self.nnz = lay.nnz
        self.key_rows = _dev_i32(lay.key_rows, dev)
        self.key_ncut = torch.as_tensor(lay.key_ncut.astype(np.int64), device=dev)
        self.key_ncut_total = int(lay.key_ncut.sum())
        self.tkey_rows = _dev_i32(lay.tkey_rows, dev)
        peers = [p for p in range(self.D) if p != self.d]
        self.peers = peers
        # data (snapshot padding rows of EvolveGCN layouts: zero features, label -1)
        real = lay.own_gid >= 0
        gid = np.maximum(lay.own_gid, 0)
        self.X = torch.as_tensor(np.where(real[:, None], X[gid], 0).astype(np.float32),
                                 device=dev).contiguous()
        self.y = torch.as_tensor(np.where(real, y[gid], -1).astype(np.int32), device=dev)
        self.n_real = int(real.sum())
        # parameters (flat) and optimizer state
        self.offs, P = flat_offsets(cfg)
        self.params = torch.zeros(P, dtype=torch.float32, device=dev)
        self.grads = torch.zeros(P, dtype=torch.float32, device=dev)
        self.m = torch.zeros(P, dtype=torch.float32, device=dev)
        self.v = torch.zeros(P, dtype=torch.float32, device=dev)
        for k, arr in params.items():
            self.p(k).copy_(torch.as_tensor(np.asarray(arr, np.float32)))
        # TF32 mode: every tensor-core operand is stored pre-rounded to TF32
        # (round-to-nearest) so the tcgen05 operand truncation is exact; the
        # optimizer keeps fp32 master weights in self.params.
        self.tf32 = cfg.precision == "tf32"
        # TF32 mode consumes the features at fp16 precision when they fit its
        # range (the same 10-bit mantissa; they then ship from the host in 2
        # bytes per value), else TF32-rounded (3 bytes per value)
        self.x_f16 = self.tf32 and bool(self.X.numel() % 8 == 0 and
                                        float(self.X.abs().max()) < 65504.0)
        if self.tf32:
            self.params_r = torch.zeros_like(self.params)
            ops.round_tf32(self.params, self.params_r)
            if self.x_f16:
                ops.round_f16(self.X, self.X)
            else:
                ops.round_tf32(self.X, self.X)
        else:
            self.params_r = self.params
        # activations
        G, GH = cfg.G, cfg.G * H
        f32 = dict(dtype=torch.float32, device=dev)
        self.Yext = [torch.zeros((self.nloc, H), **f32) for _ in range(2)]
        self.Hl = [torch.zeros((n, H), **f32) for _ in range(2)]
        # Single device (no halo exchange), TF32 mode: layer 1 aggregates first,
        # H1 = relu((A X) W1 + b1), so its weight gradient is (A X)^T dZ1 from the
        # forward's A X and the backward needs no transposed SpMM for layer 1
        # (one SpMM fewer per step; W1 is F x H either way). With D > 1 the
        # exchanged layer-1 embedding stays X W1 (H-wide, the reference's billing).
        # The fp32 parity mode keeps the oracle's association A (X W1): a
        # reassociated sum can flip a ReLU whose pre-activation is ~1e-7 from 0,
        # which moves single gradient entries by far more than 1e-4
        # (DGC_AGG_FIRST=1 forces the aggregate-first order there too).
        self.agg_first = (self.D == 1 and nh == 0 and cfg.F in (4, 8, 16, 32, 64, 128, 256, 512)
                          and (cfg.precision == "tf32" or os.environ.get("DGC_AGG_FIRST") == "1")
                          and not os.environ.get("DGC_TRANSFORM_FIRST"))
        self.AX = torch.zeros((n, cfg.F), **f32) if self.agg_first else None
        if self.agg_first and self.x_f16:
            # the features feed only the layer-1 aggregation: keep them resident as
            # fp16 (exact after round_f16), gathered by dgc_spmm_csr_h
            self.X = self.X.half()
        self.hw = cfg.carry_width
        self.gx = torch.zeros((n, GH), **f32)
        self.hbuf = [torch.zeros((n, self.hw), **f32) for _ in range(cfg.n_rnn)]
        # tensor-core recurrence: TF32 mode, LSTM, H in {32, 64, 128}
        self.tc_rnn = (cfg.precision == "tf32" and cfg.rnn == "lstm" and H in (32, 64, 128)
                       and os.environ.get("DGC_TC_RNN", "1") != "0")
        self.sf = (ops.rnn_tc_save_floats(H) if self.tc_rnn
                   else ops.rnn_save_floats(0 if cfg.rnn == "gru" else 1, H))
        self.save = [torch.zeros((n, self.sf), **f32) for _ in range(cfg.n_rnn)]
        self.carry = [torch.zeros((max(lay.n_carry, 1), self.hw), **f32) for _ in range(cfg.n_rnn)]
        self.logits = torch.zeros((n, cfg.C), **f32)
        self.dlogits = torch.zeros((n, cfg.C), **f32)
        self.loss_partial = torch.zeros(max(1, (n + 255) // 256), dtype=torch.float64, device=dev)
        self.dh = torch.zeros((n, H), **f32)
        self.dh2 = torch.zeros((n, H), **f32)
        self.dgx = torch.zeros((n, GH), **f32)
        self.Ut = torch.zeros((GH, H), **f32)
        self.Ut_f = [torch.zeros((GH, H), **f32) for _ in range(cfg.n_rnn)] if self.tc_rnn else None
        # fused input projection (F = H = 128 cluster recurrence): no gx tensor
        self.da_exp = min(100, max(0, int(round(math.log2(max(self.n_total, 1))))))
        self.inv_da_scale = 2.0 ** -self.da_exp
        self.fused_xproj = (self.tc_rnn and cfg.rnn == "lstm" and self.R > 0
                            and ops.rnn_fwd_tc_fused_available(H, H))
        # fp16 copies of each LSTM layer's input (the fused recurrence's gathered x):
        # written by the last GCN SpMM (layer 1) and by the previous LSTM layer
        self.x16 = ([torch.zeros((n, H), dtype=torch.float16, device=dev) for _ in range(cfg.n_rnn)]
                    if self.fused_xproj else None)
        # fp16 LSTM backward (the fused path's kernels): the BPTT writes S*dgx as
        # fp16 and [dWx; dU] = [x16; h_in16]^T dgx16, dx = dgx16 Wx16^T run as
        # fp16-operand GEMMs with alpha = 1/S (half the bytes of the 4H-wide dgx)
        self.f16_bwd = bool(self.fused_xproj)
        # fp16 readout (C % 8 == 0, C <= 32): the last LSTM layer also writes its h
        # as fp16 (x16[n_rnn]); logits = h16 Wo16 + bo, and the softmax emits
        # S-scaled fp16 dlogits for dWo = h16^T dlogits16 / S, dh = dlogits16 Wo16^T / S
        # EvolveGCN (TF32): the readout input is H2, whose fp16 copy the layer-2
        # SpMM writes (h2_16); dZ2 = (dlogits16 Wo16^T / S) * (H2 > 0) takes the
        # fp16 ReLU mask from it
        evolve = cfg.model == "evolve"
        self.f16_readout = bool(cfg.C <= 32 and cfg.C % 8 == 0 and
                                (self.f16_bwd or (evolve and self.tf32 and H % 8 == 0)))
        self.h2_16 = None
        if self.f16_readout:
            if evolve:
                self.h2_16 = torch.zeros((n, H), dtype=torch.float16, device=dev)
            else:
                self.x16.append(torch.zeros((n, H), dtype=torch.float16, device=dev))
            self.dlogits16 = torch.zeros((n, cfg.C), dtype=torch.float16, device=dev)
        if self.f16_bwd:
            self.dgx = torch.zeros((n, GH), dtype=torch.float16, device=dev)
        # fp16 LSTM output gradients: with the fp16 readout the dh the BPTT reads
        # (readout dh = dlogits16 Wo16^T, layer k's dx = dgx16 Wx16^T for layer k-1)
        # leaves its GEMM as S-scaled fp16 (S dh, the same scale as dgx16) instead
        # of fp32: half the bytes written and read back per LSTM layer
        self.dh16 = None
        if (self.f16_bwd and self.f16_readout and not evolve
                and not os.environ.get("DGC_BPTT_2SM") and os.environ.get("DGC_DH16", "1") != "0"):
            self.dh16 = [torch.zeros((n, H), dtype=torch.float16, device=dev) for _ in range(2)]
        # fused fp16 readout (dgc_readout_f16): logits, softmax-xent, S dh and dWo in
        # one tcgen05 launch that reads h16 once (replaces 4 launches)
        self.fused_readout = bool(self.dh16 is not None and H == 128 and cfg.C in (16, 32)
                                  and cfg.n_rnn > 0 and os.environ.get("DGC_FUSED_READOUT", "1") != "0")
        # EvolveGCN-O: the same kernel writes dZ2 = dh * (H2 > 0) (fp32) and the b2 partials
        self.fused_readout_evo = bool(evolve and self.f16_readout and H == 128 and cfg.C in (16, 32)
                                      and os.environ.get("DGC_FUSED_READOUT", "1") != "0")
        if self.fused_readout or self.fused_readout_evo:
            ro_tiles = 4 * max(1, (n + 127) // 128)  # partial rows per (tile, lane quadrant)
            self.loss_partial = torch.zeros(ro_tiles, dtype=torch.float64, device=dev)
            self.dl_partial = torch.zeros(ro_tiles * cfg.C, **f32)
            self.ro_grid = ops.readout_f16_grid(max(n, 1))
            self.dwo_partial = torch.zeros(self.ro_grid * H * cfg.C, **f32)
        self.params16 = None
        if self.f16_bwd or self.f16_readout:
            # fp16 mirror of the (TF32-rounded) parameters: the fp16 GEMMs' weights
            self.params16 = torch.zeros(self.params.numel(), dtype=torch.float16, device=dev)
            ops.to_f16(self.params_r, self.params16)
        if self.tc_rnn:
            self.rnn_dc_scratch = torch.zeros(((max(self.R, 1) + 127) // 128 * 128, H), **f32)
            self.rnn_tc_prows = ops.rnn_tc_tiles(max(self.R, 1), H)
        self.dYext = torch.zeros((self.nloc, H), **f32)
        # K1's row work counter (two int32, left zeroed by every launch)
        self.spmm_work = torch.zeros(2, dtype=torch.int32, device=dev)
        self.colsum_scratch = torch.zeros(2 * 148 * max(GH, cfg.C, H), **f32)
        # fused bias-gradient partial sums (produced inside the kernels that write
        # the gradient tensors, reduced in fixed order by dgc_reduce_rows)
        self.m_tiles = max(1, (n + 127) // 128)
        self.rnn_prows = ops.rnn_bwd_partial_rows(self.R, H) if self.R else 1
        if not (self.fused_readout or self.fused_readout_evo):
            self.dl_partial = torch.zeros(max(1, (n + 255) // 256) * cfg.C, **f32)
        prows = max(self.rnn_prows, ops.rnn_tc_tiles(max(self.R, 1), H))
        # one partial buffer per bias gradient: their fixed-order reductions run
        # together at the end of the backward (dgc_reduce_rows_batched, 2 launches)
        self.bp_b = [torch.zeros(4 * self.m_tiles * H, **f32) for _ in range(2)]      # b1, b2
        self.bp_r = [torch.zeros(prows * GH, **f32) for _ in range(max(cfg.n_rnn, 1))]  # br_k
        # split-K for weight gradients: ~one wave of 148 SMs
        kb = max(1, (n + 31) // 32)
        self.ksplit = max(1, min(148, kb // 4))
        n_split = ops.gemm_splits(max(n, 1), self.prec, self.ksplit)
        self.partial = torch.zeros(n_split * max(F, 2 * H) * max(GH, H, cfg.C), **f32)
        # stale caches (spatial per GCN layer, temporal per RNN layer)
        stale_on = stale.mode is not StaleMode.OFF and self.D > 1
        self.stale_on = stale_on
        self.scache = [EmbeddingCacheGPU(len(lay.key_rows), H, dev) for _ in range(2)] if stale_on else None
        self.tcache = [EmbeddingCacheGPU(len(lay.tkey_rows), self.hw, dev) for _ in range(cfg.n_rnn)] if stale_on else None
        self.evolve = cfg.model == "evolve"
        if self.evolve:
            self._init_evolve(lay, cfg, dev)
        # fp16 GCN (single device, aggregate-first, fused LSTM model): every
        # structure-encoder tensor exists once, as fp16 -- A X, H1, Y2, H2 (the
        # LSTM's x16[0]) forward; dZ2, dY2, dZ1 backward as S-scaled fp16 -- and
        # the GEMMs / SpMMs read and write them directly (fp32 accumulation)
        self.f16_gcn = bool(self.f16_bwd and self.agg_first and not self.evolve
                            and self.X.dtype == torch.float16)
        if self.f16_gcn:
            h16 = dict(dtype=torch.float16, device=dev)
            self.AX = None
            self.AX16 = torch.zeros((n, cfg.F), **h16)
            self.H1_16, self.Y16 = torch.zeros((n, H), **h16), torch.zeros((n, H), **h16)
            self.dZ2_16, self.dY16 = torch.zeros((n, H), **h16), torch.zeros((n, H), **h16)
            self.dZ1_16 = torch.zeros((n, H), **h16)
        # exchange data plane (D > 1): one record buffer per exchange, all peers
        # per launch; interior rows (no halo column) aggregate while it is in
        # flight, boundary rows after it lands
        if self.D > 1:
            rp = np.asarray(lay.row_ptr, np.int64)
            bnd_nnz = np.zeros(n, bool)
            if nh:
                hit = np.asarray(lay.col) >= n
                bnd_nnz = np.add.reduceat(hit.astype(np.int64), rp[:-1]) > 0 if len(hit) else bnd_nnz
                bnd_nnz &= np.diff(rp) > 0
            self.rows_bnd = _dev_i32(np.flatnonzero(bnd_nnz), dev)
            self.rows_int = _dev_i32(np.flatnonzero(~bnd_nnz), dev)
            deg = np.diff(rp)
            self.nnz_bnd, self.nnz_int = int(deg[bnd_nnz].sum()), int(deg[~bnd_nnz].sum())
            self.xs = [ExchangePlan(self.D, lay.send_ptr, lay.send_pos, lay.recv_ptr, lay.recv_slot,
                                    H, dev, len(lay.key_rows)) for _ in range(2)]
            self.xt = [ExchangePlan(self.D, lay.tsend_ptr, lay.tsend_pos, lay.trecv_ptr,
                                    lay.trecv_carry, self.hw, dev, len(lay.tkey_rows), backward=False)
                       for _ in range(cfg.n_rnn)]
            self.tkey_ncut = torch.ones(max(1, len(lay.tkey_rows)), dtype=torch.int64, device=dev)
            # device counters: reference-billed cut messages (spatial, temporal) of
            # this epoch's send masks; D_r per cache (read once per epoch)
            self.billed_dev = torch.zeros(2, dtype=torch.int64, device=dev)
        self.step_count = 0
        self.step_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        self.loss_sum = torch.zeros(1, dtype=torch.float64, device=dev)
        # concurrent LSTM weight-/input-gradient GEMMs (CTA split, e.g. "74,74";
        # DGC_CONC_BWD=0 runs them one after the other)
        conc = os.environ.get("DGC_CONC_BWD", "74,74")
        self.conc_split = None if conc in ("0", "") else tuple(int(v) for v in conc.split(","))
        self._side = torch.cuda.Stream(dev) if self.conc_split else None
        self._ev_fork, self._ev_join = torch.cuda.Event(), torch.cuda.Event()
        self.events = None
        self.timing = None  # list of (start, end) events of compute-stream stalls

    def _init_evolve(self, lay, cfg, dev):
        """Per-snapshot weight machinery of EvolveGCN-O (C3)."""
        H, T = cfg.H, cfg.T
        f32 = dict(dtype=torch.float32, device=dev)
        seg = lay.seg_ptr.astype(np.int64)
        assert len(seg) == T + 1, (len(seg), T)
        m_tiles = max(1, self.n // 128)
        tile_seg = np.zeros(m_tiles, np.int32)
        for t in range(T):
            tile_seg[seg[t] // 128:seg[t + 1] // 128] = t
        self.seg_of_mtile = torch.as_tensor(tile_seg, device=dev)
        items, item_ptr = k_segment_items(seg, T, self.prec == 3)
        self.kitems = torch.as_tensor(np.asarray(items, np.int32).reshape(-1), device=dev)
        self.n_kitems = len(items)
        self.item_ptr = torch.as_tensor(np.asarray(item_ptr, np.int32), device=dev)
        Fmax = max(cfg.F, H)
        self.evo_partial = torch.zeros(max(1, self.n_kitems) * Fmax * H, **f32)
        self.evo = []
        for Fl in (cfg.F, H):
            e = dict(Fl=Fl,
                     Wstack=torch.zeros(((T + 1) * Fl, H), **f32),
                     sv=[torch.zeros((Fl, T * H), **f32) for _ in range(5)],  # r z c w rw
                     dW_direct=torch.zeros((T * Fl, H), **f32),
                     da_all=torch.zeros((3 * Fl, T * H), **f32))
            e["da"] = [e["da_all"][i * Fl:(i + 1) * Fl] for i in range(3)]  # r z c, contiguous
            self.evo.append(e)
        self.evo_gsplit = max(1, min(64, (T * H) // 128))
        self.evo_gpartial = torch.zeros(
            ops.gemm_splits(T * H, self.prec, self.evo_gsplit) * 3 * Fmax * Fmax, **f32)
        # dS_r, dS_z, dP_c share the operand w: one M = 3 F_l GEMM when their
        # gradients are adjacent in the flat buffer (param_shapes order Sr Sz Pc Qc)
        self.evo_stack3 = all(
            self.offs[f"Sz{l}"][0] == self.offs[f"Sr{l}"][0] + Fl * Fl
            and self.offs[f"Pc{l}"][0] == self.offs[f"Sz{l}"][0] + Fl * Fl
            for l, Fl in ((1, cfg.F), (2, H)))

    def p(self, name):
        o, shape = self.offs[name]
        n = int(np.prod(shape))
        return self.params[o:o + n].view(*shape)

    def _x16_out(self, l):
        """fp16 copy target of GCN layer l's output: the first LSTM layer's x16, or
        (EvolveGCN, fp16 readout) the readout's input h2_16."""
        if l == 1 and self.evolve:
            return self.h2_16
        return self.x16[0] if (self.x16 is not None and l == 1 and not self.evolve) else None

    def p16(self, name):
        """fp16 view of a parameter (the fp16-operand GEMMs' weights)."""
        o, shape = self.offs[name]
        n = int(np.prod(shape))
        return self.params16[o:o + n].view(*shape)

    def pr(self, name):
        """GEMM operand view of a parameter (TF32-rounded copy in TF32 mode)."""
        o, shape = self.offs[name]
        n = int(np.prod(shape))
        return self.params_r[o:o + n].view(*shape)

    def g(self, name):
        o, shape = self.offs[name]
        n = int(np.prod(shape))
        return self.grads[o:o + n].view(*shape)

    def gp(self, name):
        """data pointer offset helper for column slices"""
        return self.offs[name][0]

    # -- exchanges ------------------------------------------------------------
    def _stale_select(self, r, trace, Y, keys, cache, ncut, billed):
        """Stale decision of one cache on the device (K5): distances, one MAX
        all-reduce of D_r (the reference's one global cache, sim.py:455-459),
        theta = coef * D_r in the select kernel (threshold(), stale.py:97-108,
        with coef from the loss trace known on the host), billed messages
        accumulated on the device. No host round trip. Returns (coef, D_r
        device tensor or None); the send mask is left in cache.send."""
        if r >= 2:
            coef = threshold(trace, r, 1.0, self.stale)  # threshold is linear in D_r
            cache_gap_gpu(Y, keys, cache)
            dmax = yield ("max", cache.dmax)
            ops.stale_select_dev(Y, keys, cache.dist, dmax, coef, cache.values, cache.cached,
                                 cache.send, cache.width, ncut=ncut, billed=billed)
            return coef, dmax
        ops.stale_select_dev(Y, keys, cache.dist, None, 0.0, cache.values, cache.cached,
                             cache.send, cache.width, ncut=ncut, billed=billed, theta=0.0)
        return 0.0, None

    def _send(self, xp: "ExchangePlan", Y, width, keys, cache):
        """Pack this exchange's records (stale-compacted on the device when a
        cache is given) and start the all-to-allv. Returns the runner token."""
        slot = None
        if cache is not None:
            ops.exchange_rank(xp.ent_key, xp.ent_ptr, self.D, cache.send, xp.ent_slot, xp.counts)
            slot = xp.ent_slot
        ops.exchange_pack(Y, width, keys, xp.ent_key, xp.ent_idx, slot, xp.sendbuf)
        tok = yield ("a2a_start", xp.sendbuf, None if cache is not None else xp.send_static,
                     xp.counts, xp.recvbuf, width + 4, xp.recv_static, xp.rcounts)
        return tok

    def _land(self, xp: "ExchangePlan", tok, width, dst):
        """Finish an all-to-allv and unpack it into dst (on the runner's comm
        stream when it has one: overlaps the compute stream). Returns the
        event the consumer waits on (None: same stream)."""
        res = yield ("a2a_finish", tok)
        xp.sent_host, xp.recv_host = res["send_counts"], res["recv_counts"]
        st = res.get("stream")
        ctx = torch.cuda.stream(st) if st is not None else _nullctx()
        with ctx:
            ops.exchange_unpack(xp.recvbuf, width, xp.rcounts, self.D, xp.rlist, xp.rlist_ptr,
                                sum(xp.recv_host), dst)
            ev = None
            if st is not None:
                ev = torch.cuda.Event()
                ev.record(st)
        return ev

    def _wait(self, ev):
        if ev is not None:
            self._stall(lambda: torch.cuda.current_stream(self.device).wait_event(ev))

    def _stall(self, fn):
        """Run fn (a stream wait / blocking collective on the compute stream),
        timing the compute stream's stall when per-device timing is on."""
        if self.timing is None:
            return fn()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        self.timing.append((a, b))
        return out

    # -- one training step ----------------------------------------------------
    def step(self, r: int, trace: EpochLossTrace):
        cfg, H, n, prec = self.cfg, self.cfg.H, self.n, self.prec
        G, GH = cfg.G, cfg.G * cfg.H
        cell = 0 if cfg.rnn == "gru" else 1
        rflag = 0x100 if self.tf32 else 0   # DGC_RNN_ROUND_TF32
        rnd2 = 2 if self.tf32 else 0        # spmm: round output to TF32
        info = {"coef": {}, "d_r": {}, "rows": 0, "xbytes": 0}
        D = self.D
        pending_t = []  # temporal carry exchanges: landed at the end of the step
        if D > 1 and self.stale_on:
            self.billed_dev.zero_()
        # ---------------- forward: structure encoder ----------------
        if self.evolve:  # EvolveGCN-O: W_t for every snapshot, per layer
            for l, e in enumerate(self.evo, start=1):
                ops.evolve_fwd(e["Fl"], H, cfg.T, self.p(f"W{l}_0"),
                               *[self.p(f"{k}{l}") for k in ("Sr", "Sz", "Pc", "Qc")], self.p(f"Br{l}"),
                               self.p(f"Bz{l}"), self.p(f"Bc{l}"), e["Wstack"], e["sv"],
                               rnd=self.tf32)
        hin, ldin, kin = self.X, cfg.F, cfg.F
        for l, (W, b) in enumerate((("W1", "b1"), ("W2", "b2"))):
            Y = self.Yext[l]
            if l == 0 and self.f16_gcn:  # A X and H1 = relu((A X) W1 + b1), fp16 only
                ops.spmm_csr_h(self.row_ptr, self.col, self.dinv, self.X, None, None, act=0,
                               nnz=self.nnz, n_cols=self.nloc, work=self.spmm_work,
                               out16=self.AX16)
                ops.gemm_f16(self.AX16, self.p16(W), None, n, H, kin, lda=kin, bias=self.p(b),
                             act=1, C16=self.H1_16)
                continue
            if l == 1 and self.f16_gcn:  # Y2 = H1 W2 and H2 = relu(A Y2 + b2), fp16 only
                ops.gemm_f16(self.H1_16, self.p16(W), None, n, H, H, lda=H, C16=self.Y16)
                ops.spmm_csr_h(self.row_ptr, self.col, self.dinv, self.Y16, self.p(b), None, act=1,
                               nnz=self.nnz, n_cols=self.nloc, work=self.spmm_work,
                               out16=self.x16[0])
                continue
            if l == 0 and self.agg_first:
                if self.X.dtype == torch.float16:
                    ops.spmm_csr_h(self.row_ptr, self.col, self.dinv, self.X, None, self.AX,
                                   act=rnd2, nnz=self.nnz, n_cols=self.nloc, work=self.spmm_work)
                else:
                    ops.spmm_csr(self.row_ptr, self.col, self.dinv, self.X, None, self.AX,
                                 act=rnd2, nnz=self.nnz, n_cols=self.nloc, work=self.spmm_work)
                oact = 1 | rnd2  # ReLU (+ TF32 rounding of the next GEMM's operand)
                if self.evolve:
                    ops.gemm_segmented(self.AX, self.evo[0]["Wstack"][kin:], self.Hl[0], n, H, kin,
                                       lda=kin, precision=prec, seg_of_mtile=self.seg_of_mtile,
                                       b_nseg=cfg.T, bias=self.p(b), act=oact)
                else:
                    ops.gemm(self.AX, self.pr(W), self.Hl[0], n, H, kin, lda=kin,
                             precision=self.prec_gcn, bias=self.p(b), act=oact)
                hin, ldin, kin = self.Hl[0], H, H
                continue
            if self.evolve:
                e = self.evo[l]
                ops.gemm_segmented(hin, e["Wstack"][kin:], Y, n, H, kin, lda=ldin, precision=prec,
                                   seg_of_mtile=self.seg_of_mtile, b_nseg=cfg.T)
            else:
                ops.gemm(hin, self.pr(W), Y, n, H, kin, lda=ldin, precision=self.prec_gcn)
            if D > 1:
                cache = self.scache[l] if self.stale_on else None
                xp = self.xs[l]
                if cache is not None:
                    coef, dr = yield from self._stale_select(r, trace, Y, self.key_rows, cache,
                                                             self.key_ncut, self.billed_dev[0:1])
                    info["coef"][f"s{l}"], info["d_r"][f"s{l}"] = coef, dr
                tok = yield from self._send(xp, Y, H, self.key_rows, cache)
                # interior rows need no halo row: they aggregate while the exchange flies
                ops.spmm_csr_rows(self.row_ptr, self.col, self.dinv, Y, self.p(b), self.Hl[l],
                                  act=1 | rnd2, rows=self.rows_int, nnz=self.nnz_int,
                                  n_cols=self.rows_int.numel(), out16=self._x16_out(l), work=self.spmm_work)
                ev = yield from self._land(xp, tok, H, Y)
                info["rows"] += sum(xp.sent_host)
                info["xbytes"] += sum(xp.sent_host) * (H + 4) * 4
                self._wait(ev)
                ops.spmm_csr_rows(self.row_ptr, self.col, self.dinv, Y, self.p(b), self.Hl[l],
                                  act=1 | rnd2, rows=self.rows_bnd, nnz=self.nnz_bnd,
                                  n_cols=self.nh + self.rows_bnd.numel(), out16=self._x16_out(l), work=self.spmm_work)
            else:
                ops.spmm_csr(self.row_ptr, self.col, self.dinv, Y, self.p(b), self.Hl[l],
                             act=1 | rnd2, nnz=self.nnz, n_cols=self.nloc, out16=self._x16_out(l), work=self.spmm_work)
            hin, ldin, kin = self.Hl[l], H, H
        # ---------------- forward: time encoder ----------------
        xr, ldx = self.Hl[1], H
        for k in range(cfg.n_rnn if not self.evolve else 0):
            hb = self.hbuf[k]
            c_out = hb[:, H:] if cell == 1 else None
            if self.fused_xproj:
                # x Wx + h U + b in one tensor-core recurrence (fp16 operands,
                # resident weights; no gx round trip)
                # the fp16 copy feeds the next layer (or the fp16 readout): the
                # fp32 h is then needed only at run ends (the carries)
                h16 = self.x16[k + 1] if k + 1 < len(self.x16) else None
                ops.lstm_fwd_tc_f16x(self.x16[k], self.p(f"Wx{k}"), self.p(f"U{k}"),
                                     self.p(f"br{k}"), self.slot_row, self.slot_mask,
                                     self.slot_carry, self.carry[k], self.R, self.L, H, self.hw,
                                     hb, c_out, self.save[k],
                                     h_out16=h16, c_rows=self.n_run_ends,
                                     h32_run_ends_only=h16 is not None)
            elif self.tc_rnn:
                ops.gemm(xr, self.pr(f"Wx{k}"), self.gx, n, GH, H, lda=ldx, precision=prec,
                         bias=self.p(f"br{k}"))
                ops.transpose(self.pr(f"U{k}"), self.Ut_f[k])
                ops.rnn_fwd_tc(cell, self.gx, self.Ut_f[k], self.slot_row, self.slot_mask,
                               self.slot_carry, self.carry[k], self.R, self.L, H, self.hw, hb,
                               c_out, self.save[k])
            else:
                ops.gemm(xr, self.pr(f"Wx{k}"), self.gx, n, GH, H, lda=ldx, precision=prec,
                         bias=self.p(f"br{k}"))
                ops.rnn_fwd(cell | rflag, self.gx, self.pr(f"U{k}"), self.slot_row,
                            self.slot_mask, self.slot_carry, self.carry[k], self.R, self.L, H,
                            self.hw, hb, c_out, self.save[k])
            if D > 1:
                # carries for the NEXT epoch (carry-from-cache): the exchange is
                # landed at the end of the step, overlapping everything after it
                cache = self.tcache[k] if self.stale_on else None
                if cache is not None:
                    coef, dr = yield from self._stale_select(r, trace, hb, self.tkey_rows, cache,
                                                             self.tkey_ncut, self.billed_dev[1:2])
                    info["coef"][f"t{k}"], info["d_r"][f"t{k}"] = coef, dr
                tok = yield from self._send(self.xt[k], hb, self.hw, self.tkey_rows, cache)
                pending_t.append((k, tok))
            xr, ldx = hb, self.hw
        # ---------------- readout + loss ----------------
        f16r = self.f16_readout and (cfg.n_rnn > 0 or self.evolve)
        if self.fused_readout:  # logits, loss, S dh (into dh16[0]) and dWo partials
            ops.readout_f16(self.x16[cfg.n_rnn], self.p16("Wo"), self.p("bo"), self.y, cfg.C,
                            1.0 / self.n_total, 2.0 ** self.da_exp, self.dh16[0], self.loss_partial,
                            self.dl_partial, self.dwo_partial)
        elif self.fused_readout_evo:  # + dZ2 = dh * (H2 > 0) into self.dh, b2 partials
            ops.readout_f16_evolve(self.h2_16, self.p16("Wo"), self.p("bo"), self.y, cfg.C,
                                   1.0 / self.n_total, 2.0 ** self.da_exp, self.dh, self.bp_b[1],
                                   self.loss_partial, self.dl_partial, self.dwo_partial)
        elif f16r:
            xr16 = self.h2_16 if self.evolve else self.x16[cfg.n_rnn]
            ops.gemm_f16(xr16, self.p16("Wo"), self.logits, n, cfg.C, H, lda=H, bias=self.p("bo"))
            ops.softmax_xent(self.logits, self.y, cfg.C, 1.0 / self.n_total, None,
                             self.loss_partial, dl_partial=self.dl_partial,
                             dlogits16=self.dlogits16, scale16=2.0 ** self.da_exp)
        else:
            ops.gemm(xr, self.pr("Wo"), self.logits, n, cfg.C, H, lda=ldx, precision=prec,
                     bias=self.p("bo"))
            ops.softmax_xent(self.logits, self.y, cfg.C, 1.0 / self.n_total, self.dlogits,
                             self.loss_partial, round_tf32=self.tf32, dl_partial=self.dl_partial)
        # ---------------- backward ----------------
        ops.zero_(self.grads)
        ks, part = self.ksplit, self.partial
        if self.fused_readout or self.fused_readout_evo:
            pass  # dWo partials came with the forward readout (reduced below)
        elif f16r:
            ops.gemm_f16(xr16, self.dlogits16, self.g("Wo"), H, cfg.C, n, a_mn=True, lda=H,
                         alpha=self.inv_da_scale, k_splits=ks, partial=part)
        else:
            ops.gemm(xr, self.dlogits, self.g("Wo"), H, cfg.C, n, a_mn=True, lda=ldx,
                     precision=prec, k_splits=ks, partial=part)
        if self.fused_readout or self.fused_readout_evo:
            rjobs = [(self.dl_partial, 4 * max(1, (n + 127) // 128), cfg.C, self.g("bo")),
                     (self.dwo_partial, self.ro_grid, H * cfg.C, self.g("Wo"))]
        else:
            rjobs = [(self.dl_partial, max(1, (n + 255) // 256), cfg.C, self.g("bo"))]
        if self.fused_readout_evo:  # dZ2 and its b2 partials came with the forward readout
            rjobs.append((self.bp_b[1], 4 * self.m_tiles, H, self.g("b2")))
        elif f16r and self.evolve:  # dZ2 = (dlogits Wo^T) * (H2 > 0), b2 fused
            ops.gemm_f16(self.dlogits16, self.p16("Wo"), self.dh, n, H, cfg.C, b_mn=False,
                         ldb=cfg.C, alpha=self.inv_da_scale, relu16=self.h2_16,
                         colsum_partial=self.bp_b[1])
            rjobs.append((self.bp_b[1], 4 * self.m_tiles, H, self.g("b2")))
        elif self.fused_readout:
            pass  # S dh16 came with the forward readout
        elif f16r and self.dh16 is not None:  # S dh as fp16 (the BPTT unscales it)
            ops.gemm_f16(self.dlogits16, self.p16("Wo"), None, n, H, cfg.C, b_mn=False,
                         ldb=cfg.C, alpha=self.inv_da_scale, C16=self.dh16[0],
                         c16_scale=2.0 ** self.da_exp)
        elif f16r:
            ops.gemm_f16(self.dlogits16, self.p16("Wo"), self.dh, n, H, cfg.C, b_mn=False,
                         ldb=cfg.C, alpha=self.inv_da_scale)
        elif self.evolve:  # no time encoder: dZ2 = (dlogits Wo^T) * (H2 > 0), b2 fused
            ops.gemm(self.dlogits, self.pr("Wo"), self.dh, n, H, cfg.C, b_mn=False, ldb=cfg.C,
                     precision=prec, relu_src=self.Hl[1], colsum_partial=self.bp_b[1])
            rjobs.append((self.bp_b[1], 4 * self.m_tiles, H, self.g("b2")))
        else:
            ops.gemm(self.dlogits, self.pr("Wo"), self.dh, n, H, cfg.C, b_mn=False, ldb=cfg.C,
                     precision=prec)
        for k in reversed(range(cfg.n_rnn if not self.evolve else 0)):
            if self.tc_rnn:
                # the H = 128 cluster BPTT multiplies fp16 S*da by resident fp16 U:
                # S = 2^round(log2 n_total) lifts da ~ 1/n_total into fp16's normal range
                ops.rnn_bwd_tc(cell | rflag | (self.da_exp << 16), self.pr(f"U{k}"), self.slot_row,
                               self.slot_mask, self.R, self.L, H, self.save[k],
                               self.dh16[0] if self.dh16 is not None else self.dh, self.dgx,
                               self.rnn_dc_scratch, bias_partial=self.bp_r[k])
                rjobs.append((self.bp_r[k], self.rnn_tc_prows, GH, self.g(f"br{k}")))
            else:
                ops.transpose(self.pr(f"U{k}"), self.Ut)
                ops.rnn_bwd(cell | rflag, self.Ut, self.slot_row, self.slot_mask, self.R, self.L,
                            H, self.save[k], self.dh, self.dgx, bias_partial=self.bp_r[k])
                rjobs.append((self.bp_r[k], self.rnn_prows, GH, self.g(f"br{k}")))
            xin, ldxin = (self.Hl[1], H) if k == 0 else (self.hbuf[k - 1], self.hw)
            gU = self.g(f"U{k}")
            conc = self.f16_bwd and self.conc_split is not None
            if conc:
                # the weight-gradient GEMM and the input-gradient GEMM below both
                # stream dgx (4H fp16 per instance): run them side by side on
                # parts of the machine so the second reader of a dgx tile finds
                # it in L2 (one HBM pass instead of two)
                main = torch.cuda.current_stream()
                self._ev_fork.record(main)
                self._side.wait_event(self._ev_fork)
                prev_cap = ops.gemm_max_ctas(self.conc_split[0])
            if self.f16_bwd:
                # [dWx; dU] = [x16; h_in16]^T (S dgx16) / S, fp16 operands, one launch
                with torch.cuda.stream(self._side if conc else torch.cuda.current_stream()):
                    ops.gemm_f16_stacked_a(self.x16[k], self.save[k].view(torch.float16), self.dgx,
                                           self.g(f"Wx{k}"), H, 2 * H, GH, n, a_mn=True, lda0=H,
                                           lda1=2 * self.sf, ldb=GH, ldc=GH,
                                           alpha=self.inv_da_scale, k_splits=ks, partial=part)
                if conc:
                    ops.gemm_max_ctas(self.conc_split[1])
            elif cell == 1 and H % 128 == 0:
                # [dWx; dU] = [x; h_in]^T dgx in ONE launch: dgx is streamed once
                # (Wx{k} and U{k} are adjacent in the flat gradient buffer)
                ops.gemm_stacked_a(xin, self.save[k], self.dgx, self.g(f"Wx{k}"), H, 2 * H, GH, n,
                                   a_mn=True, lda0=ldxin, lda1=self.sf, ldb=GH, ldc=GH,
                                   precision=prec, k_splits=ks, partial=part)
            else:
                ops.gemm(xin, self.dgx, self.g(f"Wx{k}"), H, GH, n, a_mn=True, lda=ldxin,
                         precision=prec, k_splits=ks, partial=part)
                if cell == 0:
                    ops.gemm(self.save[k], self.dgx, gU, H, 2 * H, n, a_mn=True, lda=self.sf,
                             ldb=GH, ldc=GH, precision=prec, k_splits=ks, partial=part)
                    ops.gemm(self.save[k][:, H:], self.dgx[:, 2 * H:], gU[:, 2 * H:], H, H, n,
                             a_mn=True, lda=self.sf, ldb=GH, ldc=GH, precision=prec, k_splits=ks,
                             partial=part)
                else:
                    ops.gemm(self.save[k], self.dgx, gU, H, GH, n, a_mn=True, lda=self.sf,
                             ldb=GH, ldc=GH, precision=prec, k_splits=ks, partial=part)
            relu_src = self.Hl[1] if k == 0 else None
            if self.f16_gcn and k == 0:  # dZ2 = (dgx Wx^T) * (H2 > 0) as S-scaled fp16
                ops.gemm_f16(self.dgx, self.p16(f"Wx{k}"), None, n, H, GH, b_mn=False, ldb=GH,
                             alpha=self.inv_da_scale, relu16=self.x16[0],
                             colsum_partial=self.bp_b[1], C16=self.dZ2_16,
                             c16_scale=2.0 ** self.da_exp)
            elif self.f16_bwd and self.dh16 is not None and k > 0:  # S dx as fp16
                ops.gemm_f16(self.dgx, self.p16(f"Wx{k}"), None, n, H, GH, b_mn=False, ldb=GH,
                             alpha=self.inv_da_scale, C16=self.dh16[1],
                             c16_scale=2.0 ** self.da_exp)
            elif self.f16_bwd:
                ops.gemm_f16(self.dgx, self.p16(f"Wx{k}"), self.dh2, n, H, GH, b_mn=False, ldb=GH,
                             alpha=self.inv_da_scale, relu_src=relu_src,
                             colsum_partial=self.bp_b[1] if k == 0 else None)
            else:
                ops.gemm(self.dgx, self.pr(f"Wx{k}"), self.dh2, n, H, GH, b_mn=False, ldb=GH,
                         precision=prec, relu_src=relu_src,
                         colsum_partial=self.bp_b[1] if k == 0 else None)
            if conc:  # join before the next BPTT rewrites dgx
                ops.gemm_max_ctas(prev_cap)
                self._ev_join.record(self._side)
                main.wait_event(self._ev_join)
            if k == 0:  # dZ2 = dH2 * (H2 > 0): its column sums are the b2 gradient
                rjobs.append((self.bp_b[1], 4 * self.m_tiles, H, self.g("b2")))
            self.dh, self.dh2 = self.dh2, self.dh
            if self.dh16 is not None:
                self.dh16.reverse()
        dZ = self.dh  # = dH2 * (H2 > 0), fused into the last GEMM epilogue
        for l in (1, 0):
            W, b = ("W1", "b1") if l == 0 else ("W2", "b2")
            if self.f16_gcn:  # S-scaled fp16 gradients, alpha = 1/S in every contraction
                inv, S = self.inv_da_scale, 2.0 ** self.da_exp
                if l == 1:
                    ops.spmm_csr_h(self.t_row_ptr, self.t_col, self.dinv, self.dZ2_16, None, None,
                                   act=0, nnz=self.nnz, n_cols=n, work=self.spmm_work,
                                   out16=self.dY16, name="spmm_csr_t")
                    ops.gemm_f16(self.H1_16, self.dY16, self.g(W), H, H, n, a_mn=True, lda=H,
                                 ldb=H, alpha=inv, k_splits=ks, partial=part)
                    ops.gemm_f16(self.dY16, self.p16(W), None, n, H, H, b_mn=False, ldb=H,
                                 alpha=inv, relu16=self.H1_16, colsum_partial=self.bp_b[0],
                                 C16=self.dZ1_16, c16_scale=S)
                    rjobs.append((self.bp_b[0], 4 * self.m_tiles, H, self.g("b1")))
                else:
                    ops.gemm_f16(self.AX16, self.dZ1_16, self.g(W), cfg.F, H, n, a_mn=True,
                                 lda=cfg.F, ldb=H, alpha=inv, k_splits=ks, partial=part)
                continue
            if l == 0 and self.agg_first:  # dW1 = (A X)^T dZ1: no transposed SpMM
                if self.evolve:
                    ops.gemm_segmented(self.AX, dZ, self.evo[0]["dW_direct"], cfg.F, H, n,
                                       a_mn=True, lda=cfg.F, ldb=H, precision=prec,
                                       kitems=self.kitems, n_kitems=self.n_kitems,
                                       item_ptr=self.item_ptr, n_seg=cfg.T, partial=self.evo_partial)
                else:
                    ops.gemm(self.AX, dZ, self.g(W), cfg.F, H, n, a_mn=True, lda=cfg.F, ldb=H,
                             precision=prec, k_splits=ks, partial=part)
                continue
            if D > 1:
                # halo block first: its gradients go back to their owners while
                # the own block aggregates (Appendix B.4: only fresh rows return)
                xp = self.xs[l]
                ops.spmm_csr_rows(self.t_row_ptr, self.t_col, self.dinv, dZ, None, self.dYext,
                                  act=rnd2, n_rows=self.nh, row_begin=n, name="spmm_csr_t", work=self.spmm_work)
                ops.exchange_pack_back(xp.recvbuf, H, xp.rcounts, D, xp.rlist, xp.rlist_ptr,
                                       sum(xp.recv_host), self.dYext, xp.backsend)
                tok = yield ("a2a_start", xp.backsend, list(xp.recv_host), None, xp.backrecv, H,
                             list(xp.sent_host), None)
                ops.spmm_csr_rows(self.t_row_ptr, self.t_col, self.dinv, dZ, None, self.dYext,
                                  act=rnd2, n_rows=n, row_begin=0, nnz=self.nnz, n_cols=n,
                                  name="spmm_csr_t", work=self.spmm_work)
                res = yield ("a2a_finish", tok)
                info["xbytes"] += sum(xp.recv_host) * H * 4
                if res.get("stream") is not None:
                    ev = torch.cuda.Event()
                    ev.record(res["stream"])
                    self._wait(ev)
                ops.exchange_add_back(xp.backrecv, H, self.key_rows, xp.kent_ptr, xp.kent,
                                      xp.ent_slot if self.stale_on else None, self.dYext)
            else:
                ops.spmm_csr(self.t_row_ptr, self.t_col, self.dinv, dZ, None, self.dYext,
                             act=rnd2, nnz=self.nnz, n_cols=n, work=self.spmm_work)
            hin_l, ldin_l, kin_l = (self.X, cfg.F, cfg.F) if l == 0 else (self.Hl[0], H, H)
            if self.evolve:
                e = self.evo[l]
                ops.gemm_segmented(hin_l, self.dYext, e["dW_direct"], kin_l, H, n, a_mn=True,
                                   lda=ldin_l, ldb=H, precision=prec, kitems=self.kitems,
                                   n_kitems=self.n_kitems, item_ptr=self.item_ptr, n_seg=cfg.T,
                                   partial=self.evo_partial)
                if l == 1:
                    ops.gemm_segmented(self.dYext, e["Wstack"][kin_l:], self.dh2, n, H, H,
                                       b_mn=False, ldb=H, precision=prec, relu_src=self.Hl[0],
                                       seg_of_mtile=self.seg_of_mtile, b_nseg=cfg.T,
                                       colsum_partial=self.bp_b[0])
                    rjobs.append((self.bp_b[0], 4 * self.m_tiles, H, self.g("b1")))
                    dZ = self.dh2
                continue
            ops.gemm(hin_l, self.dYext, self.g(W), kin_l, H, n, a_mn=True, lda=ldin_l, ldb=H,
                     precision=prec, k_splits=ks, partial=part)
            if l == 1:
                ops.gemm(self.dYext, self.pr("W2"), self.dh2, n, H, H, b_mn=False, ldb=H,
                         precision=prec, relu_src=self.Hl[0], colsum_partial=self.bp_b[0])
                rjobs.append((self.bp_b[0], 4 * self.m_tiles, H, self.g("b1")))
                dZ = self.dh2
        if self.evolve:  # BPTT through the weight evolution, gate-matrix grads by K2
            for l, e in enumerate(self.evo, start=1):
                Fl, TH = e["Fl"], cfg.T * H
                ops.evolve_bwd(Fl, H, cfg.T, self.pr(f"Sr{l}"), self.pr(f"Sz{l}"),
                               self.pr(f"Pc{l}"), self.pr(f"Qc{l}"), e["sv"], e["dW_direct"],
                               self.g(f"W{l}_0"), e["da"],
                               (self.g(f"Br{l}"), self.g(f"Bz{l}"), self.g(f"Bc{l}")),
                               rnd=self.tf32)
                if self.evo_stack3:  # [dS_r; dS_z; dP_c] = [da_r; da_z; da_c] w^T
                    gS = self.grads[self.offs[f"Sr{l}"][0]:self.offs[f"Sr{l}"][0] + 3 * Fl * Fl]
                    ops.gemm(e["da_all"], e["sv"][3], gS.view(3 * Fl, Fl), 3 * Fl, Fl, TH,
                             b_mn=False, ldb=TH, precision=prec, k_splits=self.evo_gsplit,
                             partial=self.evo_gpartial)
                    pairs = (("Qc", e["da"][2], e["sv"][4]),)
                else:
                    pairs = (("Sr", e["da"][0], e["sv"][3]), ("Sz", e["da"][1], e["sv"][3]),
                             ("Pc", e["da"][2], e["sv"][3]), ("Qc", e["da"][2], e["sv"][4]))
                for k, da, op in pairs:
                    ops.gemm(da, op, self.g(f"{k}{l}"), Fl, Fl, TH, b_mn=False, ldb=TH,
                             precision=prec, k_splits=self.evo_gsplit, partial=self.evo_gpartial)
        for j0 in range(0, len(rjobs), 8):  # bias gradients, fixed order, 2 launches
            ops.reduce_rows_batched(rjobs[j0:j0 + 8])
        # ---------------- land the carries, all-reduces, update ----------------
        for k, tok in pending_t:
            xp = self.xt[k]
            ev = yield from self._land(xp, tok, self.hw, self.carry[k])
            info["rows"] += sum(xp.sent_host)
            info["xbytes"] += sum(xp.sent_host) * (self.hw + 4) * 4
            self._wait(ev)
        # loss sum + the device step count (the epoch is replayable as a graph)
        adam = cfg.optimizer == "adam"
        ops.epoch_finish(self.loss_partial, self.loss_sum, self.step_dev if adam else None)
        loss_local = self.loss_sum
        info["loss_sum"] = (yield ("sum", loss_local)) if D > 1 else loss_local
        if D > 1:
            yield ("sum", self.grads)
        self.step_count += 1
        if adam:
            ops.adam_mirror(self.params, self.grads, self.m, self.v, cfg.lr, cfg.beta1, cfg.beta2,
                            cfg.eps, self.step_dev, p_r=self.params_r if self.tf32 else None,
                            p16=self.params16)
            return info
        ops.sgd(self.params, self.grads, self.m, cfg.lr, cfg.momentum)
        if self.tf32:
            ops.round_tf32(self.params, self.params_r)
        if self.params16 is not None:
            ops.to_f16(self.params_r, self.params16)
        return info


# -- runners ------------------------------------------------------------------

class LocalRunner:
    """Services the collectives of all shards of one process by direct device
    copies (D virtual devices on one GPU). The shards advance in lock-step:
    every shard yields the same request kind at the same point of the step.

    With ``timing`` (a list per shard), each shard's generator segments are
    bracketed by CUDA events: its compute time is the sum of its segments."""

    def __init__(self):
        self.timing = None
        self._tokens = {}

    def run(self, gens):
        results = [None] * len(gens)
        reqs = [self._advance(i, g, None, first=True) for i, g in enumerate(gens)]
        live = [True] * len(gens)
        for i, r in enumerate(reqs):
            if isinstance(r, _Done):
                results[i], live[i] = r.value, False
        while any(live):
            kind = next(r for r, a in zip(reqs, live) if a)[0]
            outs = self._service(kind, reqs)
            for i, g in enumerate(gens):
                if not live[i]:
                    continue
                r = self._advance(i, g, outs[i])
                if isinstance(r, _Done):
                    results[i], live[i] = r.value, False
                else:
                    reqs[i] = r
        return results

    def _advance(self, i, g, value, first=False):
        a = b = None
        if self.timing is not None:
            a = torch.cuda.Event(enable_timing=True)
            a.record()
        try:
            out = next(g) if first else g.send(value)
        except StopIteration as stop:
            out = _Done(stop.value)
        if a is not None:
            b = torch.cuda.Event(enable_timing=True)
            b.record()
            self.timing[i].append((a, b))
        return out

    def _service(self, kind, reqs):
        D = len(reqs)
        if kind == "max":
            m = torch.stack([r[1].reshape(-1)[0] for r in reqs]).max().reshape(1)
            return [m for _ in reqs]
        if kind == "sum":
            if D == 1:  # nothing to combine
                return [reqs[0][1]]
            acc = reqs[0][1].clone()
            for r in reqs[1:]:
                acc += r[1]
            for r in reqs:
                r[1].copy_(acc)
            return [r[1] for r in reqs]
        if kind == "a2a_start":
            # (sendbuf, send_counts|None, counts_dev, recvbuf, rw, recv_counts|None, rcounts_dev)
            sc = [list(r[2]) if r[2] is not None else [int(x) for x in r[3].tolist()] for r in reqs]
            outs = []
            for d in range(D):
                rw, recvbuf = reqs[d][5], reqs[d][4]
                roff = 0
                for p in range(D):
                    n = sc[p][d] if p != d else 0
                    if n:
                        off = sum(sc[p][:d])
                        recvbuf[roff * rw:(roff + n) * rw].copy_(reqs[p][1][off * rw:(off + n) * rw])
                    roff += n
                rc = [sc[p][d] if p != d else 0 for p in range(D)]
                if reqs[d][2] is None and reqs[d][7] is not None:  # dynamic counts -> device
                    reqs[d][7].copy_(torch.stack([reqs[p][3][d] for p in range(D)]))
                outs.append(dict(send_counts=sc[d], recv_counts=rc, stream=None))
            return outs
        if kind == "a2a_finish":
            return [r[1] for r in reqs]
        raise ValueError(kind)


class _Done:
    def __init__(self, value):
        self.value = value


class NcclRunner:
    """One shard per process; collectives through torch.distributed (NCCL).

    Boundary all-to-allvs run on a dedicated comm stream: "a2a_start" makes
    the comm stream wait for the packed send buffer only, so the compute
    stream keeps running (interior rows) while the transfer is in flight;
    "a2a_finish" hands the comm stream back to the shard, which unpacks on it
    and joins. Stale-filtered (device-counted) exchanges first swap their
    per-peer counts (one int per peer) and read them once on the host."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.timing = None
        self.comm = None
        # optional [(start, end, bytes out, bytes in)] of every payload
        # all-to-allv on the comm stream (bench.py: exchange GB/s vs NVLink)
        self.comm_timing = None

    def _stall(self, fn):
        if self.timing is None:
            return fn()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        self.timing[0].append((a, b))
        return out

    def run(self, gens):
        (g,) = gens
        dist = self.dist
        try:
            req = next(g)
            while True:
                kind = req[0]
                if kind == "max":
                    t = req[1].clone()
                    self._stall(lambda: dist.all_reduce(t, op=dist.ReduceOp.MAX, group=self.group))
                    out = t
                elif kind == "sum":
                    self._stall(lambda: dist.all_reduce(req[1], op=dist.ReduceOp.SUM,
                                                        group=self.group))
                    out = req[1]
                elif kind == "a2a_start":
                    out = self._start(*req[1:])
                elif kind == "a2a_finish":
                    out = self._finish(req[1])
                else:
                    raise ValueError(kind)
                req = g.send(out)
        except StopIteration as stop:
            return [stop.value]

    def _start(self, sendbuf, sc, counts_dev, recvbuf, rw, rc, rcounts_dev):
        dist = self.dist
        tok = dict(sendbuf=sendbuf, recvbuf=recvbuf, rw=rw, sc=sc, rc=rc, cuda=sendbuf.is_cuda)
        if tok["cuda"] and self.comm is None:
            self.comm = torch.cuda.Stream()
        ctx = _nullctx()
        if tok["cuda"]:
            ev = torch.cuda.Event()
            ev.record()
            ctx = torch.cuda.stream(self.comm)
        with ctx:
            if tok["cuda"]:
                self.comm.wait_event(ev)
            if sc is None:  # device-counted (stale-filtered): swap the counts first
                dist.all_to_all_single(rcounts_dev, counts_dev, group=self.group)
                pin = torch.empty(2, counts_dev.numel(), dtype=torch.int32,
                                  pin_memory=tok["cuda"])
                pin[0].copy_(counts_dev, non_blocking=True)
                pin[1].copy_(rcounts_dev, non_blocking=True)
                tok["pin"] = pin
                if tok["cuda"]:
                    tok["ev"] = torch.cuda.Event()
                    tok["ev"].record(self.comm)
            else:
                self._payload(tok)
        return tok

    def _payload(self, tok):
        rw, sc, rc = tok["rw"], tok["sc"], tok["rc"]
        timed = self.comm_timing is not None and tok["cuda"]
        with torch.cuda.stream(self.comm) if tok["cuda"] else _nullctx():
            if timed:
                a = torch.cuda.Event(enable_timing=True)
                a.record(self.comm)
            self.dist.all_to_all_single(tok["recvbuf"][:sum(rc) * rw], tok["sendbuf"][:sum(sc) * rw],
                                        [c * rw for c in rc], [c * rw for c in sc],
                                        group=self.group)
            if timed:
                b = torch.cuda.Event(enable_timing=True)
                b.record(self.comm)
                self.comm_timing.append((a, b, 4 * rw * sum(sc), 4 * rw * sum(rc)))
        tok["done"] = True

    def _finish(self, tok):
        if not tok.get("done"):
            if tok["cuda"]:
                tok["ev"].synchronize()  # the only host wait: one per stale-filtered exchange
            tok["sc"] = [int(x) for x in tok["pin"][0].tolist()]
            tok["rc"] = [int(x) for x in tok["pin"][1].tolist()]
            self._payload(tok)
        return dict(send_counts=tok["sc"], recv_counts=tok["rc"],
                    stream=self.comm if tok["cuda"] else None)


# -- the trainer ----------------------------------------------------------------

class PendingEpoch:
    """An enqueued epoch (DGNNTrainer.submit_epoch); result() -> EpochReport."""

    def __init__(self, trainer, r, t0, t1, done_ev, slot, infos, timed):
        self.trainer, self.r, self.t0, self.t1 = trainer, r, t0, t1
        self.done_ev, self.slot, self.infos, self.timed = done_ev, slot, infos, timed
        self.done = False
        self._report = None

    def result(self):
        if not self.done:
            self._report = self.trainer._finish_epoch(self)
            self.done = True
        return self._report


class DGNNTrainer:
    """Chunk-partitioned DGNN training on B200 driven by the reference plan.

    ``distributed=True``: this process owns the shard of rank
    torch.distributed.get_rank() (one GPU per rank, NCCL). Otherwise all D
    shards of the plan live on ``device`` and exchange locally."""

    def __init__(self, pa: PlanArrays, cfg: DGNNConfig, stale_config=None, seed: int = 0,
                 device=None, distributed: bool = False, features=None, labels=None,
                 params=None, cuda_graph: bool = False):
        self.pa, self.cfg = pa, cfg
        # cuda_graph: a single-process epoch without staleness (any number of
        # local shards) is a fixed kernel sequence with no host sync; capture it
        # once (after one eager epoch) and replay it, so the step is not bound
        # by per-launch host latency
        self.cuda_graph = cuda_graph
        self._graphs = {}
        self._loss_host = None
        self._unread = []  # submitted graph epochs whose result() was not read yet
        self._epoch_ev = None
        self._alt_free_ev = None
        # double-buffered input staging (stage_inputs / run_epoch(next_inputs=...))
        self._copy_stream = None
        self._staged_ev = None
        self.stale = StaleConfig.coerce(stale_config)
        self.device = torch.device(device or "cuda")
        self.trace = EpochLossTrace()
        X, y = (features, labels) if features is not None else synthetic_inputs(
            pa.n_instances, cfg.F, cfg.C, seed)
        self.params0 = params if params is not None else init_params(cfg, seed)
        if distributed:
            import torch.distributed as dist
            ranks = [dist.get_rank()]
            if dist.get_world_size() != pa.n_devices:
                raise ValueError("world size must equal the plan's n_devices")
            self.runner = NcclRunner()
        else:
            ranks = list(range(pa.n_devices))
            self.runner = LocalRunner()
        seg_rows = 128 if cfg.model == "evolve" else 0
        if cfg.model == "evolve" and cfg.T == 0:
            cfg.T = int(pa.inst_t.max())
        self.layouts = [build_layout(pa, d, segment_rows=seg_rows) for d in ranks]
        self.shards = [Shard(pa, lay, cfg, self.params0, X, y, self.stale, pa.n_instances,
                             self.device) for lay in self.layouts]
        prof = pa.profile or {}
        self.s_bytes = int(prof.get("bytes_per_scalar", 4))
        self.blocks = int(prof.get("blocks", 1))
        self.method = str(pa.meta.get("method", "pgc"))
        self.epoch_no = 0

    def host_inputs(self, features: np.ndarray, labels: np.ndarray):
        """Per-shard pinned host tensors (own-row order; padding rows zero /
        label -1) of global per-instance features and labels, for
        stage_inputs / run_epoch(next_inputs=...)."""
        xs, ys = [], []
        for sh in self.shards:
            real = sh.lay.own_gid >= 0
            gid = np.maximum(sh.lay.own_gid, 0)
            x = np.where(real[:, None], features[gid], 0).astype(np.float32)
            if sh.x_f16:
                # TF32 mode, in-range features: consumed at fp16 precision, so they
                # ship as fp16 (half the PCIe bytes; numpy's round-to-nearest-even
                # equals the device-side dgc_round_f16 of the fp32 values)
                x = x.astype(np.float16)
            elif sh.tf32 and x.size % 4 == 0:
                # TF32 mode: the features are consumed TF32-rounded, so they ship as
                # the 3 significant bytes of the rounded value (25% fewer PCIe bytes;
                # bit-identical to the device-side rounding of the fp32 values)
                x = ops.pack_tf32x24(x)
            xs.append(torch.as_tensor(x).pin_memory())
            ys.append(torch.as_tensor(np.where(real, labels[gid], -1).astype(np.int32)).pin_memory())
        return xs, ys

    def stage_inputs(self, xs, ys):
        """Start the host->device copy of the NEXT epoch's features / labels
        (per-shard pinned host tensors, see host_inputs) on a side stream and
        expand them there (TF32 unpack / rounding) into each shard's second
        input buffer; the next run_epoch() switches to that buffer (and to the
        CUDA graph captured for it) after a stream wait. Copy and expansion
        overlap whatever the compute stream is running: a prefetching input
        pipeline, two input buffers per shard."""
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
            # one pinned H2D copy stream moved 26-35 GB/s on the B200 boxes, four
            # concurrent ones 45 GB/s (tools/h2d_bw.py): big inputs go in 4 slices
            self._copy_lanes = [torch.cuda.Stream(self.device) for _ in range(4)]
            for sh, x in zip(self.shards, xs):
                sh.X_stage = (None if sh.X.dtype == torch.float16 else
                              torch.empty(x.shape, dtype=x.dtype, device=self.device))
                sh.X_alt = torch.empty_like(sh.X)
                sh.y_alt = torch.empty_like(sh.y)
        def h2d(dst, src):  # dst <- src (pinned host), in row slices on the copy lanes
            rows = src.shape[0]
            k = len(self._copy_lanes) if src.numel() * src.element_size() >= (8 << 20) else 1
            step = (rows + k - 1) // k
            for i in range(k):
                lane = self._copy_lanes[i]
                lane.wait_stream(self._copy_stream)
                with torch.cuda.stream(lane):
                    dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
            for i in range(k):
                self._copy_stream.wait_stream(self._copy_lanes[i])

        with torch.cuda.stream(self._copy_stream):
            # the second buffers were last read by the epoch before the running one
            if self._alt_free_ev is not None:
                self._copy_stream.wait_event(self._alt_free_ev)
            for sh, x, y in zip(self.shards, xs, ys):
                if sh.X.dtype == torch.float16:  # resident fp16 features: straight in
                    h2d(sh.X_alt, x)
                    sh.y_alt.copy_(y, non_blocking=True)
                    continue
                h2d(sh.X_stage, x)
                if sh.X_stage.dtype == torch.float16:  # fp16 features
                    ops.unpack_f16(sh.X_stage, sh.X_alt)
                elif sh.X_stage.dtype == torch.uint8:  # TF32 values shipped in 3 bytes
                    ops.unpack_tf32x24(sh.X_stage, sh.X_alt)
                elif sh.tf32:  # tensor-core operands are kept TF32-rounded
                    ops.round_tf32(sh.X_stage, sh.X_alt)
                else:
                    sh.X_alt.copy_(sh.X_stage)
                sh.y_alt.copy_(y, non_blocking=True)
            self._staged_ev = torch.cuda.Event()
            self._staged_ev.record(self._copy_stream)

    def _install_staged(self):
        torch.cuda.current_stream(self.device).wait_event(self._staged_ev)
        for sh in self.shards:
            sh.X, sh.X_alt = sh.X_alt, sh.X
            sh.y, sh.y_alt = sh.y_alt, sh.y
        self._staged_ev = None

    def run_epoch(self, next_inputs=None):
        """One training epoch (simulate_epoch's role, sim.py:423-566) -> EpochReport.
        If inputs were staged (stage_inputs) they are installed first;
        next_inputs = (xs, ys) stages the following epoch's inputs so their
        copy overlaps this epoch."""
        pend = self.submit_epoch(next_inputs)
        torch.cuda.synchronize(self.device)  # every stream: the staged inputs too
        return pend.result()

    def submit_epoch(self, next_inputs=None):
        """Enqueue one epoch without waiting for it -> PendingEpoch, whose
        result() waits for that epoch alone and returns its EpochReport. A
        training loop that submits epoch i+1 before reading epoch i's result
        keeps the device busy while the host reads the loss (at most one epoch
        in flight ahead: the double-buffered inputs and the loss slots are
        ordered by stream events). Epochs with host-side count exchanges (the
        multi-process runner, staleness) complete inside submit_epoch."""
        # at most two unread epochs: epoch i+2 reuses epoch i's pinned loss slot
        self._unread = [p for p in self._unread if not p.done]
        while len(self._unread) >= 2:
            self._unread.pop(0).result()
        r = self.epoch_no + 1
        # (no host synchronisation here: the previous epoch ended with one, and
        # staged inputs are ordered by stream events, so the install and the
        # epoch are enqueued while the device may still be draining earlier work)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        if self._staged_ev is not None:
            self._install_staged()
        # one process, no staleness: the step (all D local shards and their
        # exchanges) has no host synchronisation -> capturable
        graphable = (self.cuda_graph and self.stale.mode is StaleMode.OFF
                     and isinstance(self.runner, LocalRunner))
        # one captured graph per input buffer set (the staged inputs alternate)
        key = tuple(sh.X.data_ptr() for sh in self.shards)
        if graphable and r >= 2 and key not in self._graphs:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                infos_g = self.runner.run([s.step(r, self.trace) for s in self.shards])
            self._graphs[key] = (g, infos_g)
            torch.cuda.synchronize(self.device)
        replay = graphable and key in self._graphs
        # per-device times (EpochReport.per_device_*): eager epochs bracket every
        # shard's work / stalls with events; a replayed graph reuses the last
        # eager measurement (single device: the epoch itself)
        timed = not replay and len(self.shards) + (self.pa.n_devices > 1) > 1
        if timed:
            self.runner.timing = [[] for _ in self.shards]
            for sh in self.shards:
                sh.timing = []
        t0.record()
        if replay:
            g, infos = self._graphs[key]
            g.replay()
        else:
            infos = self.runner.run([s.step(r, self.trace) for s in self.shards])
        t1.record()
        self.runner.timing = None if not timed else self.runner.timing
        if self._loss_host is None:  # two pinned slots: one epoch may be in flight ahead
            self._loss_host = [torch.empty(1, dtype=infos[0]["loss_sum"].dtype, pin_memory=True)
                               for _ in range(2)]
        slot = self._loss_host[r & 1]
        slot.copy_(infos[0]["loss_sum"].reshape(1), non_blocking=True)
        # this epoch's input buffers become the next staging target only after
        # the epoch that follows it; the previous epoch's are free once it is done
        self._alt_free_ev, self._epoch_ev = self._epoch_ev, torch.cuda.Event()
        self._epoch_ev.record()
        done_ev = self._epoch_ev
        if next_inputs is not None:
            self.stage_inputs(*next_inputs)
        self.epoch_no = r
        pend = PendingEpoch(self, r, t0, t1, done_ev, slot, infos, timed)
        if not replay:  # eager epochs: host-synchronous bookkeeping (stale trace, timings)
            torch.cuda.synchronize(self.device)
            pend.result()
        else:
            self._unread.append(pend)
        return pend

    def _finish_epoch(self, p):
        """PendingEpoch.result(): wait for epoch p, read its loss, build the report."""
        p.done_ev.synchronize()
        ms = p.t0.elapsed_time(p.t1)
        if p.timed:
            self._device_times(ms)
            self.runner.timing = None
            for sh in self.shards:
                sh.timing = None
        loss = float(p.slot[0]) / self.pa.n_instances
        self.trace.append(loss)
        return self._report(p.r, ms, p.infos, loss)

    def _device_times(self, ms):
        """Per-device compute and wall ms of the epoch just measured.
        NCCL (one shard per rank): wall = the rank's epoch, compute = wall minus
        the compute stream's stalls on collectives / exchange arrivals;
        all-gathered over ranks. Local shards: compute = the sum of the shard's
        own segments, wall = compute + the exchange service time."""
        if isinstance(self.runner, NcclRunner):
            sh = self.shards[0]
            stall = sum(a.elapsed_time(b) for a, b in (sh.timing or []) + self.runner.timing[0])
            import torch.distributed as dist
            mine = torch.tensor([max(ms - stall, 0.0), ms], dtype=torch.float64, device=self.device)
            out = [torch.zeros_like(mine) for _ in range(dist.get_world_size())]
            dist.all_gather(out, mine)
            vals = torch.stack(out).cpu().numpy()
            self._dev_times = ([float(v) for v in vals[:, 0]], [float(v) for v in vals[:, 1]])
            return
        comp = [sum(a.elapsed_time(b) for a, b in seg) for seg in self.runner.timing]
        service = max(ms - sum(comp), 0.0)
        self._dev_times = (comp, [c + service for c in comp])

    def _report_static(self):
        """Plan-constant report fields (computed once). Billing follows the
        reference's MessageSet bytes (costmodel.py:95-103): per message and GCN
        (RNN) layer, blocks * profile.embedding_dim * bytes_per_scalar."""
        if getattr(self, "_static_rep", None) is None:
            cfg = self.cfg
            prof = self.pa.profile or {}
            emb = int(prof.get("embedding_dim", cfg.H))
            per_msg = self.blocks * emb * self.s_bytes
            lays = self.layouts
            full = np.asarray([2 * sum(int(l.key_ncut.sum()) for l in lays),
                               cfg.n_rnn * sum(len(l.tkey_rows) for l in lays)], np.int64)
            self._static_rep = dict(
                per_msg=per_msg, full=full,
                loading=sum(l.loaded_rows for l in lays) * self.pa.feature_dim * self.s_bytes,
                padding=sum(l.padding for l in lays),
                naive_padding=sum(l.naive_padding for l in lays))
        return self._static_rep

    def _report(self, r, ms, infos, loss):
        cfg = self.cfg
        st = self._report_static()
        per_msg = st["per_msg"]
        stale_on = self.stale.mode is not StaleMode.OFF and self.pa.n_devices > 1
        full = st["full"].copy()
        if self.pa.n_devices > 1 and len(self.shards) == 1:  # NCCL: this rank's share
            full = np.asarray([2 * int(self.layouts[0].key_ncut.sum()),
                               cfg.n_rnn * len(self.layouts[0].tkey_rows)], np.int64)
        rows = [sum(i["rows"] for i in infos), sum(i["xbytes"] for i in infos)]
        nccl = self.pa.n_devices > 1 and len(self.shards) == 1
        if stale_on or nccl:  # device-side counters / a cross-rank sum
            if stale_on:
                billed = torch.stack([sh.billed_dev for sh in self.shards]).sum(0)
            else:
                billed = torch.as_tensor(full, device=self.device)
            acc = torch.cat([billed.to(torch.int64), torch.as_tensor(full, device=self.device),
                             torch.tensor(rows, dtype=torch.int64, device=self.device)])
            if nccl:
                import torch.distributed as dist
                dist.all_reduce(acc)
            acc = [int(x) for x in acc.tolist()]
        else:  # host values only: no stream work behind an epoch that may already be queued
            acc = [int(full[0]), int(full[1]), int(full[0]), int(full[1]), rows[0], rows[1]]
        billed_sp, billed_tm = acc[0] * per_msg, acc[1] * per_msg
        full_b = (acc[2] + acc[3]) * per_msg
        n_rows, xbytes = acc[4], acc[5]
        sent = billed_sp + billed_tm
        avoided = full_b - sent
        i0 = infos[0]
        d_r = {k: (float(v.reshape(-1)[0].item()) if v is not None else 0.0)
               for k, v in i0["d_r"].items()}
        theta = {k: i0["coef"][k] * d_r[k] for k in d_r}
        comp, walls = getattr(self, "_dev_times", ([ms], [ms]))
        if self.pa.n_devices == 1:
            comp, walls = [ms], [ms]
        lam = max(walls) / min(walls) if walls and min(walls) > 0 else 1.0
        return EpochReport(
            method=self.method, epoch=r, per_device_compute_ms=list(comp),
            per_device_wall_ms=list(walls),
            spatial_traffic_bytes=billed_sp, temporal_traffic_bytes=billed_tm, shuffle_bytes=0,
            loading_bytes=st["loading"] if r == 1 else 0,
            padding_slots=st["padding"], naive_padding_slots=st["naive_padding"],
            load_divergence=lam, wall_ms=ms, stale_theta=theta.get("s0", 0.0),
            stale_d=d_r.get("s0", 0.0),
            stale_sent_bytes=sent if stale_on else 0,
            stale_avoided_bytes=avoided if stale_on else 0,
            stale_reduction_pct=(100.0 * avoided / full_b if full_b and stale_on else 0.0),
            loss=loss, exchanged_rows=n_rows, exchanged_bytes=xbytes,
            stale_detail={"theta": theta, "d_r": d_r})

    def params(self, shard: int = 0) -> dict:
        sh = self.shards[shard]
        return {k: sh.p(k).detach().cpu().numpy().copy() for k in sh.offs}

    def grads(self, shard: int = 0) -> dict:
        sh = self.shards[shard]
        return {k: sh.g(k).detach().cpu().numpy().copy() for k in sh.offs}

    def optimizer_state(self, shard: int = 0):
        """(first moments, second moments, step count) per parameter name."""
        sh = self.shards[shard]

        def view(buf, k):
            o, shape = sh.offs[k]
            return buf[o:o + int(np.prod(shape))].view(*shape).detach().cpu().numpy().copy()
        return ({k: view(sh.m, k) for k in sh.offs}, {k: view(sh.v, k) for k in sh.offs},
                int(sh.step_dev.item()) if self.cfg.optimizer == "adam" else sh.step_count)

    def relu_masks(self, shard: int = 0):
        """{GCN layer: bool (n_own, H)} -- this epoch's ReLU decisions (H_l > 0;
        the fp16 activations the next layer consumed on the fp16 GCN path)."""
        sh = self.shards[shard]
        if sh.f16_gcn:
            return {0: (sh.H1_16 > 0).cpu().numpy(), 1: (sh.x16[0] > 0).cpu().numpy()}
        return {l: (sh.Hl[l] > 0).cpu().numpy() for l in range(2)}


def reference_billed_messages(layouts, spatial_sends, temporal_sends):
    """Host restatement of the reference's billing for given send masks:
    the cut messages whose source is sent (sim.py:464-469,
    ``msgs.nbytes[cut & send[src]]``), counted per GCN layer (spatial) and per
    RNN layer (temporal). ``spatial_sends[l][d]`` / ``temporal_sends[k][d]``:
    bool per key of device d (layouts' key_rows / tkey_rows). Returns
    (spatial messages, temporal messages); bytes = messages * blocks *
    embedding_dim * bytes_per_scalar (costmodel.py:95-103)."""
    sp = sum(int(np.asarray(lay.key_ncut)[np.asarray(m[d], bool)].sum())
             for m in spatial_sends for d, lay in enumerate(layouts))
    tm = sum(int(np.asarray(m[d], bool).sum()) for m in temporal_sends for d in range(len(layouts)))
    return sp, tm


class StaleState:
    """Cross-epoch state of the B200 step, the role of sim.StaleState
    (sim.py:306-324): the trainer (parameters, optimizer moments, embedding
    caches, halo rows, carries, the real epoch-loss trace). Built once from
    the reference graph + plan (or a PlanArrays) and threaded through
    simulate_epoch calls."""

    def __init__(self, g, plan=None, profile=None, cluster=None, stale_config=None, seed=0, *,
                 cfg: DGNNConfig | None = None, F: int | None = None, H: int | None = None,
                 distributed: bool = False, device=None, cuda_graph: bool = False):
        from .plan import from_dynpart
        pa = g if isinstance(g, PlanArrays) else from_dynpart(g, plan)
        prof = profile.to_dict() if hasattr(profile, "to_dict") else (profile or pa.profile)
        pa.profile = dict(prof or {})
        if cfg is None:
            cfg = DGNNConfig.for_profile(pa.profile, F=F or pa.feature_dim, H=H)
        self.pa, self.cfg = pa, cfg
        self.trainer = DGNNTrainer(pa, cfg, stale_config, seed=seed, device=device,
                                   distributed=distributed, cuda_graph=cuda_graph)

    @property
    def trace(self):
        return self.trainer.trace


def _check_plan(g, plan, cluster):
    """The reference's guards (sim.py:433-437), raised before any GPU work."""
    from .plan import PlanGraphMismatch
    n_inst = g.n_instances
    sdev = plan.structure_device if plan is not None else g.structure_device
    if len(sdev) != n_inst:
        raise PlanGraphMismatch(f"plan covers {len(sdev)} instances, graph has {n_inst}")
    n_dev = plan.n_devices if plan is not None else g.n_devices
    c_dev = getattr(cluster, "n_devices", cluster)
    if c_dev is not None and int(c_dev) != int(n_dev):
        raise PlanGraphMismatch("plan and cluster disagree on device count")


def simulate_epoch(g, plan, profile=None, cluster=None, stale_config=None, epoch: int = 1,
                   coeffs=None, stale_state: StaleState | None = None, **kw):
    """Drop-in for dynpart.sim.simulate_epoch (sim.py:423-432): same
    positional signature; one REAL training epoch (fwd + bwd + exchange +
    all-reduce + update) on the B200 step, reported in the reference's
    EpochReport fields (sim.py:259-303) with measured per-device times,
    lambda = max/min of the per-device walls (assign.py:98-104) and the
    reference-billed bytes of the actual send masks. ``g``/``plan``: a dynpart
    DynamicGraph + Plan (converted unchanged) or a PlanArrays (plan=None).
    Without ``stale_state`` a fresh state is built (epoch 1 from the initial
    parameters); threading one state through consecutive epochs trains.
    ``coeffs`` (the reference's analytic cost coefficients) is unused: times are
    measured."""
    _check_plan(g, plan, cluster)
    state = stale_state if stale_state is not None else StaleState(
        g, plan, profile, cluster, stale_config, **kw)
    tr = state.trainer
    if epoch != tr.epoch_no + 1:
        raise ValueError(f"epoch {epoch} requested, the state is at epoch {tr.epoch_no}")
    if stale_config is not None and StaleConfig.coerce(stale_config) != tr.stale:
        raise ValueError("stale_config differs from the one the state was built with")
    return tr.run_epoch()


def run_epochs(g, plan=None, profile=None, cluster=None, epochs: int = 1, stale_config=None,
               drift_spec=None, seed: int = 0, coeffs=None, initial_loss=None, loss_decay=None,
               *, cfg: DGNNConfig | None = None, F: int | None = None, H: int | None = None,
               distributed: bool = False, device=None, cuda_graph: bool = False):
    """Drop-in for dynpart.sim.run_epochs (sim.py:569-599): same positional
    signature, real training through simulate_epoch with one StaleState.
    drift_spec, coeffs, initial_loss and loss_decay drive the reference's
    simulated embeddings/loss and are unused: the embeddings and the loss
    trace are real."""
    if plan is not None or not isinstance(g, PlanArrays):
        _check_plan(g, plan, cluster)
    state = StaleState(g, plan, profile, cluster, stale_config, seed, cfg=cfg, F=F, H=H,
                       distributed=distributed, device=device, cuda_graph=cuda_graph)
    return [simulate_epoch(g, plan, profile, cluster, stale_config, r, coeffs, state)
            for r in range(1, epochs + 1)]
