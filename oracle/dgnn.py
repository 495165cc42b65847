"""fp64 oracle of the chunk-partitioned DGNN training step.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). All devices of a plan run
in one process; exchanges are direct array copies. The semantics are the ones
DESIGN.md §3 fixes, mirrored by the GPU trainer:

  per GCN layer l:  Y = H_{l-1} W_l (own rows) -> stale filter on boundary keys
                    (stale.py:154-176, global D_r via max over devices) ->
                    halo rows of Y refreshed for sent keys (persist otherwise) ->
                    H_l = relu(dinv_i * sum_j dinv_j Y_j + b_l)   (GCNConv norm)
  RNN layer k:      reference-form GRU (fusion.py:409-413) or LSTM over the
                    FFD-packed per-device runs (fusion.py:278-313, sim.py:401-420)
                    with the reference carry mask; a run whose predecessor
                    presence lives on another device starts from the carry that
                    device last transmitted (epoch 1: zero, = the reference);
                    the carries are exchanged after the forward through their
                    own stale cache (carry-from-cache, Appendix B.2(a)).
  readout:          logits = Hr Wo + bo; loss = mean CE over all instances.
  backward:         exact gradients; reused (stale) halo rows return no
                    gradient (Appendix B.4); carries are constants.
  update:           grads summed over devices; SGD(momentum) or Adam.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .reference_path import threshold

GATES = {"gru": 3, "lstm": 4}


def sig(x):
    return 1.0 / (1.0 + np.exp(-x))


@dataclass
class OracleConfig:
    F: int
    H: int
    C: int
    rnn: str = "gru"
    n_rnn: int = 1
    stale_mode: str = "off"
    static_fraction: float = 0.5
    optimizer: str = "sgd"
    model: str = "rnn"        # "rnn" (GCN + GRU/LSTM) or "evolve" (EvolveGCN-O)
    T: int = 0                # snapshots (evolve)
    lr: float = 0.05
    momentum: float = 0.9
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


def evolve_forward(W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, T):
    """EvolveGCN-O with the reference GRU form (fusion.py:409-413), input =
    hidden = W_{t-1}: returns [W_0..W_T] and the per-step saves."""
    Ws, saves = [W0], []
    w = W0
    for _ in range(T):
        r = sig(Sr @ w + Br)
        z = sig(Sz @ w + Bz)
        c = np.tanh(Pc @ w + Qc @ (r * w) + Bc)
        saves.append((w, r, z, c))
        w = (1.0 - z) * c + z * w
        Ws.append(w)
    return Ws, saves


def evolve_backward(Sr, Sz, Pc, Qc, saves, dW_direct):
    """BPTT of evolve_forward; dW_direct[t-1] = d loss / d W_t (t = 1..T)."""
    g_Sr, g_Sz, g_Pc, g_Qc = (np.zeros_like(Sr) for _ in range(4))
    g_Br = np.zeros_like(saves[0][0]) if saves else 0.0
    g_Bz, g_Bc = np.zeros_like(g_Br), np.zeros_like(g_Br)
    carry = np.zeros_like(g_Br)
    for t in reversed(range(len(saves))):
        w, r, z, c = saves[t]
        g = carry + dW_direct[t]
        dz = g * (w - c)
        dc = g * (1.0 - z)
        dw = g * z
        dac = dc * (1.0 - c * c)
        g_Pc += dac @ w.T
        g_Qc += dac @ (r * w).T
        g_Bc += dac
        drw = Qc.T @ dac
        dw += drw * r + Pc.T @ dac
        dar = drw * w * r * (1.0 - r)
        daz = dz * z * (1.0 - z)
        g_Sr += dar @ w.T
        g_Sz += daz @ w.T
        g_Br += dar
        g_Bz += daz
        dw += Sr.T @ dar + Sz.T @ daz
        carry = dw
    return carry, g_Sr, g_Sz, g_Pc, g_Qc, g_Br, g_Bz, g_Bc


EVOLVE_KEYS = ("Sr", "Sz", "Pc", "Qc", "Br", "Bz", "Bc")


def param_names(cfg: OracleConfig):
    if cfg.model == "evolve":
        names = []
        for l in (1, 2):
            names += [f"W{l}_0"] + [f"{k}{l}" for k in EVOLVE_KEYS] + [f"b{l}"]
        return names + ["Wo", "bo"]
    names = ["W1", "b1", "W2", "b2"]
    for k in range(cfg.n_rnn):
        names += [f"Wx{k}", f"U{k}", f"br{k}"]
    return names + ["Wo", "bo"]


class OracleDGNN:
    def __init__(self, layouts, X, y, params: dict, cfg: OracleConfig, inst_t=None):
        self.L = layouts
        self.t_own = None
        if cfg.model == "evolve":
            # snapshot (0-based) of every own row; -1 on padding rows
            self.t_own = [np.where(lay.own_gid >= 0, np.asarray(inst_t)[np.maximum(lay.own_gid, 0)] - 1, -1)
                          for lay in layouts]
        self.D = len(layouts)
        self.cfg = cfg
        self.G = GATES[cfg.rnn]
        self.X = [np.where((lay.own_gid >= 0)[:, None],
                           np.asarray(X, np.float64)[np.maximum(lay.own_gid, 0)], 0.0)
                  for lay in layouts]
        self.y = [np.where(lay.own_gid >= 0, np.asarray(y)[np.maximum(lay.own_gid, 0)], -1)
                  for lay in layouts]
        self.n_total = sum(int((lay.own_gid >= 0).sum()) for lay in layouts)
        self.p = {k: np.array(v, dtype=np.float64) for k, v in params.items()}
        self.A = []
        for lay in layouts:
            nnz_row = np.repeat(np.arange(lay.n_own), np.diff(lay.row_ptr))
            val = lay.dinv[nnz_row] * lay.dinv[lay.col]
            self.A.append(sp.csr_matrix((val, (nnz_row, lay.col)),
                                        shape=(lay.n_own, lay.n_own + lay.n_halo)))
        H = cfg.H
        cw = H * (2 if cfg.rnn == "lstm" else 1)
        # persistent cross-epoch state
        self.halo = [[np.zeros((lay.n_halo, H)) for lay in layouts] for _ in range(2)]
        self.scache = [[np.zeros((len(lay.key_rows), H)) for lay in layouts] for _ in range(2)]
        self.scached = [[np.zeros(len(lay.key_rows), bool) for lay in layouts] for _ in range(2)]
        self.carry = [[np.zeros((lay.n_carry, cw)) for lay in layouts] for _ in range(cfg.n_rnn)]
        self.tcache = [[np.zeros((len(lay.tkey_rows), cw)) for lay in layouts] for _ in range(cfg.n_rnn)]
        self.tcached = [[np.zeros(len(lay.tkey_rows), bool) for lay in layouts] for _ in range(cfg.n_rnn)]
        self.losses: list[float] = []
        self.mom = {k: np.zeros_like(v) for k, v in self.p.items()}
        self.vel = {k: np.zeros_like(v) for k, v in self.p.items()}
        self.step_count = 0
        self.tie_log: list[dict] = []
        self.relu_log: list[dict] = []

    # -- staleness (stale.py) ------------------------------------------------
    def _decide(self, r, values, cache, cached, forced=None, tag=""):
        """One global decision per cache: D_r = max over devices (sim.py:455-459).

        ``forced`` (per-device bool arrays) replays another implementation's
        decisions; the oracle's own decision is still computed and every key
        where they differ is recorded in self.tie_log with its distance and
        theta, so tests can assert the disagreement lies in the fp32 tie band
        (SURVEY.md §7 (ii))."""
        if self.D == 1:
            return [np.zeros(0, bool) for _ in values], 0.0, 0.0
        mode = self.cfg.stale_mode
        if mode == "off":
            return [np.ones(len(v), bool) for v in values], 0.0, 0.0
        dists = []
        for v, c in zip(values, cache):
            df = v - c
            dists.append(np.sqrt((df * df).sum(axis=1)))
        d_r = 0.0
        theta = 0.0
        if r >= 2:
            d_r = max([float(dd[cc].max()) for dd, cc in zip(dists, cached) if cc.any()] or [0.0])
            theta = threshold(self.losses, r, d_r, mode, self.cfg.static_fraction)
        sends = []
        for d, (v, c, cc, dd) in enumerate(zip(values, cache, cached, dists)):
            s = (~cc) | (dd > theta)
            if forced is not None:
                f = np.asarray(forced[d], bool)
                for k in np.flatnonzero(f != s):
                    self.tie_log.append(dict(epoch=r, cache=tag, device=d, key=int(k),
                                             dist=float(dd[k]), theta=float(theta),
                                             scale=float(np.abs(v[k]).max()),
                                             norm=float(np.sqrt((v[k] * v[k]).sum()))))
                s = f
            c[s] = v[s]
            cc |= s
            sends.append(s)
        return sends, theta, d_r

    # -- forward/backward of one epoch ---------------------------------------
    def epoch(self, r, forced=None, forced_relu=None):
        """One epoch; ``forced`` = {cache tag: per-device send masks} replays
        externally made stale decisions (see _decide). ``forced_relu`` =
        {GCN layer 0/1: per-device bool (n_own, H) masks} replays another
        implementation's ReLU decisions the same way: the oracle's own
        pre-activation z is still computed, and every element where
        (z > 0) differs from the forced mask is logged in self.relu_log with
        z and the layer's max|z| (tests assert they are near-ties, i.e. the
        discontinuity of relu' at 0 sits inside the other side's rounding)."""
        forced = forced or {}
        forced_relu = forced_relu or {}
        cfg, D, G, H = self.cfg, self.D, self.G, self.cfg.H
        out = {"send": {}, "theta": {}, "d_r": {}}
        hin = self.X
        acts = []
        fresh_all = []
        evo = []
        if cfg.model == "evolve":
            for l in (1, 2):
                Ws, sv = evolve_forward(self.p[f"W{l}_0"], *[self.p[f"{k}{l}"] for k in EVOLVE_KEYS],
                                        cfg.T)
                evo.append((Ws, sv))
        for l, (W, b) in enumerate([("W1", "b1"), ("W2", "b2")]):
            if cfg.model == "evolve":
                Ws = evo[l][0]
                Y = []
                for d in range(D):
                    yd = np.zeros((len(hin[d]), H))
                    for t in range(cfg.T):
                        rows = self.t_own[d] == t
                        if rows.any():
                            yd[rows] = hin[d][rows] @ Ws[t + 1]
                    Y.append(yd)
            else:
                Y = [h @ self.p[W] for h in hin]
            vals = [Y[d][self.L[d].key_rows] for d in range(D)]
            sends, theta, d_r = self._decide(r, vals, self.scache[l], self.scached[l],
                                             forced.get(f"s{l}"), f"s{l}")
            fresh = [np.zeros(self.L[d].n_halo, bool) for d in range(D)]
            for d in range(D):
                lay = self.L[d]
                for p in range(D):
                    if p == d:
                        continue
                    pos = lay.send_pos[lay.send_ptr[p]:lay.send_ptr[p + 1]]
                    dst = self.L[p]
                    slots = dst.recv_slot[dst.recv_ptr[d]:dst.recv_ptr[d + 1]] - dst.n_own
                    m = sends[d][pos] if D > 1 else np.ones(len(pos), bool)
                    self.halo[l][p][slots[m]] = vals[d][pos[m]]
                    fresh[p][slots[m]] = True
            out["send"][f"s{l}"] = sends
            out["theta"][f"s{l}"] = theta
            out["d_r"][f"s{l}"] = d_r
            Hl, masks = [], []
            for d in range(D):
                Yext = np.concatenate([Y[d], self.halo[l][d]])
                z = self.A[d] @ Yext + self.p[b]
                m = z > 0
                if l in forced_relu:
                    f = np.asarray(forced_relu[l][d], bool)
                    diff = np.flatnonzero((f != m).reshape(-1))
                    if len(diff):
                        zs = float(np.abs(z).max())
                        for i in diff:
                            self.relu_log.append(dict(epoch=r, layer=l, device=d, index=int(i),
                                                      z=float(z.reshape(-1)[i]), scale=zs))
                    m = f
                Hl.append(np.where(m, z, 0.0))
                masks.append(m)
            acts.append((hin, Hl, masks))
            fresh_all.append(fresh)
            hin = Hl
        # time encoder
        rnn_saves = []
        xr = hin
        for k in range(cfg.n_rnn if cfg.model == "rnn" else 0):
            outs, saves = [], []
            for d in range(D):
                o, s = self._rnn_fwd(d, k, xr[d])
                outs.append(o)
                saves.append(s)
            rnn_saves.append((xr, saves))
            # carry exchange for the next epoch (Appendix B.2(a))
            tvals = []
            for d in range(D):
                lay = self.L[d]
                h_out, c_out = saves[d]["h_inst"], saves[d].get("c_inst")
                v = h_out[lay.tkey_rows]
                if cfg.rnn == "lstm":
                    v = np.concatenate([v, c_out[lay.tkey_rows]], axis=1)
                tvals.append(v)
            tsends, ttheta, td_r = self._decide(r, tvals, self.tcache[k], self.tcached[k],
                                                forced.get(f"t{k}"), f"t{k}")
            for d in range(D):
                lay = self.L[d]
                for p in range(D):
                    if p == d:
                        continue
                    pos = lay.tsend_pos[lay.tsend_ptr[p]:lay.tsend_ptr[p + 1]]
                    dst = self.L[p]
                    cs = dst.trecv_carry[dst.trecv_ptr[d]:dst.trecv_ptr[d + 1]]
                    m = tsends[d][pos]
                    self.carry[k][p][cs[m]] = tvals[d][pos[m]]
            out["send"][f"t{k}"] = tsends
            out["theta"][f"t{k}"] = ttheta
            out["d_r"][f"t{k}"] = td_r
            xr = outs
        # readout + CE
        loss_sum = 0.0
        dlogits, hr = [], xr
        for d in range(D):
            logits = hr[d] @ self.p["Wo"] + self.p["bo"]
            m = logits.max(axis=1, keepdims=True)
            e = np.exp(logits - m)
            s = e.sum(axis=1, keepdims=True)
            logp = logits - m - np.log(s)
            yi = self.y[d]
            real = yi >= 0
            loss_sum += -logp[np.arange(len(yi))[real], yi[real]].sum()
            g = e / s
            g[np.arange(len(yi))[real], yi[real]] -= 1.0
            g[~real] = 0.0
            dlogits.append(g / self.n_total)
        loss = loss_sum / self.n_total
        out["loss"] = loss
        out["hr"] = hr
        out["h_gcn"] = [a[1] for a in acts]
        # backward
        grads = {k: np.zeros_like(v) for k, v in self.p.items()}
        dh = []
        for d in range(D):
            grads["Wo"] += hr[d].T @ dlogits[d]
            grads["bo"] += dlogits[d].sum(axis=0)
            dh.append(dlogits[d] @ self.p["Wo"].T)
        for k in reversed(range(cfg.n_rnn if cfg.model == "rnn" else 0)):
            xr_k, saves = rnn_saves[k]
            dx = []
            for d in range(D):
                dxd, gW, gU, gb = self._rnn_bwd(d, k, xr_k[d], saves[d], dh[d])
                grads[f"Wx{k}"] += gW
                grads[f"U{k}"] += gU
                grads[f"br{k}"] += gb
                dx.append(dxd)
            dh = dx
        for l in (1, 0):
            W, b = ("W1", "b1") if l == 0 else ("W2", "b2")
            hin_l, hout_l, mask_l = acts[l]
            dY_own = []
            dY_halo = []
            for d in range(D):
                dz = dh[d] * mask_l[d]
                grads[b] += dz.sum(axis=0)
                dYext = self.A[d].T @ dz
                dY_own.append(dYext[:self.L[d].n_own].copy())
                dY_halo.append(dYext[self.L[d].n_own:])
            for d in range(D):  # reverse exchange of fresh halo rows (Appendix B.4)
                lay = self.L[d]
                for p in range(D):
                    if p == d:
                        continue
                    src = self.L[p]
                    slots = src.recv_slot[src.recv_ptr[d]:src.recv_ptr[d + 1]] - src.n_own
                    pos = lay.send_pos[lay.send_ptr[p]:lay.send_ptr[p + 1]]
                    m = fresh_all[l][p][slots]
                    rows = lay.key_rows[pos[m]]
                    np.add.at(dY_own[d], rows, dY_halo[p][slots[m]])
            dh = []
            if cfg.model == "evolve":
                Ws, sv = evo[l]
                dW_direct = [np.zeros_like(Ws[0]) for _ in range(cfg.T)]
                for d in range(D):
                    dhd = np.zeros_like(hin_l[d])
                    for t in range(cfg.T):
                        rows = self.t_own[d] == t
                        if rows.any():
                            dW_direct[t] += hin_l[d][rows].T @ dY_own[d][rows]
                            dhd[rows] = dY_own[d][rows] @ Ws[t + 1].T
                    dh.append(dhd)
                ln = l + 1
                out_g = evolve_backward(*[self.p[f"{k}{ln}"] for k in ("Sr", "Sz", "Pc", "Qc")],
                                        sv, dW_direct)
                grads[f"W{ln}_0"] += out_g[0]
                for k, gk in zip(EVOLVE_KEYS, out_g[1:]):
                    grads[f"{k}{ln}"] += gk
                continue
            for d in range(D):
                grads[W] += hin_l[d].T @ dY_own[d]
                dh.append(dY_own[d] @ self.p[W].T)
        out["grads"] = grads
        self._update(grads)
        self.losses.append(loss)
        return out

    # -- recurrent encoders ----------------------------------------------------
    def _rnn_fwd(self, d, k, x):
        cfg, lay, H = self.cfg, self.L[d], self.cfg.H
        Wx, U, b = self.p[f"Wx{k}"], self.p[f"U{k}"], self.p[f"br{k}"]
        gx = x @ Wx + b
        R, Lr = lay.n_rows, lay.row_len
        srow = lay.slot_row.reshape(R, Lr)
        smask = lay.slot_mask.reshape(R, Lr)
        scarry = lay.slot_carry.reshape(R, Lr)
        h = np.zeros((R, H))
        c = np.zeros((R, H))
        h_inst = np.zeros((lay.n_own, H))
        c_inst = np.zeros((lay.n_own, H))
        steps = []
        for p in range(Lr):
            valid = srow[:, p] >= 0
            m = smask[:, p:p + 1].astype(np.float64)
            h = h * m
            c = c * m
            cr = scarry[:, p]
            has = cr >= 0
            if has.any():
                cv = self.carry[k][d][cr[has]]
                h[has] = cv[:, :H]
                if cfg.rnn == "lstm":
                    c[has] = cv[:, H:]
            g = np.where(valid[:, None], gx[np.maximum(srow[:, p], 0)], 0.0)
            if cfg.rnn == "gru":
                a_rz = g[:, :2 * H] + h @ U[:, :2 * H]
                rg, zg = sig(a_rz[:, :H]), sig(a_rz[:, H:])
                rh = rg * h
                cg = np.tanh(g[:, 2 * H:] + rh @ U[:, 2 * H:])
                hn = (1.0 - zg) * cg + zg * h
                steps.append(dict(h_in=h, r=rg, z=zg, c=cg, rh=rh))
                h = hn
            else:
                a = g + h @ U
                ig, fg = sig(a[:, :H]), sig(a[:, H:2 * H])
                gg, og = np.tanh(a[:, 2 * H:3 * H]), sig(a[:, 3 * H:])
                cn = fg * c + ig * gg
                tc = np.tanh(cn)
                hn = og * tc
                steps.append(dict(h_in=h, c_in=c, i=ig, f=fg, g=gg, o=og, tc=tc))
                h, c = hn, cn
            h_inst[srow[valid, p]] = h[valid]
            if cfg.rnn == "lstm":
                c_inst[srow[valid, p]] = c[valid]
        return h_inst, dict(steps=steps, h_inst=h_inst, c_inst=c_inst)

    def _rnn_bwd(self, d, k, x, save, dh_inst):
        cfg, lay, H = self.cfg, self.L[d], self.cfg.H
        Wx, U = self.p[f"Wx{k}"], self.p[f"U{k}"]
        R, Lr = lay.n_rows, lay.row_len
        srow = lay.slot_row.reshape(R, Lr)
        smask = lay.slot_mask.reshape(R, Lr)
        dgx = np.zeros((lay.n_own, self.G * H))
        gU = np.zeros_like(U)
        dh = np.zeros((R, H))
        dc = np.zeros((R, H))
        for p in reversed(range(Lr)):
            st = save["steps"][p]
            valid = srow[:, p] >= 0
            dh = dh + np.where(valid[:, None], dh_inst[np.maximum(srow[:, p], 0)], 0.0)
            if cfg.rnn == "gru":
                h, rg, zg, cg, rh = st["h_in"], st["r"], st["z"], st["c"], st["rh"]
                dz = dh * (h - cg)
                dcg = dh * (1.0 - zg)
                dhp = dh * zg
                dac = dcg * (1.0 - cg * cg)
                drh = dac @ U[:, 2 * H:].T
                dr = drh * h
                dhp += drh * rg
                dar = dr * rg * (1.0 - rg)
                daz = dz * zg * (1.0 - zg)
                da = np.concatenate([dar, daz, dac], axis=1)
                dhp += da[:, :2 * H] @ U[:, :2 * H].T
                gU[:, :2 * H] += h.T @ da[:, :2 * H]
                gU[:, 2 * H:] += rh.T @ dac
                dcp = None
            else:
                h, c_in = st["h_in"], st["c_in"]
                ig, fg, gg, og, tc = st["i"], st["f"], st["g"], st["o"], st["tc"]
                do = dh * tc
                dcn = dc + dh * og * (1.0 - tc * tc)
                di, dgg, df = dcn * gg, dcn * ig, dcn * c_in
                dcp = dcn * fg
                da = np.concatenate([di * ig * (1 - ig), df * fg * (1 - fg),
                                     dgg * (1 - gg * gg), do * og * (1 - og)], axis=1)
                dhp = da @ U.T
                gU += h.T @ da
            dgx[srow[valid, p]] = da[valid]
            m = smask[:, p:p + 1].astype(np.float64)
            dh = dhp * m  # remote carries are constants: no gradient
            if dcp is not None:
                dc = dcp * m
        gW = x.T @ dgx
        gb = dgx.sum(axis=0)
        dx = dgx @ Wx.T
        return dx, gW, gU, gb

    # -- optimizer -------------------------------------------------------------
    def _update(self, grads):
        cfg = self.cfg
        self.step_count += 1
        t = self.step_count
        for k in self.p:
            g = grads[k]
            if cfg.optimizer == "sgd":
                self.mom[k] = cfg.momentum * self.mom[k] + g
                self.p[k] = self.p[k] - cfg.lr * self.mom[k]
            else:
                self.mom[k] = cfg.beta1 * self.mom[k] + (1 - cfg.beta1) * g
                self.vel[k] = cfg.beta2 * self.vel[k] + (1 - cfg.beta2) * g * g
                mh = self.mom[k] / (1 - cfg.beta1 ** t)
                vh = self.vel[k] / (1 - cfg.beta2 ** t)
                self.p[k] = self.p[k] - cfg.lr * mh / (np.sqrt(vh) + cfg.eps)
