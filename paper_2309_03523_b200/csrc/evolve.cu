// EvolveGCN-O weight evolution (BASELINE config C3).
//
// The reference has no EvolveGCN arithmetic; DESIGN.md §3
// fixes it as EvolveGCN-O with the reference's GRU form (GruCell.step,
// fusion.py:409-413) applied to the GCN weight matrix itself, input = hidden =
// W_{t-1} (per layer, W in R^{F_l x H_l}, gate matrices acting on the F_l rows):
//   R = s(S_r W + B_r), Z = s(S_z W + B_z), C = tanh(P_c W + Q_c (R*W) + B_c),
//   W_t = (1 - Z) * C + Z * W_{t-1},   t = 1..T,  snapshot t uses W_t.
// (S_g = W_g + U_g of the GRU since the input equals the hidden state.)
// Columns of W are independent recurrences: CTA = CB columns x F_l rows,
// persistent over the T snapshots. Saves are laid out [F_l][T][H_l] so the
// gate-matrix gradients are single K = T*H_l tcgen05 GEMMs afterwards.
#include "tc_common.cuh"

#include <cstdio>
#include <cstdlib>
#include <string>

namespace {

__device__ __forceinline__ float sgm(float x) { return 1.f / (1.f + __expf(-x)); }

// Thread (row i, group jj) carries NJ columns: every gate-matrix element it
// loads feeds NJ FMAs (the matrices are shared by all columns), and the
// per-column state lives in registers.
template <int NJ>
__global__ void __launch_bounds__(512) evolve_fwd_kernel(
    int Fl, int Hl, int T, const float* __restrict__ W0, const float* __restrict__ SrT,
    const float* __restrict__ SzT, const float* __restrict__ PcT, const float* __restrict__ QcT,
    const float* __restrict__ Br, const float* __restrict__ Bz, const float* __restrict__ Bc,
    float* __restrict__ Wstack, float* __restrict__ sv_r, float* __restrict__ sv_z,
    float* __restrict__ sv_c, float* __restrict__ sv_w, float* __restrict__ sv_rw, int rnd) {
  extern __shared__ float sm[];
  const int CB = blockDim.y;
  float* w_s = sm;                   // [CB*NJ][Fl]
  float* rw_s = sm + CB * NJ * Fl;   // [CB*NJ][Fl]
  const int i = threadIdx.x, jj = threadIdx.y;
  const int jb = (blockIdx.x * CB + jj) * NJ;
  float w[NJ], br[NJ], bz[NJ], bc[NJ];
#pragma unroll
  for (int n = 0; n < NJ; ++n) {
    const int j = jb + n;
    const bool ok = j < Hl;
    w[n] = ok ? W0[(int64_t)i * Hl + j] : 0.f;
    w_s[(jj * NJ + n) * Fl + i] = w[n];
    if (ok) Wstack[(int64_t)i * Hl + j] = rnd ? dgc::rna_tf32_f(w[n]) : w[n];
    br[n] = ok ? Br[(int64_t)i * Hl + j] : 0.f;
    bz[n] = ok ? Bz[(int64_t)i * Hl + j] : 0.f;
    bc[n] = ok ? Bc[(int64_t)i * Hl + j] : 0.f;
  }
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    float ar[NJ], az[NJ], ap[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) { ar[n] = br[n]; az[n] = bz[n]; ap[n] = bc[n]; }
    for (int k = 0; k < Fl; ++k) {
      const float sr = __ldg(SrT + (int64_t)k * Fl + i), sz = __ldg(SzT + (int64_t)k * Fl + i),
                  pc = __ldg(PcT + (int64_t)k * Fl + i);
#pragma unroll
      for (int n = 0; n < NJ; ++n) {
        const float wk = w_s[(jj * NJ + n) * Fl + k];
        ar[n] = fmaf(sr, wk, ar[n]);
        az[n] = fmaf(sz, wk, az[n]);
        ap[n] = fmaf(pc, wk, ap[n]);
      }
    }
    float r[NJ], z[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      r[n] = sgm(ar[n]);
      z[n] = sgm(az[n]);
      rw_s[(jj * NJ + n) * Fl + i] = r[n] * w[n];
    }
    __syncthreads();
    float aq[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) aq[n] = ap[n];
    for (int k = 0; k < Fl; ++k) {
      const float qc = __ldg(QcT + (int64_t)k * Fl + i);
#pragma unroll
      for (int n = 0; n < NJ; ++n) aq[n] = fmaf(qc, rw_s[(jj * NJ + n) * Fl + k], aq[n]);
    }
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const int j = jb + n;
      const float c = tanhf(aq[n]);
      const float wn = (1.f - z[n]) * c + z[n] * w[n];
      if (j < Hl) {
        const int64_t sidx = ((int64_t)i * T + t) * Hl + j;  // [Fl][T][Hl]
        sv_r[sidx] = r[n];
        sv_z[sidx] = z[n];
        sv_c[sidx] = c;
        sv_w[sidx] = rnd ? dgc::rna_tf32_f(w[n]) : w[n];
        sv_rw[sidx] = rnd ? dgc::rna_tf32_f(r[n] * w[n]) : r[n] * w[n];
        Wstack[((int64_t)(t + 1) * Fl + i) * Hl + j] = rnd ? dgc::rna_tf32_f(wn) : wn;
      }
      w[n] = wn;
    }
    __syncthreads();
#pragma unroll
    for (int n = 0; n < NJ; ++n) w_s[(jj * NJ + n) * Fl + i] = w[n];
    __syncthreads();
  }
}

template <int NJ>
__global__ void __launch_bounds__(512) evolve_bwd_kernel(
    int Fl, int Hl, int T, const float* __restrict__ Sr, const float* __restrict__ Sz,
    const float* __restrict__ Pc, const float* __restrict__ Qc, const float* __restrict__ sv_r,
    const float* __restrict__ sv_z, const float* __restrict__ sv_c, const float* __restrict__ sv_w,
    const float* __restrict__ dW_direct, float* __restrict__ dW0, float* __restrict__ da_r,
    float* __restrict__ da_z, float* __restrict__ da_c, float* __restrict__ dBr,
    float* __restrict__ dBz, float* __restrict__ dBc, int rnd) {
  extern __shared__ float sm[];
  const int CB = blockDim.y;
  float* dac_s = sm;                    // [CB*NJ][Fl]
  float* dar_s = sm + CB * NJ * Fl;
  float* daz_s = sm + 2 * CB * NJ * Fl;
  const int i = threadIdx.x, jj = threadIdx.y;
  const int jb = (blockIdx.x * CB + jj) * NJ;
  float carry[NJ], sbr[NJ], sbz[NJ], sbc[NJ];
#pragma unroll
  for (int n = 0; n < NJ; ++n) carry[n] = sbr[n] = sbz[n] = sbc[n] = 0.f;
  for (int t = T - 1; t >= 0; --t) {
    float r[NJ], z[NJ], c[NJ], w[NJ], dz[NJ], dw[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const int j = jb + n;
      const int64_t sidx = ((int64_t)i * T + t) * Hl + j;
      float g = carry[n];
      r[n] = z[n] = c[n] = w[n] = 0.f;
      if (j < Hl) {
        g += dW_direct[((int64_t)t * Fl + i) * Hl + j];  // grad wrt W_{t+1} (snapshot t+1)
        r[n] = sv_r[sidx];
        z[n] = sv_z[sidx];
        c[n] = sv_c[sidx];
        w[n] = sv_w[sidx];
      }
      dz[n] = g * (w[n] - c[n]);
      const float dc = g * (1.f - z[n]);
      dw[n] = g * z[n];
      dac_s[(jj * NJ + n) * Fl + i] = dc * (1.f - c[n] * c[n]);
    }
    __syncthreads();
    float drw[NJ], dpc[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) drw[n] = dpc[n] = 0.f;
    for (int k = 0; k < Fl; ++k) {
      const float qc = __ldg(Qc + (int64_t)k * Fl + i), pc = __ldg(Pc + (int64_t)k * Fl + i);
#pragma unroll
      for (int n = 0; n < NJ; ++n) {
        const float a = dac_s[(jj * NJ + n) * Fl + k];
        drw[n] = fmaf(qc, a, drw[n]);
        dpc[n] = fmaf(pc, a, dpc[n]);
      }
    }
    float dar[NJ], daz[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const float dr = drw[n] * w[n];
      dw[n] = fmaf(drw[n], r[n], dw[n]) + dpc[n];
      dar[n] = dr * r[n] * (1.f - r[n]);
      daz[n] = dz[n] * z[n] * (1.f - z[n]);
      dar_s[(jj * NJ + n) * Fl + i] = dar[n];
      daz_s[(jj * NJ + n) * Fl + i] = daz[n];
    }
    __syncthreads();
    for (int k = 0; k < Fl; ++k) {
      const float sr = __ldg(Sr + (int64_t)k * Fl + i), sz = __ldg(Sz + (int64_t)k * Fl + i);
#pragma unroll
      for (int n = 0; n < NJ; ++n)
        dw[n] = fmaf(sr, dar_s[(jj * NJ + n) * Fl + k], fmaf(sz, daz_s[(jj * NJ + n) * Fl + k], dw[n]));
    }
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const int j = jb + n;
      const float dac = dac_s[(jj * NJ + n) * Fl + i];
      if (j < Hl) {
        const int64_t sidx = ((int64_t)i * T + t) * Hl + j;
        da_r[sidx] = rnd ? dgc::rna_tf32_f(dar[n]) : dar[n];
        da_z[sidx] = rnd ? dgc::rna_tf32_f(daz[n]) : daz[n];
        da_c[sidx] = rnd ? dgc::rna_tf32_f(dac) : dac;
      }
      sbr[n] += dar[n];
      sbz[n] += daz[n];
      sbc[n] += dac;
      carry[n] = dw[n];
    }
    __syncthreads();
  }
#pragma unroll
  for (int n = 0; n < NJ; ++n) {
    const int j = jb + n;
    if (j < Hl) {
      dW0[(int64_t)i * Hl + j] = carry[n];
      dBr[(int64_t)i * Hl + j] = sbr[n];
      dBz[(int64_t)i * Hl + j] = sbz[n];
      dBc[(int64_t)i * Hl + j] = sbc[n];
    }
  }
}

// ---------------------------------------------------------------------------
// Cluster kernels (the default at F_l = 128): the gate matrices live in shared
// memory for the whole sequence. A 2-CTA cluster shares one group of NCOL
// columns and splits the F_l rows in halves: each CTA keeps its row half of all
// four gate matrices (8 F_l^2 bytes, 128 KB at F_l = 128), k-packed as
// G[g][k/4][row][k%4] so one 16-byte load feeds four FMAs, and computes those
// rows. The per-step column vectors every row needs (w and r*w forward; da_c,
// da_r, da_z backward) are exchanged by st.async into the peer's shared memory
// with complete_tx on its mbarrier, two exchanges per snapshot; each k-loop
// runs over the CTA's own half first and waits for the peer's half after it,
// so the exchange hides behind half of the loop (the halves are summed as
// separate partials, so every row uses the same order). The L2-streamed
// kernels above re-read 256 KB of gate matrices per snapshot and are
// latency-bound on those loads; they remain for the other shapes.
// ---------------------------------------------------------------------------
using dgc::tc::cluster_rank;
using dgc::tc::cluster_sync_all;
using dgc::tc::map_peer;
using dgc::tc::mbar_arrive_expect_tx;
using dgc::tc::mbar_init;
using dgc::tc::mbar_wait;
using dgc::tc::smem_u32;

__device__ __forceinline__ void put_f32(float* local, uint32_t peer, uint32_t peer_bar, float v) {
  *local = v;
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];"
               ::"r"(peer), "f"(v), "r"(peer_bar) : "memory");
}

// G[g][k/4][il][k%4] = M_g[k][row0 + il] (4-byte cp.async: the element
// transpose happens in flight; every load of the CTA is issued before the wait).
template <int RH>
__device__ __forceinline__ void stage_gates(float* G, int row0, int tid, int nthr, const float* M0,
                                            const float* M1, const float* M2, const float* M3) {
  constexpr int FL = 2 * RH, PER = FL * RH;
  for (int idx = tid; idx < 4 * PER; idx += nthr) {
    const int g = idx / PER, rem = idx - g * PER, k = rem / RH, il = rem - k * RH;
    const float* M = g == 0 ? M0 : g == 1 ? M1 : g == 2 ? M2 : M3;
    const uint32_t dst = smem_u32(G + (((g * (FL / 4) + (k >> 2)) * RH + il) << 2) + (k & 3));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst),
                 "l"(M + (int64_t)k * FL + row0 + il)
                 : "memory");
  }
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// acc[n] += sum_{k in [k0, k0 + RH)} G[k][il] * V[c0 + n][k]  for one gate.
template <int NJ, int RH>
__device__ __forceinline__ void dot_half(const float4* Gg, const float4* V, int k0, int c0,
                                         float* acc) {
  constexpr int FL = 2 * RH;
#pragma unroll 4
  for (int k4 = k0 / 4; k4 < (k0 + RH) / 4; ++k4) {
    const float4 g = Gg[k4 * RH];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const float4 v = V[(c0 + n) * (FL / 4) + k4];
      acc[n] = fmaf(g.x, v.x, fmaf(g.y, v.y, fmaf(g.z, v.z, fmaf(g.w, v.w, acc[n]))));
    }
  }
}
// three gates against one vector set (forward phase A)
template <int NJ, int RH>
__device__ __forceinline__ void dot3_half(const float4* G0, const float4* G1, const float4* G2,
                                          const float4* V, int k0, int c0, float* a0, float* a1,
                                          float* a2) {
  constexpr int FL = 2 * RH;
#pragma unroll 4
  for (int k4 = k0 / 4; k4 < (k0 + RH) / 4; ++k4) {
    const float4 g0 = G0[k4 * RH], g1 = G1[k4 * RH], g2 = G2[k4 * RH];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const float4 v = V[(c0 + n) * (FL / 4) + k4];
      a0[n] = fmaf(g0.x, v.x, fmaf(g0.y, v.y, fmaf(g0.z, v.z, fmaf(g0.w, v.w, a0[n]))));
      a1[n] = fmaf(g1.x, v.x, fmaf(g1.y, v.y, fmaf(g1.z, v.z, fmaf(g1.w, v.w, a1[n]))));
      a2[n] = fmaf(g2.x, v.x, fmaf(g2.y, v.y, fmaf(g2.z, v.z, fmaf(g2.w, v.w, a2[n]))));
    }
  }
}

template <int NJ, int CB, int RH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(RH * CB) evolve_fwd_cl_kernel(
    int Hl, int T, const float* __restrict__ W0, const float* __restrict__ SrT,
    const float* __restrict__ SzT, const float* __restrict__ PcT, const float* __restrict__ QcT,
    const float* __restrict__ Br, const float* __restrict__ Bz, const float* __restrict__ Bc,
    float* __restrict__ Wstack, float* __restrict__ sv_r, float* __restrict__ sv_z,
    float* __restrict__ sv_c, float* __restrict__ sv_w, float* __restrict__ sv_rw, int rnd) {
  constexpr int FL = 2 * RH, NCOL = CB * NJ, NT = RH * CB;
  extern __shared__ __align__(16) float sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);  // [0] r*w arrived, [1] w arrived
  float* G = sm + 4;                                 // [4][FL/4][RH][4]: Sr Sz Pc Qc rows
  float* w_s = G + 4 * FL * RH;                      // [NCOL][FL]
  float* rw_s = w_s + NCOL * FL;                     // [NCOL][FL]
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int il = threadIdx.x, jj = threadIdx.y, gi = (int)rank * RH + il;
  const int c0 = jj * NJ, j0 = (blockIdx.x >> 1) * NCOL, jb = j0 + c0;
  const int tid = threadIdx.y * RH + threadIdx.x;
  const int own0 = (int)rank * RH, peer0 = (int)peer * RH;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  stage_gates<RH>(G, own0, tid, NT, SrT, SzT, PcT, QcT);
  for (int idx = tid; idx < FL * NCOL; idx += NT) {  // W_0 for all rows of the group
    const int k = idx / NCOL, c = idx - k * NCOL, j = j0 + c;
    w_s[c * FL + k] = j < Hl ? __ldg(W0 + (int64_t)k * Hl + j) : 0.f;
  }
  cp_async_wait_all();
  cluster_sync_all();  // barriers initialised in both CTAs, shared memory staged
  const uint32_t rw_peer = map_peer(rw_s + c0 * FL + gi, peer);
  const uint32_t w_peer = map_peer(w_s + c0 * FL + gi, peer);
  const uint32_t bar_rw_peer = map_peer(&bar[0], peer), bar_w_peer = map_peer(&bar[1], peer);
  constexpr uint32_t kXBytes = RH * NCOL * sizeof(float);
  const float4* G4 = reinterpret_cast<const float4*>(G) + il;
  const float4* Gr = G4;
  const float4* Gz = G4 + (FL / 4) * RH;
  const float4* Gp = G4 + 2 * (FL / 4) * RH;
  const float4* Gq = G4 + 3 * (FL / 4) * RH;
  const float4* w4 = reinterpret_cast<const float4*>(w_s);
  const float4* rw4 = reinterpret_cast<const float4*>(rw_s);
  float w[NJ], br[NJ], bz[NJ], bc[NJ];
#pragma unroll
  for (int n = 0; n < NJ; ++n) {
    const int j = jb + n;
    const bool ok = j < Hl;
    w[n] = w_s[(c0 + n) * FL + gi];
    if (ok) Wstack[(int64_t)gi * Hl + j] = rnd ? dgc::rna_tf32_f(w[n]) : w[n];
    br[n] = ok ? Br[(int64_t)gi * Hl + j] : 0.f;
    bz[n] = ok ? Bz[(int64_t)gi * Hl + j] : 0.f;
    bc[n] = ok ? Bc[(int64_t)gi * Hl + j] : 0.f;
  }
  for (int t = 0; t < T; ++t) {
    // phase A: [Sr; Sz; Pc] w  (own row half of w first, then the peer's)
    float ar[NJ], az[NJ], ap[NJ], ar2[NJ], az2[NJ], ap2[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) ar[n] = az[n] = ap[n] = ar2[n] = az2[n] = ap2[n] = 0.f;
    dot3_half<NJ, RH>(Gr, Gz, Gp, w4, own0, c0, ar, az, ap);
    if (t > 0) mbar_wait(&bar[1], (t - 1) & 1);
    dot3_half<NJ, RH>(Gr, Gz, Gp, w4, peer0, c0, ar2, az2, ap2);
    float r[NJ], z[NJ], rw[NJ], aq[NJ], aq2[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const bool lo = rank == 0;  // partial over rows [0, RH) + partial over [RH, FL)
      r[n] = sgm((lo ? ar[n] + ar2[n] : ar2[n] + ar[n]) + br[n]);
      z[n] = sgm((lo ? az[n] + az2[n] : az2[n] + az[n]) + bz[n]);
      aq[n] = (lo ? ap[n] + ap2[n] : ap2[n] + ap[n]) + bc[n];
      rw[n] = r[n] * w[n];
      put_f32(rw_s + (c0 + n) * FL + gi, rw_peer + (uint32_t)(n * FL * 4), bar_rw_peer, rw[n]);
    }
    if (tid == 0) mbar_arrive_expect_tx(&bar[0], kXBytes);
    __syncthreads();
    // phase B: Qc (r * w)
#pragma unroll
    for (int n = 0; n < NJ; ++n) ap[n] = ap2[n] = 0.f;
    dot_half<NJ, RH>(Gq, rw4, own0, c0, ap);
    mbar_wait(&bar[0], t & 1);
    dot_half<NJ, RH>(Gq, rw4, peer0, c0, ap2);
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      aq2[n] = rank == 0 ? ap[n] + ap2[n] : ap2[n] + ap[n];
      const int j = jb + n;
      const float c = tanhf(aq[n] + aq2[n]);
      const float wn = (1.f - z[n]) * c + z[n] * w[n];
      if (j < Hl) {
        const int64_t sidx = ((int64_t)gi * T + t) * Hl + j;  // [Fl][T][Hl]
        sv_r[sidx] = r[n];
        sv_z[sidx] = z[n];
        sv_c[sidx] = c;
        sv_w[sidx] = rnd ? dgc::rna_tf32_f(w[n]) : w[n];
        sv_rw[sidx] = rnd ? dgc::rna_tf32_f(rw[n]) : rw[n];
        Wstack[((int64_t)(t + 1) * FL + gi) * Hl + j] = rnd ? dgc::rna_tf32_f(wn) : wn;
      }
      w[n] = wn;
    }
    if (t + 1 < T) {
#pragma unroll
      for (int n = 0; n < NJ; ++n)
        put_f32(w_s + (c0 + n) * FL + gi, w_peer + (uint32_t)(n * FL * 4), bar_w_peer, w[n]);
      if (tid == 0) mbar_arrive_expect_tx(&bar[1], kXBytes);
      __syncthreads();
    }
  }
  cluster_sync_all();  // no st.async may still target this CTA's shared memory
}

template <int NJ, int CB, int RH>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(RH * CB) evolve_bwd_cl_kernel(
    int Hl, int T, const float* __restrict__ Sr, const float* __restrict__ Sz,
    const float* __restrict__ Pc, const float* __restrict__ Qc, const float* __restrict__ sv_r,
    const float* __restrict__ sv_z, const float* __restrict__ sv_c, const float* __restrict__ sv_w,
    const float* __restrict__ dW_direct, float* __restrict__ dW0, float* __restrict__ da_r,
    float* __restrict__ da_z, float* __restrict__ da_c, float* __restrict__ dBr,
    float* __restrict__ dBz, float* __restrict__ dBc, int rnd) {
  constexpr int FL = 2 * RH, NCOL = CB * NJ, NT = RH * CB;
  extern __shared__ __align__(16) float sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);  // [0] da_c arrived, [1] da_r/da_z arrived
  float* G = sm + 4;                                 // [4][FL/4][RH][4]: Qc^T Pc^T Sr^T Sz^T rows
  float* dac_s = G + 4 * FL * RH;                    // [NCOL][FL]
  float* dar_s = dac_s + NCOL * FL;
  float* daz_s = dar_s + NCOL * FL;
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int il = threadIdx.x, jj = threadIdx.y, gi = (int)rank * RH + il;
  const int c0 = jj * NJ, jb = (blockIdx.x >> 1) * NCOL + c0;
  const int tid = threadIdx.y * RH + threadIdx.x;
  const int own0 = (int)rank * RH, peer0 = (int)peer * RH;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  stage_gates<RH>(G, own0, tid, NT, Qc, Pc, Sr, Sz);
  // inputs of the first BPTT step (t = T - 1) in flight with the staging
  float nxt_d[NJ], nxt_r[NJ], nxt_z[NJ], nxt_c[NJ], nxt_w[NJ];
  auto fetch = [&](int t) {
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const int j = jb + n;
      const int64_t sidx = ((int64_t)gi * T + t) * Hl + j;
      const bool ok = j < Hl;
      nxt_d[n] = ok ? __ldg(dW_direct + ((int64_t)t * FL + gi) * Hl + j) : 0.f;
      nxt_r[n] = ok ? __ldg(sv_r + sidx) : 0.f;
      nxt_z[n] = ok ? __ldg(sv_z + sidx) : 0.f;
      nxt_c[n] = ok ? __ldg(sv_c + sidx) : 0.f;
      nxt_w[n] = ok ? __ldg(sv_w + sidx) : 0.f;
    }
  };
  fetch(T - 1);
  cp_async_wait_all();
  cluster_sync_all();
  const uint32_t dac_peer = map_peer(dac_s + c0 * FL + gi, peer);
  const uint32_t dar_peer = map_peer(dar_s + c0 * FL + gi, peer);
  const uint32_t daz_peer = map_peer(daz_s + c0 * FL + gi, peer);
  const uint32_t bar_c_peer = map_peer(&bar[0], peer), bar_rz_peer = map_peer(&bar[1], peer);
  constexpr uint32_t kXBytes = RH * NCOL * sizeof(float);
  const float4* G4 = reinterpret_cast<const float4*>(G) + il;
  const float4* Gq = G4;
  const float4* Gp = G4 + (FL / 4) * RH;
  const float4* Gr = G4 + 2 * (FL / 4) * RH;
  const float4* Gz = G4 + 3 * (FL / 4) * RH;
  const float4* dac4 = reinterpret_cast<const float4*>(dac_s);
  const float4* dar4 = reinterpret_cast<const float4*>(dar_s);
  const float4* daz4 = reinterpret_cast<const float4*>(daz_s);
  const bool lo = rank == 0;
  float carry[NJ], sbr[NJ], sbz[NJ], sbc[NJ];
#pragma unroll
  for (int n = 0; n < NJ; ++n) carry[n] = sbr[n] = sbz[n] = sbc[n] = 0.f;
  for (int t = T - 1, s = 0; t >= 0; --t, ++s) {
    float r[NJ], z[NJ], w[NJ], dz[NJ], dw[NJ], dac[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const float g = carry[n] + nxt_d[n];  // grad wrt W_{t+1} (snapshot t+1)
      const float c = nxt_c[n];
      r[n] = nxt_r[n];
      z[n] = nxt_z[n];
      w[n] = nxt_w[n];
      dz[n] = g * (w[n] - c);
      dw[n] = g * z[n];
      dac[n] = g * (1.f - z[n]) * (1.f - c * c);
      put_f32(dac_s + (c0 + n) * FL + gi, dac_peer + (uint32_t)(n * FL * 4), bar_c_peer, dac[n]);
    }
    if (t > 0) fetch(t - 1);  // next step's inputs stream in under this step
    if (tid == 0) mbar_arrive_expect_tx(&bar[0], kXBytes);
    __syncthreads();
    float drw[NJ], dpc[NJ], drw2[NJ], dpc2[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) drw[n] = dpc[n] = drw2[n] = dpc2[n] = 0.f;
    dot_half<NJ, RH>(Gq, dac4, own0, c0, drw);
    dot_half<NJ, RH>(Gp, dac4, own0, c0, dpc);
    mbar_wait(&bar[0], s & 1);
    dot_half<NJ, RH>(Gq, dac4, peer0, c0, drw2);
    dot_half<NJ, RH>(Gp, dac4, peer0, c0, dpc2);
    float dar[NJ], daz[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const float drw_t = lo ? drw[n] + drw2[n] : drw2[n] + drw[n];
      const float dpc_t = lo ? dpc[n] + dpc2[n] : dpc2[n] + dpc[n];
      const float dr = drw_t * w[n];
      dw[n] = fmaf(drw_t, r[n], dw[n]) + dpc_t;
      dar[n] = dr * r[n] * (1.f - r[n]);
      daz[n] = dz[n] * z[n] * (1.f - z[n]);
      put_f32(dar_s + (c0 + n) * FL + gi, dar_peer + (uint32_t)(n * FL * 4), bar_rz_peer, dar[n]);
      put_f32(daz_s + (c0 + n) * FL + gi, daz_peer + (uint32_t)(n * FL * 4), bar_rz_peer, daz[n]);
    }
    if (tid == 0) mbar_arrive_expect_tx(&bar[1], 2 * kXBytes);
    __syncthreads();
    float e1[NJ], e2[NJ], f1[NJ], f2[NJ];
#pragma unroll
    for (int n = 0; n < NJ; ++n) e1[n] = e2[n] = f1[n] = f2[n] = 0.f;
    dot_half<NJ, RH>(Gr, dar4, own0, c0, e1);
    dot_half<NJ, RH>(Gz, daz4, own0, c0, f1);
    mbar_wait(&bar[1], s & 1);
    dot_half<NJ, RH>(Gr, dar4, peer0, c0, e2);
    dot_half<NJ, RH>(Gz, daz4, peer0, c0, f2);
#pragma unroll
    for (int n = 0; n < NJ; ++n) {
      const float er = lo ? e1[n] + e2[n] : e2[n] + e1[n];
      const float ez = lo ? f1[n] + f2[n] : f2[n] + f1[n];
      dw[n] += er + ez;
      const int j = jb + n;
      if (j < Hl) {
        const int64_t sidx = ((int64_t)gi * T + t) * Hl + j;
        da_r[sidx] = rnd ? dgc::rna_tf32_f(dar[n]) : dar[n];
        da_z[sidx] = rnd ? dgc::rna_tf32_f(daz[n]) : daz[n];
        da_c[sidx] = rnd ? dgc::rna_tf32_f(dac[n]) : dac[n];
      }
      sbr[n] += dar[n];
      sbz[n] += daz[n];
      sbc[n] += dac[n];
      carry[n] = dw[n];
    }
  }
#pragma unroll
  for (int n = 0; n < NJ; ++n) {
    const int j = jb + n;
    if (j < Hl) {
      dW0[(int64_t)gi * Hl + j] = carry[n];
      dBr[(int64_t)gi * Hl + j] = sbr[n];
      dBz[(int64_t)gi * Hl + j] = sbz[n];
      dBc[(int64_t)gi * Hl + j] = sbc[n];
    }
  }
  cluster_sync_all();
}

// Cluster-kernel shape: NJ columns per thread x CB column groups per CTA
// (DGC_EVOLVE_CL="NJ,CB" in {1,1 1,2 1,4 2,2}; "0" selects the L2-streamed kernels).
int evolve_cl_variant() {
  const char* e = getenv("DGC_EVOLVE_CL");
  if (!e) return 12;
  int nj = 0, cb = 1;
  if (sscanf(e, "%d,%d", &nj, &cb) < 1 || nj == 0) return 0;
  const int v = nj * 10 + cb;
  return (v == 11 || v == 12 || v == 14 || v == 22) ? v : 12;
}

template <int NJ, int CB, int NX>
constexpr size_t evolve_cl_smem() {
  return 16 + (size_t)(4 * 128 * 64 + NX * NJ * CB * 128) * sizeof(float);
}

template <int NJ, int CB, int NX, typename Kern, typename... Args>
int launch_cl(Kern kern, int Hl, cudaStream_t st, const char* name, Args... args) {
  constexpr int NCOL = NJ * CB;
  constexpr size_t smem = evolve_cl_smem<NJ, CB, NX>();
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::fail(DGC_ERR_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
  const unsigned groups = (unsigned)((Hl + NCOL - 1) / NCOL);
  kern<<<2 * groups, dim3(64, CB), smem, st>>>(args...);
  DGC_CHECK_LAUNCH(name);
  return DGC_OK;
}

int evolve_nj() {
  const char* e = getenv("DGC_EVOLVE_NJ");
  const int v = e ? atoi(e) : 1;
  return (v == 1 || v == 2 || v == 4 || v == 8) ? v : 1;
}

}  // namespace

#define DGC_EVOLVE_DISPATCH(KERN, SMEM_MULT, ...)                                          \
  do {                                                                                     \
    const int nj = evolve_nj();                                                            \
    const int CB = Fl <= 128 ? 2 : 1;                                                      \
    dim3 block(Fl, CB);                                                                    \
    const size_t shm = (size_t)SMEM_MULT * CB * nj * Fl * sizeof(float);                   \
    const unsigned grid = (unsigned)((Hl + CB * nj - 1) / (CB * nj));                      \
    cudaStream_t st = dgc::as_stream(stream);                                              \
    if (nj == 1) KERN<1><<<grid, block, shm, st>>>(__VA_ARGS__);                           \
    else if (nj == 2) KERN<2><<<grid, block, shm, st>>>(__VA_ARGS__);                      \
    else if (nj == 8) KERN<8><<<grid, block, shm, st>>>(__VA_ARGS__);                      \
    else KERN<4><<<grid, block, shm, st>>>(__VA_ARGS__);                                   \
  } while (0)

extern "C" int dgc_evolve_fwd(int32_t Fl, int32_t Hl, int32_t T, const float* W0, const float* SrT,
                              const float* SzT, const float* PcT, const float* QcT,
                              const float* Br, const float* Bz, const float* Bc, float* Wstack,
                              float* sv_r, float* sv_z, float* sv_c, float* sv_w, float* sv_rw,
                              int32_t flags, void* stream) {
  DGC_REQUIRE(Fl >= 1 && Fl <= 512 && Hl >= 1, "evolve_fwd: bad shape (F <= 512)");
  const int v = evolve_cl_variant();
  if (Fl == 128 && v) {
    cudaStream_t st = dgc::as_stream(stream);
#define DGC_FWD_ARGS Hl, T, W0, SrT, SzT, PcT, QcT, Br, Bz, Bc, Wstack, sv_r, sv_z, sv_c, sv_w, sv_rw, flags & 1
#define DGC_FWD(NJ, CB) launch_cl<NJ, CB, 2>(evolve_fwd_cl_kernel<NJ, CB, 64>, Hl, st, "evolve_fwd_cl", DGC_FWD_ARGS)
    if (v == 11) return DGC_FWD(1, 1);
    if (v == 14) return DGC_FWD(1, 4);
    if (v == 22) return DGC_FWD(2, 2);
    return DGC_FWD(1, 2);
#undef DGC_FWD
#undef DGC_FWD_ARGS
  }
  DGC_EVOLVE_DISPATCH(evolve_fwd_kernel, 2, Fl, Hl, T, W0, SrT, SzT, PcT, QcT, Br, Bz, Bc, Wstack,
                      sv_r, sv_z, sv_c, sv_w, sv_rw, flags & 1);
  DGC_CHECK_LAUNCH("evolve_fwd_kernel");
  return DGC_OK;
}

extern "C" int dgc_evolve_bwd(int32_t Fl, int32_t Hl, int32_t T, const float* Sr, const float* Sz,
                              const float* Pc, const float* Qc, const float* sv_r,
                              const float* sv_z, const float* sv_c, const float* sv_w,
                              const float* dW_direct, float* dW0, float* da_r, float* da_z,
                              float* da_c, float* dBr, float* dBz, float* dBc, int32_t flags,
                              void* stream) {
  DGC_REQUIRE(Fl >= 1 && Fl <= 512 && Hl >= 1, "evolve_bwd: bad shape (F <= 512)");
  const int v = evolve_cl_variant();
  if (Fl == 128 && v) {
    cudaStream_t st = dgc::as_stream(stream);
#define DGC_BWD_ARGS Hl, T, Sr, Sz, Pc, Qc, sv_r, sv_z, sv_c, sv_w, dW_direct, dW0, da_r, da_z, da_c, dBr, dBz, dBc, flags & 1
#define DGC_BWD(NJ, CB) launch_cl<NJ, CB, 3>(evolve_bwd_cl_kernel<NJ, CB, 64>, Hl, st, "evolve_bwd_cl", DGC_BWD_ARGS)
    if (v == 11) return DGC_BWD(1, 1);
    if (v == 14) return DGC_BWD(1, 4);
    if (v == 22) return DGC_BWD(2, 2);
    return DGC_BWD(1, 2);
#undef DGC_BWD
#undef DGC_BWD_ARGS
  }
  DGC_EVOLVE_DISPATCH(evolve_bwd_kernel, 3, Fl, Hl, T, Sr, Sz, Pc, Qc, sv_r, sv_z, sv_c, sv_w,
                      dW_direct, dW0, da_r, da_z, da_c, dBr, dBz, dBc, flags & 1);
  DGC_CHECK_LAUNCH("evolve_bwd_kernel");
  return DGC_OK;
}
