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
    int Fl, int Hl, int T, const float* __restrict__ W0, const float* __restrict__ Sr,
    const float* __restrict__ Sz, const float* __restrict__ Pc, const float* __restrict__ Qc,
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
      const float sr = __ldg(Sr + (int64_t)i * Fl + k), sz = __ldg(Sz + (int64_t)i * Fl + k),
                  pc = __ldg(Pc + (int64_t)i * Fl + k);
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
      const float qc = __ldg(Qc + (int64_t)i * Fl + k);
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
// Cluster kernels (the default at F_l = 128). A 2-CTA cluster shares one group
// of NCOL columns and splits the F_l rows in halves; the per-step column
// vectors every row needs (w and r*w forward; da_c, da_r, da_z backward) are
// exchanged by st.async into the peer's shared memory with complete_tx on its
// mbarrier, two exchanges per snapshot, and each lane's k-slice of its own half
// is summed before it waits for the peer's. The L2-streamed kernels above
// re-read 256 KB of gate matrices per snapshot and are latency-bound on those
// loads (2.6 ms per launch at C3 vs 0.15 ms); they remain for other shapes.
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

__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// four independent partial chains (k mod 4) keep the FMA pipe fed, summed at the end
__device__ __forceinline__ void fma4(float4& a, const float4& g, const float4& v) {
  a.x = fmaf(g.x, v.x, a.x);
  a.y = fmaf(g.y, v.y, a.y);
  a.z = fmaf(g.z, v.z, a.z);
  a.w = fmaf(g.w, v.w, a.w);
}
__device__ __forceinline__ float hsum(const float4& a) { return (a.x + a.y) + (a.z + a.w); }

// ---------------------------------------------------------------------------
// Register-resident variant (the default): the CTA's row half of the four
// gate matrices lives in REGISTERS (128 per thread), so the per-step k-loops
// read only the exchanged column vectors from shared memory. Thread
// (row il, slice q) owns k in {own0 + 16q .. +16} and {peer0 + 16q .. +16}
// (own slice first, the peer's after its mbarrier), the four slice partials
// of a row are combined with two xor-shuffles (lanes 4il..4il+3), and every
// lane of the quad then holds the full sums. Vectors are stored with a
// 20-float pitch per 16-k slice so the four slices of a quad hit disjoint banks.
// ---------------------------------------------------------------------------
constexpr int kRR_RH = 64, kRR_FL = 128, kRR_SP = 20, kRR_VP = 8 * kRR_SP;  // 160 floats
__device__ __forceinline__ int rr_pos(int k) { return (k >> 4) * kRR_SP + (k & 15); }

// One gate's row half -> registers g[0..15] (own slice), g[16..31] (peer slice):
// g[m] = A[own0 + il][k_m] where A = M (ROWS) or A = M^T (COLUMNS). The staging
// tile has pitch RH + 1 so both the in-flight transpose and the reads are
// conflict-free.
enum class RrSrc { kRows, kColumns };
template <RrSrc SRC>
__device__ __forceinline__ void rr_load_gate(float* stage, const float* M, int own0, int peer0,
                                             int il, int q, int tid, float* g) {
  constexpr int P = kRR_RH + 1;
  for (int idx = tid; idx < kRR_FL * kRR_RH; idx += 256) {
    int k, i;
    const float* src;
    if constexpr (SRC == RrSrc::kRows) {  // row own0 + i of M, coalesced along k
      i = idx / kRR_FL, k = idx - i * kRR_FL;
      src = M + (int64_t)(own0 + i) * kRR_FL + k;
    } else {  // column own0 + i of M, coalesced along i
      k = idx / kRR_RH, i = idx - k * kRR_RH;
      src = M + (int64_t)k * kRR_FL + own0 + i;
    }
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(stage + k * P + i)),
                 "l"(src)
                 : "memory");
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    g[m] = stage[(own0 + 16 * q + m) * P + il];
    g[16 + m] = stage[(peer0 + 16 * q + m) * P + il];
  }
  __syncthreads();
}

// partial dot of 16 gate registers with 16 vector entries starting at slice base
__device__ __forceinline__ float rr_dot16(const float* g, const float* v) {
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
  for (int m = 0; m < 4; ++m) fma4(a, make_float4(g[4 * m], g[4 * m + 1], g[4 * m + 2], g[4 * m + 3]),
                                   reinterpret_cast<const float4*>(v)[m]);
  return hsum(a);
}
__device__ __forceinline__ float quad_sum(float x) {
  x += __shfl_xor_sync(0xffffffffu, x, 1);
  return x + __shfl_xor_sync(0xffffffffu, x, 2);
}

template <int NCOL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) evolve_fwd_rr_kernel(
    int Hl, int T, const float* __restrict__ W0, const float* __restrict__ Sr,
    const float* __restrict__ Sz, const float* __restrict__ Pc, const float* __restrict__ Qc,
    const float* __restrict__ Br, const float* __restrict__ Bz, const float* __restrict__ Bc,
    float* __restrict__ Wstack, float* __restrict__ sv_r, float* __restrict__ sv_z,
    float* __restrict__ sv_c, float* __restrict__ sv_w, float* __restrict__ sv_rw, int rnd) {
  constexpr int RH = kRR_RH, FL = kRR_FL;
  extern __shared__ __align__(16) float sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);  // [0] r*w arrived, [1] w arrived
  float* w_s = sm + 4;                               // [NCOL][VP]
  float* rw_s = w_s + NCOL * kRR_VP;                 // [NCOL][VP]
  float* stage = rw_s + NCOL * kRR_VP;               // [FL][RH] staging of one gate
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int tid = threadIdx.x, q = tid & 3, il = tid >> 2, gi = (int)rank * RH + il;
  const int own0 = (int)rank * RH, peer0 = (int)peer * RH, j0 = (blockIdx.x >> 1) * NCOL;
  const bool lo = rank == 0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int idx = tid; idx < FL * NCOL; idx += 256) {  // W_0 for all rows of the group
    const int k = idx / NCOL, c = idx - k * NCOL, j = j0 + c;
    w_s[c * kRR_VP + rr_pos(k)] = j < Hl ? __ldg(W0 + (int64_t)k * Hl + j) : 0.f;
  }
  float gr[32], gz[32], gp[32], gq[32];
  rr_load_gate<RrSrc::kRows>(stage, Sr, own0, peer0, il, q, tid, gr);
  rr_load_gate<RrSrc::kRows>(stage, Sz, own0, peer0, il, q, tid, gz);
  rr_load_gate<RrSrc::kRows>(stage, Pc, own0, peer0, il, q, tid, gp);
  rr_load_gate<RrSrc::kRows>(stage, Qc, own0, peer0, il, q, tid, gq);
  cluster_sync_all();
  const uint32_t rw_peer = map_peer(rw_s + rr_pos(gi), peer);
  const uint32_t w_peer = map_peer(w_s + rr_pos(gi), peer);
  const uint32_t bar_rw_peer = map_peer(&bar[0], peer), bar_w_peer = map_peer(&bar[1], peer);
  constexpr uint32_t kXBytes = RH * NCOL * sizeof(float);
  const int own_off = rr_pos(own0 + 16 * q), peer_off = rr_pos(peer0 + 16 * q);
  float w[NCOL], br[NCOL], bz[NCOL], bc[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    const int j = j0 + c;
    const bool ok = j < Hl;
    w[c] = w_s[c * kRR_VP + rr_pos(gi)];
    if (ok && (c & 3) == q) Wstack[(int64_t)gi * Hl + j] = rnd ? dgc::rna_tf32_f(w[c]) : w[c];
    br[c] = ok ? __ldg(Br + (int64_t)gi * Hl + j) : 0.f;
    bz[c] = ok ? __ldg(Bz + (int64_t)gi * Hl + j) : 0.f;
    bc[c] = ok ? __ldg(Bc + (int64_t)gi * Hl + j) : 0.f;
  }
  for (int t = 0; t < T; ++t) {
    // phase A: [Sr; Sz; Pc] w over this lane's own-half slice, then the peer's
    float pr[NCOL], pz[NCOL], pp[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float* v = w_s + c * kRR_VP + own_off;
      pr[c] = rr_dot16(gr, v);
      pz[c] = rr_dot16(gz, v);
      pp[c] = rr_dot16(gp, v);
    }
    if (t > 0) mbar_wait(&bar[1], (t - 1) & 1);
    float r[NCOL], z[NCOL], rw[NCOL], aq[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float* v = w_s + c * kRR_VP + peer_off;
      const float xr = rr_dot16(gr + 16, v), xz = rr_dot16(gz + 16, v), xp = rr_dot16(gp + 16, v);
      r[c] = sgm(quad_sum(lo ? pr[c] + xr : xr + pr[c]) + br[c]);
      z[c] = sgm(quad_sum(lo ? pz[c] + xz : xz + pz[c]) + bz[c]);
      aq[c] = quad_sum(lo ? pp[c] + xp : xp + pp[c]) + bc[c];
      rw[c] = r[c] * w[c];
      if ((c & 3) == q)
        put_f32(rw_s + c * kRR_VP + rr_pos(gi), rw_peer + (uint32_t)(c * kRR_VP * 4), bar_rw_peer,
                rw[c]);
    }
    if (tid == 0) mbar_arrive_expect_tx(&bar[0], kXBytes);
    __syncthreads();
    // phase B: Qc (r * w)
    float pq[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) pq[c] = rr_dot16(gq, rw_s + c * kRR_VP + own_off);
    mbar_wait(&bar[0], t & 1);
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float xq = rr_dot16(gq + 16, rw_s + c * kRR_VP + peer_off);
      const float cc = tanhf(aq[c] + quad_sum(lo ? pq[c] + xq : xq + pq[c]));
      const float wn = (1.f - z[c]) * cc + z[c] * w[c];
      const int j = j0 + c;
      if (j < Hl && (c & 3) == q) {
        const int64_t sidx = ((int64_t)gi * T + t) * Hl + j;  // [Fl][T][Hl]
        sv_r[sidx] = r[c];
        sv_z[sidx] = z[c];
        sv_c[sidx] = cc;
        sv_w[sidx] = rnd ? dgc::rna_tf32_f(w[c]) : w[c];
        sv_rw[sidx] = rnd ? dgc::rna_tf32_f(rw[c]) : rw[c];
        Wstack[((int64_t)(t + 1) * FL + gi) * Hl + j] = rnd ? dgc::rna_tf32_f(wn) : wn;
      }
      w[c] = wn;
    }
    if (t + 1 < T) {
#pragma unroll
      for (int c = 0; c < NCOL; ++c)
        if ((c & 3) == q)
          put_f32(w_s + c * kRR_VP + rr_pos(gi), w_peer + (uint32_t)(c * kRR_VP * 4), bar_w_peer,
                  w[c]);
      if (tid == 0) mbar_arrive_expect_tx(&bar[1], kXBytes);
      __syncthreads();
    }
  }
  cluster_sync_all();  // no st.async may still target this CTA's shared memory
}

template <int NCOL>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) evolve_bwd_rr_kernel(
    int Hl, int T, const float* __restrict__ Sr, const float* __restrict__ Sz,
    const float* __restrict__ Pc, const float* __restrict__ Qc, const float* __restrict__ sv_r,
    const float* __restrict__ sv_z, const float* __restrict__ sv_c, const float* __restrict__ sv_w,
    const float* __restrict__ dW_direct, float* __restrict__ dW0, float* __restrict__ da_r,
    float* __restrict__ da_z, float* __restrict__ da_c, float* __restrict__ dBr,
    float* __restrict__ dBz, float* __restrict__ dBc, int rnd) {
  constexpr int RH = kRR_RH, FL = kRR_FL;
  extern __shared__ __align__(16) float sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm);  // [0] da_c arrived, [1] da_r/da_z arrived
  float* dac_s = sm + 4;                             // [NCOL][VP]
  float* dar_s = dac_s + NCOL * kRR_VP;
  float* daz_s = dar_s + NCOL * kRR_VP;
  float* stage = daz_s + NCOL * kRR_VP;
  const uint32_t rank = cluster_rank(), peer = rank ^ 1u;
  const int tid = threadIdx.x, q = tid & 3, il = tid >> 2, gi = (int)rank * RH + il;
  const int own0 = (int)rank * RH, peer0 = (int)peer * RH, j0 = (blockIdx.x >> 1) * NCOL;
  const bool lo = rank == 0;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // gate g's column gi over k: M_g[k][gi]
  float gq[32], gp[32], gr[32], gz[32];
  rr_load_gate<RrSrc::kColumns>(stage, Qc, own0, peer0, il, q, tid, gq);
  rr_load_gate<RrSrc::kColumns>(stage, Pc, own0, peer0, il, q, tid, gp);
  rr_load_gate<RrSrc::kColumns>(stage, Sr, own0, peer0, il, q, tid, gr);
  rr_load_gate<RrSrc::kColumns>(stage, Sz, own0, peer0, il, q, tid, gz);
  float nd[NCOL], nr[NCOL], nz[NCOL], nc[NCOL], nw[NCOL];
  auto fetch = [&](int t) {
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const int j = j0 + c;
      const int64_t sidx = ((int64_t)gi * T + t) * Hl + j;
      const bool ok = j < Hl;
      nd[c] = ok ? __ldg(dW_direct + ((int64_t)t * FL + gi) * Hl + j) : 0.f;
      nr[c] = ok ? __ldg(sv_r + sidx) : 0.f;
      nz[c] = ok ? __ldg(sv_z + sidx) : 0.f;
      nc[c] = ok ? __ldg(sv_c + sidx) : 0.f;
      nw[c] = ok ? __ldg(sv_w + sidx) : 0.f;
    }
  };
  fetch(T - 1);
  cluster_sync_all();
  const uint32_t dac_peer = map_peer(dac_s + rr_pos(gi), peer);
  const uint32_t dar_peer = map_peer(dar_s + rr_pos(gi), peer);
  const uint32_t daz_peer = map_peer(daz_s + rr_pos(gi), peer);
  const uint32_t bar_c_peer = map_peer(&bar[0], peer), bar_rz_peer = map_peer(&bar[1], peer);
  constexpr uint32_t kXBytes = RH * NCOL * sizeof(float);
  const int own_off = rr_pos(own0 + 16 * q), peer_off = rr_pos(peer0 + 16 * q);
  float carry[NCOL], sbr[NCOL], sbz[NCOL], sbc[NCOL];
#pragma unroll
  for (int c = 0; c < NCOL; ++c) carry[c] = sbr[c] = sbz[c] = sbc[c] = 0.f;
  for (int t = T - 1, s = 0; t >= 0; --t, ++s) {
    float r[NCOL], z[NCOL], w[NCOL], dz[NCOL], dw[NCOL], dac[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float g = carry[c] + nd[c];  // grad wrt W_{t+1} (snapshot t+1)
      const float cc = nc[c];
      r[c] = nr[c];
      z[c] = nz[c];
      w[c] = nw[c];
      dz[c] = g * (w[c] - cc);
      dw[c] = g * z[c];
      dac[c] = g * (1.f - z[c]) * (1.f - cc * cc);
      if ((c & 3) == q)
        put_f32(dac_s + c * kRR_VP + rr_pos(gi), dac_peer + (uint32_t)(c * kRR_VP * 4), bar_c_peer,
                dac[c]);
    }
    if (t > 0) fetch(t - 1);  // next step's inputs stream in under this step
    if (tid == 0) mbar_arrive_expect_tx(&bar[0], kXBytes);
    __syncthreads();
    float pq[NCOL], pp[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float* v = dac_s + c * kRR_VP + own_off;
      pq[c] = rr_dot16(gq, v);
      pp[c] = rr_dot16(gp, v);
    }
    mbar_wait(&bar[0], s & 1);
    float dar[NCOL], daz[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float* v = dac_s + c * kRR_VP + peer_off;
      const float xq = rr_dot16(gq + 16, v), xp = rr_dot16(gp + 16, v);
      const float drw = quad_sum(lo ? pq[c] + xq : xq + pq[c]);
      const float dpc = quad_sum(lo ? pp[c] + xp : xp + pp[c]);
      dw[c] = fmaf(drw, r[c], dw[c]) + dpc;
      dar[c] = drw * w[c] * r[c] * (1.f - r[c]);
      daz[c] = dz[c] * z[c] * (1.f - z[c]);
      if ((c & 3) == q) {
        put_f32(dar_s + c * kRR_VP + rr_pos(gi), dar_peer + (uint32_t)(c * kRR_VP * 4), bar_rz_peer,
                dar[c]);
        put_f32(daz_s + c * kRR_VP + rr_pos(gi), daz_peer + (uint32_t)(c * kRR_VP * 4), bar_rz_peer,
                daz[c]);
      }
    }
    if (tid == 0) mbar_arrive_expect_tx(&bar[1], 2 * kXBytes);
    __syncthreads();
    float pr[NCOL], pz[NCOL];
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      pr[c] = rr_dot16(gr, dar_s + c * kRR_VP + own_off);
      pz[c] = rr_dot16(gz, daz_s + c * kRR_VP + own_off);
    }
    mbar_wait(&bar[1], s & 1);
#pragma unroll
    for (int c = 0; c < NCOL; ++c) {
      const float xr = rr_dot16(gr + 16, dar_s + c * kRR_VP + peer_off);
      const float xz = rr_dot16(gz + 16, daz_s + c * kRR_VP + peer_off);
      const float er = quad_sum(lo ? pr[c] + xr : xr + pr[c]);
      const float ez = quad_sum(lo ? pz[c] + xz : xz + pz[c]);
      dw[c] += er + ez;
      const int j = j0 + c;
      if (j < Hl && (c & 3) == q) {
        const int64_t sidx = ((int64_t)gi * T + t) * Hl + j;
        da_r[sidx] = rnd ? dgc::rna_tf32_f(dar[c]) : dar[c];
        da_z[sidx] = rnd ? dgc::rna_tf32_f(daz[c]) : daz[c];
        da_c[sidx] = rnd ? dgc::rna_tf32_f(dac[c]) : dac[c];
      }
      sbr[c] += dar[c];
      sbz[c] += daz[c];
      sbc[c] += dac[c];
      carry[c] = dw[c];
    }
  }
#pragma unroll
  for (int c = 0; c < NCOL; ++c) {
    const int j = j0 + c;
    if (j < Hl && (c & 3) == q) {
      dW0[(int64_t)gi * Hl + j] = carry[c];
      dBr[(int64_t)gi * Hl + j] = sbr[c];
      dBz[(int64_t)gi * Hl + j] = sbz[c];
      dBc[(int64_t)gi * Hl + j] = sbc[c];
    }
  }
  cluster_sync_all();
}

template <int NCOL, int NX, typename Kern, typename... Args>
int launch_rr(Kern kern, int Hl, cudaStream_t st, const char* name, Args... args) {
  constexpr size_t smem = 16 + (size_t)(NX * NCOL * kRR_VP + kRR_FL * (kRR_RH + 1)) * sizeof(float);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::fail(DGC_ERR_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
  const unsigned groups = (unsigned)((Hl + NCOL - 1) / NCOL);
  kern<<<2 * groups, 256, smem, st>>>(args...);
  DGC_CHECK_LAUNCH(name);
  return DGC_OK;
}

// Weight-evolution kernel: DGC_EVOLVE_CL = "rr1" | "rr2" (default) | "rr4" columns
// per cluster for the register-resident kernels, "0" for the L2-streamed ones.
int evolve_rr_cols() {
  const char* e = getenv("DGC_EVOLVE_CL");
  if (!e) return 2;
  if (e[0] == 'r' && e[1] == 'r') {
    const int n = atoi(e + 2);
    return n == 1 || n == 4 ? n : 2;
  }
  return 0;
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

extern "C" int dgc_evolve_fwd(int32_t Fl, int32_t Hl, int32_t T, const float* W0, const float* Sr,
                              const float* Sz, const float* Pc, const float* Qc,
                              const float* Br, const float* Bz, const float* Bc, float* Wstack,
                              float* sv_r, float* sv_z, float* sv_c, float* sv_w, float* sv_rw,
                              int32_t flags, void* stream) {
  DGC_REQUIRE(Fl >= 1 && Fl <= 512 && Hl >= 1, "evolve_fwd: bad shape (F <= 512)");
  const int nc = evolve_rr_cols();
  if (Fl == 128 && nc) {  // register-resident cluster kernels
    cudaStream_t st = dgc::as_stream(stream);
#define DGC_FWD_RR(N)                                                                           \
  launch_rr<N, 2>(evolve_fwd_rr_kernel<N>, Hl, st, "evolve_fwd_rr", Hl, T, W0, Sr, Sz, Pc, \
                  Qc, Br, Bz, Bc, Wstack, sv_r, sv_z, sv_c, sv_w, sv_rw, flags & 1)
    return nc == 1 ? DGC_FWD_RR(1) : nc == 4 ? DGC_FWD_RR(4) : DGC_FWD_RR(2);
#undef DGC_FWD_RR
  }
  DGC_EVOLVE_DISPATCH(evolve_fwd_kernel, 2, Fl, Hl, T, W0, Sr, Sz, Pc, Qc, Br, Bz, Bc, Wstack,
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
  const int nc = evolve_rr_cols();
  if (Fl == 128 && nc) {
    cudaStream_t st = dgc::as_stream(stream);
#define DGC_BWD_RR(N)                                                                              \
  launch_rr<N, 3>(evolve_bwd_rr_kernel<N>, Hl, st, "evolve_bwd_rr", Hl, T, Sr, Sz, Pc, Qc, sv_r, \
                  sv_z, sv_c, sv_w, dW_direct, dW0, da_r, da_z, da_c, dBr, dBz, dBc, flags & 1)
    return nc == 1 ? DGC_BWD_RR(1) : nc == 4 ? DGC_BWD_RR(4) : DGC_BWD_RR(2);
#undef DGC_BWD_RR
  }
  DGC_EVOLVE_DISPATCH(evolve_bwd_kernel, 3, Fl, Hl, T, Sr, Sz, Pc, Qc, sv_r, sv_z, sv_c, sv_w,
                      dW_direct, dW0, da_r, da_z, da_c, dBr, dBz, dBc, flags & 1);
  DGC_CHECK_LAUNCH("evolve_bwd_kernel");
  return DGC_OK;
}
