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
#include "common.cuh"

namespace {

__device__ __forceinline__ float sgm(float x) { return 1.f / (1.f + __expf(-x)); }
constexpr int CB = 2;  // columns per CTA

__global__ void __launch_bounds__(256) evolve_fwd_kernel(
    int Fl, int Hl, int T, const float* __restrict__ W0, const float* __restrict__ SrT,
    const float* __restrict__ SzT, const float* __restrict__ PcT, const float* __restrict__ QcT,
    const float* __restrict__ Br, const float* __restrict__ Bz, const float* __restrict__ Bc,
    float* __restrict__ Wstack, float* __restrict__ sv_r, float* __restrict__ sv_z,
    float* __restrict__ sv_c, float* __restrict__ sv_w, float* __restrict__ sv_rw, int rnd) {
  extern __shared__ float sm[];
  float* w_s = sm;             // [CB][Fl]
  float* rw_s = sm + CB * Fl;  // [CB][Fl]
  const int i = threadIdx.x, jj = threadIdx.y;
  const int j = blockIdx.x * CB + jj;
  const bool ok = j < Hl;
  float w = ok ? W0[(int64_t)i * Hl + j] : 0.f;
  w_s[jj * Fl + i] = w;
  if (ok) Wstack[(int64_t)i * Hl + j] = rnd ? dgc::rna_tf32_f(w) : w;
  const float br = ok ? Br[(int64_t)i * Hl + j] : 0.f, bz = ok ? Bz[(int64_t)i * Hl + j] : 0.f,
              bc = ok ? Bc[(int64_t)i * Hl + j] : 0.f;
  __syncthreads();
  for (int t = 0; t < T; ++t) {
    float ar = br, az = bz, ap = bc;
    for (int k = 0; k < Fl; ++k) {
      const float wk = w_s[jj * Fl + k];
      ar = fmaf(__ldg(SrT + (int64_t)k * Fl + i), wk, ar);
      az = fmaf(__ldg(SzT + (int64_t)k * Fl + i), wk, az);
      ap = fmaf(__ldg(PcT + (int64_t)k * Fl + i), wk, ap);
    }
    const float r = sgm(ar), z = sgm(az);
    rw_s[jj * Fl + i] = r * w;
    __syncthreads();
    float aq = ap;
    for (int k = 0; k < Fl; ++k) aq = fmaf(__ldg(QcT + (int64_t)k * Fl + i), rw_s[jj * Fl + k], aq);
    const float c = tanhf(aq);
    const float wn = (1.f - z) * c + z * w;
    if (ok) {
      const int64_t sidx = ((int64_t)i * T + t) * Hl + j;  // [Fl][T][Hl]
      sv_r[sidx] = r;
      sv_z[sidx] = z;
      sv_c[sidx] = c;
      sv_w[sidx] = rnd ? dgc::rna_tf32_f(w) : w;
      sv_rw[sidx] = rnd ? dgc::rna_tf32_f(r * w) : r * w;
      Wstack[((int64_t)(t + 1) * Fl + i) * Hl + j] = rnd ? dgc::rna_tf32_f(wn) : wn;
    }
    w = wn;
    __syncthreads();
    w_s[jj * Fl + i] = w;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(256) evolve_bwd_kernel(
    int Fl, int Hl, int T, const float* __restrict__ Sr, const float* __restrict__ Sz,
    const float* __restrict__ Pc, const float* __restrict__ Qc, const float* __restrict__ sv_r,
    const float* __restrict__ sv_z, const float* __restrict__ sv_c, const float* __restrict__ sv_w,
    const float* __restrict__ dW_direct, float* __restrict__ dW0, float* __restrict__ da_r,
    float* __restrict__ da_z, float* __restrict__ da_c, float* __restrict__ dBr,
    float* __restrict__ dBz, float* __restrict__ dBc, int rnd) {
  extern __shared__ float sm[];
  float* dac_s = sm;               // [CB][Fl]
  float* dar_s = sm + CB * Fl;
  float* daz_s = sm + 2 * CB * Fl;
  const int i = threadIdx.x, jj = threadIdx.y;
  const int j = blockIdx.x * CB + jj;
  const bool ok = j < Hl;
  float carry = 0.f, sbr = 0.f, sbz = 0.f, sbc = 0.f;
  for (int t = T - 1; t >= 0; --t) {
    const int64_t sidx = ((int64_t)i * T + t) * Hl + j;
    float g = carry, r = 0.f, z = 0.f, c = 0.f, w = 0.f;
    if (ok) {
      g += dW_direct[((int64_t)t * Fl + i) * Hl + j];  // grad wrt W_{t+1} (snapshot t+1)
      r = sv_r[sidx];
      z = sv_z[sidx];
      c = sv_c[sidx];
      w = sv_w[sidx];
    }
    const float dz = g * (w - c);
    const float dc = g * (1.f - z);
    float dw = g * z;
    const float dac = dc * (1.f - c * c);
    dac_s[jj * Fl + i] = dac;
    __syncthreads();
    float drw = 0.f, dpc = 0.f;
    for (int k = 0; k < Fl; ++k) {
      const float a = dac_s[jj * Fl + k];
      drw = fmaf(__ldg(Qc + (int64_t)k * Fl + i), a, drw);
      dpc = fmaf(__ldg(Pc + (int64_t)k * Fl + i), a, dpc);
    }
    const float dr = drw * w;
    dw = fmaf(drw, r, dw) + dpc;
    const float dar = dr * r * (1.f - r);
    const float daz = dz * z * (1.f - z);
    dar_s[jj * Fl + i] = dar;
    daz_s[jj * Fl + i] = daz;
    __syncthreads();
    for (int k = 0; k < Fl; ++k)
      dw = fmaf(__ldg(Sr + (int64_t)k * Fl + i), dar_s[jj * Fl + k],
                fmaf(__ldg(Sz + (int64_t)k * Fl + i), daz_s[jj * Fl + k], dw));
    if (ok) {
      da_r[sidx] = rnd ? dgc::rna_tf32_f(dar) : dar;
      da_z[sidx] = rnd ? dgc::rna_tf32_f(daz) : daz;
      da_c[sidx] = rnd ? dgc::rna_tf32_f(dac) : dac;
    }
    sbr += dar;
    sbz += daz;
    sbc += dac;
    carry = dw;
    __syncthreads();
  }
  if (ok) {
    dW0[(int64_t)i * Hl + j] = carry;
    dBr[(int64_t)i * Hl + j] = sbr;
    dBz[(int64_t)i * Hl + j] = sbz;
    dBc[(int64_t)i * Hl + j] = sbc;
  }
}

}  // namespace

extern "C" int dgc_evolve_fwd(int32_t Fl, int32_t Hl, int32_t T, const float* W0, const float* SrT,
                              const float* SzT, const float* PcT, const float* QcT,
                              const float* Br, const float* Bz, const float* Bc, float* Wstack,
                              float* sv_r, float* sv_z, float* sv_c, float* sv_w, float* sv_rw,
                              int32_t flags, void* stream) {
  DGC_REQUIRE(Fl >= 1 && Fl * CB <= 1024 && Hl >= 1, "evolve_fwd: bad shape");
  dim3 block(Fl, CB), grid((Hl + CB - 1) / CB);
  evolve_fwd_kernel<<<grid, block, 2 * CB * Fl * sizeof(float), dgc::as_stream(stream)>>>(
      Fl, Hl, T, W0, SrT, SzT, PcT, QcT, Br, Bz, Bc, Wstack, sv_r, sv_z, sv_c, sv_w, sv_rw,
      flags & 1);
  DGC_CHECK_LAUNCH("evolve_fwd_kernel");
  return DGC_OK;
}

extern "C" int dgc_evolve_bwd(int32_t Fl, int32_t Hl, int32_t T, const float* Sr, const float* Sz,
                              const float* Pc, const float* Qc, const float* sv_r,
                              const float* sv_z, const float* sv_c, const float* sv_w,
                              const float* dW_direct, float* dW0, float* da_r, float* da_z,
                              float* da_c, float* dBr, float* dBz, float* dBc, int32_t flags,
                              void* stream) {
  DGC_REQUIRE(Fl >= 1 && Fl * CB <= 1024 && Hl >= 1, "evolve_bwd: bad shape");
  dim3 block(Fl, CB), grid((Hl + CB - 1) / CB);
  evolve_bwd_kernel<<<grid, block, 3 * CB * Fl * sizeof(float), dgc::as_stream(stream)>>>(
      Fl, Hl, T, Sr, Sz, Pc, Qc, sv_r, sv_z, sv_c, sv_w, dW_direct, dW0, da_r, da_z, da_c, dBr,
      dBz, dBc, flags & 1);
  DGC_CHECK_LAUNCH("evolve_bwd_kernel");
  return DGC_OK;
}
