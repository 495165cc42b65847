// K3/K4: masked recurrent time encoders over FFD-packed per-device runs.
//
// Forward semantics are those of the reference's only numeric kernel,
// gru_forward_masked (fusion.py:428-469) with GruCell.step (fusion.py:409-413):
//   r = s(x W_r + h U_r + b_r), z = s(x W_z + h U_z + b_z),
//   c = tanh(x W_c + (r*h) U_c + b_c), h' = (1-z) c + z h
// with h <- h * mask[:, p] before every step (fusion.py:459-462). The LSTM uses
// the same conventions (gates i,f,g,o; h and c both carry-masked). Outside the
// reference: a run whose predecessor presence sits on another device starts
// from the carry that device last transmitted (Appendix B.2(a)).
//
// The input projections x W + b of every slot are one tcgen05 GEMM (K2) ahead
// of this kernel; here each CTA owns TR packed rows for the whole sequence and
// walks the L positions persistently, keeping h in shared memory for the
// h·U products (U streamed through L1/L2, reused across the CTA's rows) and c
// in registers. Backward is BPTT over the same packing and writes the
// pre-activation gradients dgx; dWx / dU / db / dx are K2 GEMMs afterwards.
#include "common.cuh"

namespace {

__device__ __forceinline__ float sigm(float x) { return 1.f / (1.f + __expf(-x)); }

// ------------------------------- GRU ----------------------------------------
template <int RPT>
__global__ void __launch_bounds__(256, 3) gru_fwd_kernel(const float* __restrict__ gx, const float* __restrict__ U,
                               const int32_t* __restrict__ slot_row,
                               const uint8_t* __restrict__ slot_mask,
                               const int32_t* __restrict__ slot_carry,
                               const float* __restrict__ carry, int64_t R, int L, int H,
                               int64_t ld, float* __restrict__ h_out, float* __restrict__ save,
                               int rnd) {
  extern __shared__ float sm[];
  const int TY = blockDim.y, TR = TY * RPT;
  float* hs = sm;            // [TR][H]
  float* rhs = sm + TR * H;  // [TR][H]
  const int j = threadIdx.x, ty = threadIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * TR;
  const int G3 = 3 * H;
  float h[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) h[q] = 0.f;
  for (int p = 0; p < L; ++p) {
    int inst[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = ty + TY * q;
      const int64_t row = row0 + lr;
      inst[q] = -1;
      if (row < R) {
        const int64_t s = row * L + p;
        inst[q] = slot_row[s];
        h[q] *= (float)slot_mask[s];
        const int ci = slot_carry[s];
        if (ci >= 0) h[q] = carry[(int64_t)ci * H + j];
      }
      hs[lr * H + j] = h[q];
    }
    __syncthreads();
    float ar[RPT], az[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      ar[q] = inst[q] >= 0 ? gx[(int64_t)inst[q] * G3 + j] : 0.f;
      az[q] = inst[q] >= 0 ? gx[(int64_t)inst[q] * G3 + H + j] : 0.f;
    }
    for (int k = 0; k < H; ++k) {
      const float ur = __ldg(U + (int64_t)k * G3 + j), uz = __ldg(U + (int64_t)k * G3 + H + j);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const float hk = hs[(ty + TY * q) * H + k];
        ar[q] = fmaf(hk, ur, ar[q]);
        az[q] = fmaf(hk, uz, az[q]);
      }
    }
    float r[RPT], z[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      r[q] = sigm(ar[q]);
      z[q] = sigm(az[q]);
      rhs[(ty + TY * q) * H + j] = r[q] * h[q];
    }
    __syncthreads();
    float ac[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) ac[q] = inst[q] >= 0 ? gx[(int64_t)inst[q] * G3 + 2 * H + j] : 0.f;
    for (int k = 0; k < H; ++k) {
      const float uc = __ldg(U + (int64_t)k * G3 + 2 * H + j);
#pragma unroll
      for (int q = 0; q < RPT; ++q) ac[q] = fmaf(rhs[(ty + TY * q) * H + k], uc, ac[q]);
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const float c = tanhf(ac[q]);
      float hn = (1.f - z[q]) * c + z[q] * h[q];
      if (rnd) hn = dgc::rna_tf32_f(hn);
      if (inst[q] >= 0) {
        float* sv = save + (int64_t)inst[q] * 5 * H;
        sv[j] = h[q];
        sv[H + j] = rnd ? dgc::rna_tf32_f(r[q] * h[q]) : r[q] * h[q];
        sv[2 * H + j] = r[q];
        sv[3 * H + j] = z[q];
        sv[4 * H + j] = c;
        h_out[(int64_t)inst[q] * ld + j] = hn;
      }
      h[q] = hn;
    }
    __syncthreads();  // hs / rhs reused next step
  }
}

template <int RPT>
__global__ void __launch_bounds__(256, 3) gru_bwd_kernel(const float* __restrict__ Ut, const int32_t* __restrict__ slot_row,
                               const uint8_t* __restrict__ slot_mask, int64_t R, int L, int H,
                               const float* __restrict__ save, const float* __restrict__ dh_out,
                               float* __restrict__ dgx, int rnd, float* __restrict__ bias_partial) {
  extern __shared__ float sm[];
  const int TY = blockDim.y, TR = TY * RPT;
  float* dar_s = sm;
  float* daz_s = sm + TR * H;
  float* dac_s = sm + 2 * TR * H;
  const int j = threadIdx.x, ty = threadIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * TR;
  const int G3 = 3 * H;
  float bsum[3] = {0.f, 0.f, 0.f};
  float dh[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) dh[q] = 0.f;
  for (int p = L - 1; p >= 0; --p) {
    int inst[RPT];
    float m[RPT], hin[RPT], r[RPT], z[RPT], dhp[RPT], dz[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = ty + TY * q;
      const int64_t row = row0 + lr;
      inst[q] = -1;
      m[q] = 0.f;
      if (row < R) {
        const int64_t s = row * L + p;
        inst[q] = slot_row[s];
        m[q] = (float)slot_mask[s];
      }
      float dac = 0.f;
      hin[q] = r[q] = z[q] = dhp[q] = dz[q] = 0.f;
      if (inst[q] >= 0) {
        const float* sv = save + (int64_t)inst[q] * 5 * H;
        hin[q] = sv[j];
        r[q] = sv[2 * H + j];
        z[q] = sv[3 * H + j];
        const float c = sv[4 * H + j];
        const float g = dh[q] + dh_out[(int64_t)inst[q] * H + j];
        dz[q] = g * (hin[q] - c);
        const float dc = g * (1.f - z[q]);
        dhp[q] = g * z[q];
        dac = dc * (1.f - c * c);
      }
      dac_s[lr * H + j] = dac;
    }
    __syncthreads();
    float drh[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) drh[q] = 0.f;
    for (int k = 0; k < H; ++k) {
      const float u = __ldg(Ut + (int64_t)(2 * H + k) * H + j);  // U_c[j][k]
#pragma unroll
      for (int q = 0; q < RPT; ++q) drh[q] = fmaf(dac_s[(ty + TY * q) * H + k], u, drh[q]);
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = ty + TY * q;
      float dar = 0.f, daz = 0.f;
      if (inst[q] >= 0) {
        dhp[q] = fmaf(drh[q], r[q], dhp[q]);
        const float dr = drh[q] * hin[q];
        dar = dr * r[q] * (1.f - r[q]);
        daz = dz[q] * z[q] * (1.f - z[q]);
        float* o = dgx + (int64_t)inst[q] * G3;
        const float dac = dac_s[lr * H + j];
        o[j] = rnd ? dgc::rna_tf32_f(dar) : dar;
        o[H + j] = rnd ? dgc::rna_tf32_f(daz) : daz;
        o[2 * H + j] = rnd ? dgc::rna_tf32_f(dac) : dac;
        bsum[0] += dar;
        bsum[1] += daz;
        bsum[2] += dac;
      }
      dar_s[lr * H + j] = dar;
      daz_s[lr * H + j] = daz;
    }
    __syncthreads();
    for (int k = 0; k < H; ++k) {
      const float u_r = __ldg(Ut + (int64_t)k * H + j), u_z = __ldg(Ut + (int64_t)(H + k) * H + j);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int lr = ty + TY * q;
        dhp[q] = fmaf(dar_s[lr * H + k], u_r, fmaf(daz_s[lr * H + k], u_z, dhp[q]));
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) dh[q] = inst[q] >= 0 ? dhp[q] * m[q] : 0.f;
    __syncthreads();
  }
  if (bias_partial) {  // per-CTA column sums of dgx, combined over ty in fixed order
    for (int gi = 0; gi < 3; ++gi) {
      dar_s[ty * H + j] = bsum[gi];
      __syncthreads();
      if (ty == 0) {
        float acc = 0.f;
        for (int t = 0; t < TY; ++t) acc += dar_s[t * H + j];
        bias_partial[(int64_t)blockIdx.x * G3 + gi * H + j] = acc;
      }
      __syncthreads();
    }
  }
}

// ------------------------------- LSTM ---------------------------------------
template <int RPT>
__global__ void __launch_bounds__(256, 3) lstm_fwd_kernel(const float* __restrict__ gx, const float* __restrict__ U,
                                const int32_t* __restrict__ slot_row,
                                const uint8_t* __restrict__ slot_mask,
                                const int32_t* __restrict__ slot_carry,
                                const float* __restrict__ carry, int64_t R, int L, int H,
                                int64_t ld, float* __restrict__ h_out, float* __restrict__ c_out,
                                float* __restrict__ save, int rnd) {
  extern __shared__ float sm[];
  const int TY = blockDim.y, TR = TY * RPT;
  float* hs = sm;
  const int j = threadIdx.x, ty = threadIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * TR;
  const int G4 = 4 * H;
  float h[RPT], c[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) h[q] = c[q] = 0.f;
  for (int p = 0; p < L; ++p) {
    int inst[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = ty + TY * q;
      const int64_t row = row0 + lr;
      inst[q] = -1;
      if (row < R) {
        const int64_t s = row * L + p;
        inst[q] = slot_row[s];
        const float mk = (float)slot_mask[s];
        h[q] *= mk;
        c[q] *= mk;
        const int ci = slot_carry[s];
        if (ci >= 0) {
          h[q] = carry[(int64_t)ci * 2 * H + j];
          c[q] = carry[(int64_t)ci * 2 * H + H + j];
        }
      }
      hs[lr * H + j] = h[q];
    }
    __syncthreads();
    float a[4][RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q)
#pragma unroll
      for (int g = 0; g < 4; ++g)
        a[g][q] = inst[q] >= 0 ? gx[(int64_t)inst[q] * G4 + g * H + j] : 0.f;
    for (int k = 0; k < H; ++k) {
      float u[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) u[g] = __ldg(U + (int64_t)k * G4 + g * H + j);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const float hk = hs[(ty + TY * q) * H + k];
#pragma unroll
        for (int g = 0; g < 4; ++g) a[g][q] = fmaf(hk, u[g], a[g][q]);
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const float ig = sigm(a[0][q]), fg = sigm(a[1][q]), gg = tanhf(a[2][q]), og = sigm(a[3][q]);
      const float cn = fg * c[q] + ig * gg;
      const float tc = tanhf(cn);
      const float hn = rnd ? dgc::rna_tf32_f(og * tc) : og * tc;
      if (inst[q] >= 0) {
        float* sv = save + (int64_t)inst[q] * 7 * H;
        sv[j] = h[q];
        sv[H + j] = c[q];
        sv[2 * H + j] = ig;
        sv[3 * H + j] = fg;
        sv[4 * H + j] = gg;
        sv[5 * H + j] = og;
        sv[6 * H + j] = tc;
        h_out[(int64_t)inst[q] * ld + j] = hn;
        if (c_out) c_out[(int64_t)inst[q] * ld + j] = cn;
      }
      h[q] = hn;
      c[q] = cn;
    }
    __syncthreads();
  }
}

template <int RPT>
__global__ void __launch_bounds__(256, 3) lstm_bwd_kernel(const float* __restrict__ Ut, const int32_t* __restrict__ slot_row,
                                const uint8_t* __restrict__ slot_mask, int64_t R, int L, int H,
                                const float* __restrict__ save, const float* __restrict__ dh_out,
                                float* __restrict__ dgx, int rnd, float* __restrict__ bias_partial) {
  extern __shared__ float sm[];
  const int TY = blockDim.y, TR = TY * RPT;
  float* da_s = sm;  // [TR][4][H]
  const int j = threadIdx.x, ty = threadIdx.y;
  const int64_t row0 = (int64_t)blockIdx.x * TR;
  const int G4 = 4 * H;
  float bsum[4] = {0.f, 0.f, 0.f, 0.f};
  float dh[RPT], dc[RPT];
#pragma unroll
  for (int q = 0; q < RPT; ++q) dh[q] = dc[q] = 0.f;
  for (int p = L - 1; p >= 0; --p) {
    int inst[RPT];
    float m[RPT], dcp[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      const int lr = ty + TY * q;
      const int64_t row = row0 + lr;
      inst[q] = -1;
      m[q] = 0.f;
      if (row < R) {
        const int64_t s = row * L + p;
        inst[q] = slot_row[s];
        m[q] = (float)slot_mask[s];
      }
      float da[4] = {0.f, 0.f, 0.f, 0.f};
      dcp[q] = 0.f;
      if (inst[q] >= 0) {
        const float* sv = save + (int64_t)inst[q] * 7 * H;
        const float c_in = sv[H + j], ig = sv[2 * H + j], fg = sv[3 * H + j], gg = sv[4 * H + j],
                    og = sv[5 * H + j], tc = sv[6 * H + j];
        const float g = dh[q] + dh_out[(int64_t)inst[q] * H + j];
        const float d_o = g * tc;
        const float dcn = dc[q] + g * og * (1.f - tc * tc);
        da[0] = dcn * gg * ig * (1.f - ig);
        da[1] = dcn * c_in * fg * (1.f - fg);
        da[2] = dcn * ig * (1.f - gg * gg);
        da[3] = d_o * og * (1.f - og);
        dcp[q] = dcn * fg;
        float* o = dgx + (int64_t)inst[q] * G4;
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          o[gi * H + j] = rnd ? dgc::rna_tf32_f(da[gi]) : da[gi];
          bsum[gi] += da[gi];
        }
      }
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) da_s[(lr * 4 + gi) * H + j] = da[gi];
    }
    __syncthreads();
    float dhp[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) dhp[q] = 0.f;
    for (int k = 0; k < H; ++k) {
      float u[4];
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) u[gi] = __ldg(Ut + (int64_t)(gi * H + k) * H + j);
#pragma unroll
      for (int q = 0; q < RPT; ++q) {
        const int lr = ty + TY * q;
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) dhp[q] = fmaf(da_s[(lr * 4 + gi) * H + k], u[gi], dhp[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
      dh[q] = inst[q] >= 0 ? dhp[q] * m[q] : 0.f;
      dc[q] = inst[q] >= 0 ? dcp[q] * m[q] : 0.f;
    }
    __syncthreads();
  }
  if (bias_partial) {  // per-CTA column sums of dgx, combined over ty in fixed order
    for (int gi = 0; gi < 4; ++gi) {
      da_s[ty * H + j] = bsum[gi];
      __syncthreads();
      if (ty == 0) {
        float acc = 0.f;
        for (int t = 0; t < TY; ++t) acc += da_s[t * H + j];
        bias_partial[(int64_t)blockIdx.x * G4 + gi * H + j] = acc;
      }
      __syncthreads();
    }
  }
}

__global__ void transpose_kernel(const float* __restrict__ in, int64_t rows, int64_t cols,
                                 float* __restrict__ out) {
  __shared__ float tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][i];
  }
}

#ifndef RPT_SEL
#define RPT_SEL 4
#endif
struct Shape {
  int ty, rpt;
};
inline Shape pick_shape(int H) {
  // ~256 threads per CTA; rows per CTA = ty * rpt
  const int ty = H >= 256 ? 1 : 256 / H;
  return {ty < 1 ? 1 : ty, RPT_SEL};
}

}  // namespace

extern "C" int dgc_rnn_save_floats(int32_t cell, int32_t H) { return (cell == 0 ? 5 : 7) * H; }

extern "C" int64_t dgc_rnn_bwd_partial_rows(int64_t n_rows, int32_t H) {
  const Shape sh = pick_shape(H);
  const int64_t TR = (int64_t)sh.ty * sh.rpt;
  return (n_rows + TR - 1) / TR;
}

extern "C" int dgc_transpose(const float* in, int64_t rows, int64_t cols, float* out, void* stream) {
  if (rows == 0 || cols == 0) return DGC_OK;
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, dgc::as_stream(stream)>>>(in, rows, cols, out);
  DGC_CHECK_LAUNCH("transpose_kernel");
  return DGC_OK;
}

extern "C" int dgc_rnn_fwd(int32_t cell_flags, const float* gx, const float* U, const int32_t* slot_row,
                           const uint8_t* slot_mask, const int32_t* slot_carry, const float* carry,
                           int64_t n_rows, int32_t row_len, int32_t H, int64_t ld_out,
                           float* h_out, float* c_out, float* save, void* stream) {
  const int cell = cell_flags & 0xff, rnd = (cell_flags >> 8) & 1;
  DGC_REQUIRE(cell == 0 || cell == 1, "rnn_fwd: cell must be 0 (GRU) or 1 (LSTM)");
  DGC_REQUIRE(H >= 1 && H <= 1024, "rnn_fwd: H out of range");
  if (n_rows == 0 || row_len == 0) return DGC_OK;
  const Shape sh = pick_shape(H);
  const int TR = sh.ty * sh.rpt;
  dim3 block(H, sh.ty), grid((unsigned)((n_rows + TR - 1) / TR));
  cudaStream_t s = dgc::as_stream(stream);
  if (cell == 0) {
    const size_t smem = 2 * (size_t)TR * H * sizeof(float);
    gru_fwd_kernel<RPT_SEL><<<grid, block, smem, s>>>(gx, U, slot_row, slot_mask, slot_carry, carry,
                                                n_rows, row_len, H, ld_out, h_out, save, rnd);
    DGC_CHECK_LAUNCH("gru_fwd_kernel");
  } else {
    const size_t smem = (size_t)TR * H * sizeof(float);
    lstm_fwd_kernel<RPT_SEL><<<grid, block, smem, s>>>(gx, U, slot_row, slot_mask, slot_carry, carry,
                                                 n_rows, row_len, H, ld_out, h_out, c_out, save, rnd);
    DGC_CHECK_LAUNCH("lstm_fwd_kernel");
  }
  return DGC_OK;
}

extern "C" int dgc_rnn_bwd(int32_t cell_flags, const float* Ut, const int32_t* slot_row,
                           const uint8_t* slot_mask, int64_t n_rows, int32_t row_len, int32_t H,
                           const float* save, const float* dh_out, float* dgx,
                           float* bias_partial, void* stream) {
  const int cell = cell_flags & 0xff, rnd = (cell_flags >> 8) & 1;
  DGC_REQUIRE(cell == 0 || cell == 1, "rnn_bwd: cell must be 0 (GRU) or 1 (LSTM)");
  if (n_rows == 0 || row_len == 0) return DGC_OK;
  const Shape sh = pick_shape(H);
  const int TR = sh.ty * sh.rpt;
  dim3 block(H, sh.ty), grid((unsigned)((n_rows + TR - 1) / TR));
  cudaStream_t s = dgc::as_stream(stream);
  if (cell == 0) {
    const size_t smem = 3 * (size_t)TR * H * sizeof(float);
    if (smem > 48 * 1024) {
      cudaFuncSetAttribute(gru_bwd_kernel<RPT_SEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    gru_bwd_kernel<RPT_SEL><<<grid, block, smem, s>>>(Ut, slot_row, slot_mask, n_rows, row_len, H, save,
                                                dh_out, dgx, rnd, bias_partial);
    DGC_CHECK_LAUNCH("gru_bwd_kernel");
  } else {
    const size_t smem = 4 * (size_t)TR * H * sizeof(float);
    if (smem > 48 * 1024) {
      cudaFuncSetAttribute(lstm_bwd_kernel<RPT_SEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    }
    lstm_bwd_kernel<RPT_SEL><<<grid, block, smem, s>>>(Ut, slot_row, slot_mask, n_rows, row_len, H, save,
                                                 dh_out, dgx, rnd, bias_partial);
    DGC_CHECK_LAUNCH("lstm_bwd_kernel");
  }
  return DGC_OK;
}
