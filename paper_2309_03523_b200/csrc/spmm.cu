// K1: batched gather-SpMM of the GCN structure encoder.
//
// One launch covers every fusion group of a device: rows are laid out in
// fusion-group order, so a fused group is a contiguous row
// segment and the whole device is one batched CSR. Each row is handled by a
// sub-warp of LPR lanes; every lane owns NV 16-byte vectors of the row, so a
// neighbour row is fetched as LPR*NV coalesced 16-byte loads. Neighbour
// indices are broadcast within the sub-warp and unrolled UNR deep to keep
// enough loads in flight; the reduction order is the CSR order, so the result
// is bitwise deterministic (no atomics).
//
// The gathered operand Y is fp32 (parity mode) or bf16 (TF32 mode: the
// neighbour-row gathers, ~9 per output row and served by L2, are the kernel's
// dominant byte stream; bf16 halves them). Accumulation and the output are fp32.
//
// Semantics replace the analytic structure-encoder cost of the reference
// (costmodel.py:259-263 via sim.py:339-360,485-486) with real arithmetic:
//   out[i] = act( dinv[i] * sum_{c in row i} dinv[c] * Y[c] + bias ).
#include <cuda_bf16.h>

#include "common.cuh"

namespace {

// 16-byte vector of the gathered operand -> EPV fp32 values
template <typename TY> struct Vec;
template <> struct Vec<float> {
  static constexpr int EPV = 4;
  __device__ static void fma(float w, const uint4& u, float* acc) {
    acc[0] = fmaf(w, __uint_as_float(u.x), acc[0]);
    acc[1] = fmaf(w, __uint_as_float(u.y), acc[1]);
    acc[2] = fmaf(w, __uint_as_float(u.z), acc[2]);
    acc[3] = fmaf(w, __uint_as_float(u.w), acc[3]);
  }
};
template <> struct Vec<__nv_bfloat16> {
  static constexpr int EPV = 8;
  __device__ static void fma(float w, const uint4& u, float* acc) {
    const uint32_t a[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      acc[2 * k] = fmaf(w, __uint_as_float(a[k] << 16), acc[2 * k]);
      acc[2 * k + 1] = fmaf(w, __uint_as_float(a[k] & 0xffff0000u), acc[2 * k + 1]);
    }
  }
};

template <typename TY, int LPR, int NV, int UNR>
__global__ void __launch_bounds__(256) spmm_csr_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
    const float* __restrict__ dinv, const uint4* __restrict__ Y,
    const float* __restrict__ bias, float* __restrict__ out, const int32_t* __restrict__ rows,
    int64_t n_rows, int64_t row_begin, int act) {
  constexpr int EPV = Vec<TY>::EPV;
  constexpr int V = LPR * NV;          // 16-byte vectors per Y row
  constexpr int W = V * EPV;           // row width (elements)
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t i = tid / LPR; i < n_rows; i += stride) {
    const int64_t row = rows ? (int64_t)__ldg(rows + i) : row_begin + i;
    const int beg = __ldg(row_ptr + row), end = __ldg(row_ptr + row + 1);
    float acc[NV][EPV];
#pragma unroll
    for (int v = 0; v < NV; ++v)
#pragma unroll
      for (int k = 0; k < EPV; ++k) acc[v][k] = 0.f;
    int e = beg;
    for (; e + UNR <= end; e += UNR) {
      int c[UNR];
      float w[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) c[u] = __ldg(col + e + u);
#pragma unroll
      for (int u = 0; u < UNR; ++u) w[u] = __ldg(dinv + c[u]);
      uint4 y[UNR][NV];
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) y[u][v] = __ldg(Y + (int64_t)c[u] * V + lane + v * LPR);
#pragma unroll
      for (int u = 0; u < UNR; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) Vec<TY>::fma(w[u], y[u][v], acc[v]);
    }
    for (; e < end; ++e) {
      const int c = __ldg(col + e);
      const float w = __ldg(dinv + c);
#pragma unroll
      for (int v = 0; v < NV; ++v) Vec<TY>::fma(w, __ldg(Y + (int64_t)c * V + lane + v * LPR), acc[v]);
    }
    const float di = __ldg(dinv + row);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int j0 = (lane + v * LPR) * EPV;
#pragma unroll
      for (int k = 0; k < EPV; k += 4) {
        float4 b = bias ? __ldg(reinterpret_cast<const float4*>(bias + j0 + k))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        float o[4] = {fmaf(di, acc[v][k], b.x), fmaf(di, acc[v][k + 1], b.y),
                      fmaf(di, acc[v][k + 2], b.z), fmaf(di, acc[v][k + 3], b.w)};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (act & 1) o[q] = fmaxf(o[q], 0.f);
          if (act & 2) o[q] = dgc::rna_tf32_f(o[q]);
        }
        *reinterpret_cast<float4*>(out + row * W + j0 + k) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

template <typename TY, int LPR, int NV, int UNR>
int launch(const int32_t* rp, const int32_t* col, const float* dinv, const void* Y,
           const float* bias, float* out, const int32_t* rows, int64_t n, int64_t row_begin,
           int act, cudaStream_t s) {
  const int block = 256;
  const int grid = dgc::grid_for(n * LPR, block, 8);
  spmm_csr_kernel<TY, LPR, NV, UNR><<<grid, block, 0, s>>>(
      rp, col, dinv, reinterpret_cast<const uint4*>(Y), bias, out, rows, n, row_begin, act);
  DGC_CHECK_LAUNCH("spmm_csr_kernel");
  return DGC_OK;
}

// neighbours per batch of loads (DGC_SPMM_UNR = 2 | 4 | 8; measured on B200 at
// C2/C3: 2 is fastest, tools/time_spmm.py)
int unroll_depth() {
  static const int u = [] {
    const char* e = getenv("DGC_SPMM_UNR");
    return e ? atoi(e) : 2;
  }();
  return u;
}

template <typename TY, int LPR, int NV>
int launch_u(const int32_t* rp, const int32_t* col, const float* dinv, const void* Y,
             const float* bias, float* out, const int32_t* rows, int64_t n, int64_t row_begin,
             int act, cudaStream_t s) {
  switch (unroll_depth()) {
    case 2: return launch<TY, LPR, NV, 2>(rp, col, dinv, Y, bias, out, rows, n, row_begin, act, s);
    case 8: return launch<TY, LPR, NV, 8>(rp, col, dinv, Y, bias, out, rows, n, row_begin, act, s);
    default: return launch<TY, LPR, NV, 4>(rp, col, dinv, Y, bias, out, rows, n, row_begin, act, s);
  }
}

}  // namespace

extern "C" int dgc_spmm_csr_ex(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                               const void* Y, int32_t y_dtype, const float* bias, float* out,
                               const int32_t* rows, int64_t n_rows, int64_t row_begin,
                               int32_t width, int32_t act, void* stream) {
  DGC_REQUIRE(width > 0 && width % 4 == 0, "spmm: width must be a positive multiple of 4");
  DGC_REQUIRE(y_dtype == DGC_F32 || y_dtype == DGC_BF16, "spmm: Y must be fp32 or bf16");
  if (n_rows == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
#define DGC_SPMM_L(T, LPR, NV) \
  launch_u<T, LPR, NV>(row_ptr, col, dinv, Y, bias, out, rows, n_rows, row_begin, act, s)
  if (y_dtype == DGC_F32) {
    switch (width) {
      case 4: return DGC_SPMM_L(float, 1, 1);
      case 8: return DGC_SPMM_L(float, 2, 1);
      case 16: return DGC_SPMM_L(float, 4, 1);
      case 32: return DGC_SPMM_L(float, 8, 1);
      case 64: return DGC_SPMM_L(float, 16, 1);
      case 128: return DGC_SPMM_L(float, 32, 1);
      case 256: return DGC_SPMM_L(float, 32, 2);
      case 512: return DGC_SPMM_L(float, 32, 4);
      default: break;
    }
  } else {
    switch (width) {
      case 8: return DGC_SPMM_L(__nv_bfloat16, 1, 1);
      case 16: return DGC_SPMM_L(__nv_bfloat16, 2, 1);
      case 32: return DGC_SPMM_L(__nv_bfloat16, 4, 1);
      case 64: return DGC_SPMM_L(__nv_bfloat16, 8, 1);
      case 128: return DGC_SPMM_L(__nv_bfloat16, 16, 1);
      case 256: return DGC_SPMM_L(__nv_bfloat16, 32, 1);
      case 512: return DGC_SPMM_L(__nv_bfloat16, 32, 2);
      default: break;
    }
  }
#undef DGC_SPMM_L
  return dgc::fail(DGC_ERR_ARG, "spmm: unsupported width (fp32 4..512, bf16 8..512, power of two)");
}

extern "C" int dgc_spmm_csr_rows(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                                 const float* Y, const float* bias, float* out,
                                 const int32_t* rows, int64_t n_rows, int64_t row_begin,
                                 int32_t width, int32_t act, void* stream) {
  return dgc_spmm_csr_ex(row_ptr, col, dinv, Y, DGC_F32, bias, out, rows, n_rows, row_begin, width,
                         act, stream);
}

extern "C" int dgc_spmm_csr(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                            const float* Y, const float* bias, float* out, int64_t n_rows,
                            int32_t width, int32_t act, void* stream) {
  return dgc_spmm_csr_ex(row_ptr, col, dinv, Y, DGC_F32, bias, out, nullptr, n_rows, 0, width, act,
                         stream);
}
