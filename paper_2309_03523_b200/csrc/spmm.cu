// K1: batched gather-SpMM of the GCN structure encoder (fp32).
//
// One launch covers every fusion group of a device: rows are laid out in
// fusion-group order, so a fused group is a contiguous row
// segment and the whole device is one batched CSR. Each row is handled by a
// sub-warp of LPR lanes; every lane owns NV float4 columns, so one neighbour
// row is fetched as LPR*NV coalesced 16-byte loads (a 512-byte row at W = 128
// is one fully coalesced warp transaction). Neighbour indices are broadcast
// within the sub-warp and unrolled kUnr deep; the reduction order is the CSR
// order, so the result is bitwise deterministic (no atomics).
//
// The gather is latency-bound on the neighbour rows served by L2, so the
// kernel is held to 32 registers (8 resident 256-thread CTAs = 64 warps per
// SM) and the grid is exactly the resident capacity (a partial second wave
// doubled the time when a variant needed 40 registers). Measured on B200 at
// C2/C3 (tools/time_spmm.py, profiles/r2_summary.md): unroll 2 beats 4 and 8;
// a bf16 gathered operand (half the bytes) was no faster, and TMA tile::gather4
// staging of the neighbour rows in shared memory tops out near 8.9 TB/s of
// 512-B row copies (tools/probes/tma_rate.cu), below this register gather.
//
// Semantics replace the analytic structure-encoder cost of the reference
// (costmodel.py:259-263 via sim.py:339-360,485-486) with real arithmetic:
//   out[i] = act( dinv[i] * sum_{c in row i} dinv[c] * Y[c] + bias ),
// optionally also written as fp16 to out16 (the fused recurrence's x operand).
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

constexpr int kUnr = 2;  // neighbours per batch of loads

template <int LPR, int NV, bool F16>
__global__ void __launch_bounds__(256, NV == 1 ? 8 : 4) spmm_csr_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
    const float* __restrict__ dinv, const float4* __restrict__ Y,
    const float* __restrict__ bias, float4* __restrict__ out, __half* __restrict__ out16,
    const int32_t* __restrict__ rows, int64_t n_rows, int64_t row_begin, int act,
    int32_t* __restrict__ work, float scale16) {
  constexpr int W4 = LPR * NV;  // float4 per row
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  auto process = [&](int64_t i) {
    const int64_t row = rows ? (int64_t)__ldg(rows + i) : row_begin + i;
    const int beg = __ldg(row_ptr + row), end = __ldg(row_ptr + row + 1);
    float4 acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = make_float4(0.f, 0.f, 0.f, 0.f);
    int e = beg;
    for (; e + kUnr <= end; e += kUnr) {
      int c[kUnr];
      float w[kUnr];
#pragma unroll
      for (int u = 0; u < kUnr; ++u) c[u] = __ldg(col + e + u);
#pragma unroll
      for (int u = 0; u < kUnr; ++u) w[u] = __ldg(dinv + c[u]);
      float4 y[kUnr][NV];
#pragma unroll
      for (int u = 0; u < kUnr; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) y[u][v] = __ldg(Y + (int64_t)c[u] * W4 + lane + v * LPR);
#pragma unroll
      for (int u = 0; u < kUnr; ++u)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
          acc[v].x = fmaf(w[u], y[u][v].x, acc[v].x);
          acc[v].y = fmaf(w[u], y[u][v].y, acc[v].y);
          acc[v].z = fmaf(w[u], y[u][v].z, acc[v].z);
          acc[v].w = fmaf(w[u], y[u][v].w, acc[v].w);
        }
    }
    for (; e < end; ++e) {
      const int c = __ldg(col + e);
      const float w = __ldg(dinv + c);
#pragma unroll
      for (int v = 0; v < NV; ++v) {
        const float4 y = __ldg(Y + (int64_t)c * W4 + lane + v * LPR);
        acc[v].x = fmaf(w, y.x, acc[v].x);
        acc[v].y = fmaf(w, y.y, acc[v].y);
        acc[v].z = fmaf(w, y.z, acc[v].z);
        acc[v].w = fmaf(w, y.w, acc[v].w);
      }
    }
    const float di = __ldg(dinv + row);
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      const int j4 = lane + v * LPR;
      float4 b = bias ? __ldg(reinterpret_cast<const float4*>(bias) + j4)
                      : make_float4(0.f, 0.f, 0.f, 0.f);
      float4 o;
      o.x = fmaf(di, acc[v].x, b.x);
      o.y = fmaf(di, acc[v].y, b.y);
      o.z = fmaf(di, acc[v].z, b.z);
      o.w = fmaf(di, acc[v].w, b.w);
      if (act & 1) {
        o.x = fmaxf(o.x, 0.f);
        o.y = fmaxf(o.y, 0.f);
        o.z = fmaxf(o.z, 0.f);
        o.w = fmaxf(o.w, 0.f);
      }
      if (act & 2) {
        o.x = dgc::rna_tf32_f(o.x);
        o.y = dgc::rna_tf32_f(o.y);
        o.z = dgc::rna_tf32_f(o.z);
        o.w = dgc::rna_tf32_f(o.w);
      }
      if (out) out[row * W4 + j4] = o;
      if (F16) {
        const __half2 a = __floats2half2_rn(o.x * scale16, o.y * scale16),
                      h = __floats2half2_rn(o.z * scale16, o.w * scale16);
        reinterpret_cast<uint2*>(out16)[row * W4 + j4] =
            make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&h));
      }
    }
  };
  if (!work) {  // static: grid-stride over the rows
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
    for (int64_t i = tid / LPR; i < n_rows; i += stride) process(i);
    return;
  }
  // dynamic: warps take the next 16 x (32 / LPR) rows from a global counter, so
  // the rows in flight stay one compact window of the (snapshot-major) row
  // order and their neighbour rows stay L2-resident (a grid-stride walk lets
  // the warps drift apart: 29% L2 hits and 2.6x re-read DRAM traffic at C5).
  // The per-row reduction order is unchanged (bitwise the static result).
  constexpr int RPI = 32 / LPR, kIt = 16, kGrab = kIt * RPI;
  const int wl = threadIdx.x & 31, sub = wl / LPR;
  while (true) {
    int base = 0;
    if (wl == 0) base = atomicAdd(work, kGrab);
    base = __shfl_sync(0xffffffffu, base, 0);
    if ((int64_t)base >= n_rows) break;
#pragma unroll 1
    for (int k = 0; k < kIt; ++k) {
      const int64_t i = (int64_t)base + k * RPI + sub;
      if (i < n_rows) process(i);
    }
  }
  // the last CTA out leaves the counter pair zeroed for the next launch
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(work + 1, 1) == (int)gridDim.x - 1) {
      work[0] = 0;
      work[1] = 0;
      __threadfence();
    }
  }
}

// fp16 gathered operand (TF32 mode's resident fp16 features: no fp32 copy and
// no expansion kernel in the input pipeline); lane = 8 halves (16 B), fp32
// accumulation in the same CSR order, rows scheduled as spmm_csr_kernel.
template <int LPR>
__global__ void __launch_bounds__(256, 8) spmm_csr_h_kernel(
    const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
    const float* __restrict__ dinv, const uint4* __restrict__ Y,
    const float* __restrict__ bias, float* __restrict__ out, __half* __restrict__ out16,
    float scale16, int64_t n_rows, int act, int32_t* __restrict__ work) {
  constexpr int W = LPR * 8;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  auto fma8 = [](float w, const uint4& u, float* a) {
    const uint32_t q[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&q[k]));
      a[2 * k] = fmaf(w, f.x, a[2 * k]);
      a[2 * k + 1] = fmaf(w, f.y, a[2 * k + 1]);
    }
  };
  auto process = [&](int64_t row) {
    const int beg = __ldg(row_ptr + row), end = __ldg(row_ptr + row + 1);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int e = beg;
    for (; e + kUnr <= end; e += kUnr) {
      int c[kUnr];
      float w[kUnr];
      uint4 y[kUnr];
#pragma unroll
      for (int u = 0; u < kUnr; ++u) c[u] = __ldg(col + e + u);
#pragma unroll
      for (int u = 0; u < kUnr; ++u) w[u] = __ldg(dinv + c[u]);
#pragma unroll
      for (int u = 0; u < kUnr; ++u) y[u] = __ldg(Y + (int64_t)c[u] * LPR + lane);
#pragma unroll
      for (int u = 0; u < kUnr; ++u) fma8(w[u], y[u], acc);
    }
    for (; e < end; ++e) {
      const int c = __ldg(col + e);
      fma8(__ldg(dinv + c), __ldg(Y + (int64_t)c * LPR + lane), acc);
    }
    const float di = __ldg(dinv + row);
    float o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float v = fmaf(di, acc[k], bias ? __ldg(bias + lane * 8 + k) : 0.f);
      if (act & 1) v = fmaxf(v, 0.f);
      if (act & 2) v = dgc::rna_tf32_f(v);
      o[k] = v;
    }
    if (out) {
      float4* op = reinterpret_cast<float4*>(out + row * W + lane * 8);
      op[0] = make_float4(o[0], o[1], o[2], o[3]);
      op[1] = make_float4(o[4], o[5], o[6], o[7]);
    }
    if (out16) {
      __half2 h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = __floats2half2_rn(o[2 * k] * scale16, o[2 * k + 1] * scale16);
      reinterpret_cast<uint4*>(out16)[row * LPR + lane] = *reinterpret_cast<const uint4*>(h);
    }
  };
  if (!work) {
    const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
    for (int64_t i = tid / LPR; i < n_rows; i += stride) process(i);
    return;
  }
  constexpr int RPI = 32 / LPR, kIt = 16, kGrab = kIt * RPI;
  const int wl = threadIdx.x & 31, sub = wl / LPR;
  while (true) {
    int base = 0;
    if (wl == 0) base = atomicAdd(work, kGrab);
    base = __shfl_sync(0xffffffffu, base, 0);
    if ((int64_t)base >= n_rows) break;
#pragma unroll 1
    for (int k = 0; k < kIt; ++k) {
      const int64_t i = (int64_t)base + k * RPI + sub;
      if (i < n_rows) process(i);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(work + 1, 1) == (int)gridDim.x - 1) {
      work[0] = 0;
      work[1] = 0;
      __threadfence();
    }
  }
}

template <int LPR>
int launch_h(const int32_t* rp, const int32_t* col, const float* dinv, const void* Y,
             const float* bias, float* out, __half* out16, float scale16, int64_t n, int act,
             int32_t* work, cudaStream_t s) {
  static const int resident = [] {
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, spmm_csr_h_kernel<LPR>, 256, 0) !=
            cudaSuccess || b < 1)
      b = 1;
    return b;
  }();
  const int grid = dgc::grid_for(n * LPR, 256, resident);
  const int64_t warps = (int64_t)grid * 8;
  if (n * LPR / 32 < 256 * warps) work = nullptr;  // as spmm_csr_kernel
  spmm_csr_h_kernel<LPR><<<grid, 256, 0, s>>>(rp, col, dinv, static_cast<const uint4*>(Y), bias,
                                               out, out16, scale16, n, act, work);
  DGC_CHECK_LAUNCH("spmm_csr_h_kernel");
  return DGC_OK;
}

template <int LPR, int NV, bool F16>
int launch(const int32_t* rp, const int32_t* col, const float* dinv, const float* Y,
           const float* bias, float* out, __half* out16, const int32_t* rows, int64_t n,
           int64_t row_begin, int act, int32_t* work, float scale16, cudaStream_t s) {
  const int block = 256;
  static const int resident = [] {  // CTAs per SM at this instantiation's register count
    int b = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, spmm_csr_kernel<LPR, NV, F16>, 256, 0) !=
            cudaSuccess || b < 1)
      b = 1;
    return b;
  }();
  const int grid = dgc::grid_for(n * LPR, block, resident);
  // dynamic row scheduling pays only when every warp has many rows to walk
  // (C5: 1056 rows per warp, 6.2 -> 3.9 ms); on smaller graphs the grid-stride
  // walk keeps its neighbour rows L2-resident anyway and the counter's atomics
  // and the coarser tail cost more (C2 82 -> 125+ us, C3 330 -> 405+ us)
  const int64_t warps = (int64_t)grid * (block / 32);
  if (n * LPR / 32 < 256 * warps) work = nullptr;
  spmm_csr_kernel<LPR, NV, F16><<<grid, block, 0, s>>>(
      rp, col, dinv, reinterpret_cast<const float4*>(Y), bias, reinterpret_cast<float4*>(out),
      out16, rows, n, row_begin, act, work, scale16);
  DGC_CHECK_LAUNCH("spmm_csr_kernel");
  return DGC_OK;
}

template <int LPR, int NV>
int launch_f(const int32_t* rp, const int32_t* col, const float* dinv, const float* Y,
             const float* bias, float* out, __half* out16, const int32_t* rows, int64_t n,
             int64_t row_begin, int act, int32_t* work, float scale16, cudaStream_t s) {
  return out16 ? launch<LPR, NV, true>(rp, col, dinv, Y, bias, out, out16, rows, n, row_begin, act, work,
                                       scale16, s)
               : launch<LPR, NV, false>(rp, col, dinv, Y, bias, out, nullptr, rows, n, row_begin, act, work,
                                        1.f, s);
}

}  // namespace

extern "C" int dgc_spmm_csr_x(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                              const float* Y, const float* bias, float* out, void* out16,
                              const int32_t* rows, int64_t n_rows, int64_t row_begin,
                              int32_t width, int32_t act, int32_t* work, float scale16,
                              void* stream) {
  DGC_REQUIRE(n_rows < (int64_t)INT32_MAX - 4096, "spmm: too many rows for the work counter");
  if (n_rows == 0) return DGC_OK;  // (an empty output tensor has a null data pointer)
  DGC_REQUIRE(out || out16, "spmm: no output");
  DGC_REQUIRE(width > 0 && width % 4 == 0, "spmm: width must be a positive multiple of 4");
  if (n_rows == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  __half* o16 = static_cast<__half*>(out16);
#define DGC_SPMM_L(LPR, NV) \
  launch_f<LPR, NV>(row_ptr, col, dinv, Y, bias, out, o16, rows, n_rows, row_begin, act, work, scale16, s)
  switch (width) {
    case 4: return DGC_SPMM_L(1, 1);
    case 8: return DGC_SPMM_L(2, 1);
    case 16: return DGC_SPMM_L(4, 1);
    case 32: return DGC_SPMM_L(8, 1);
    case 64: return DGC_SPMM_L(16, 1);
    case 128: return DGC_SPMM_L(32, 1);
    case 256: return DGC_SPMM_L(32, 2);
    case 512: return DGC_SPMM_L(32, 4);
    default: return dgc::fail(DGC_ERR_ARG, "spmm: unsupported width (use 4..512, power of two)");
  }
#undef DGC_SPMM_L
}

extern "C" int dgc_spmm_csr_rows(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                                 const float* Y, const float* bias, float* out,
                                 const int32_t* rows, int64_t n_rows, int64_t row_begin,
                                 int32_t width, int32_t act, void* stream) {
  return dgc_spmm_csr_x(row_ptr, col, dinv, Y, bias, out, nullptr, rows, n_rows, row_begin, width,
                        act, nullptr, 1.f, stream);
}

extern "C" int dgc_spmm_csr(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                            const float* Y, const float* bias, float* out, int64_t n_rows,
                            int32_t width, int32_t act, void* stream) {
  return dgc_spmm_csr_x(row_ptr, col, dinv, Y, bias, out, nullptr, nullptr, n_rows, 0, width, act,
                        nullptr, 1.f, stream);
}

extern "C" int dgc_spmm_csr_h(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                              const void* Y16, const float* bias, float* out, void* out16,
                              float scale16, int64_t n_rows, int32_t width, int32_t act,
                              int32_t* work, void* stream) {
  DGC_REQUIRE(n_rows < (int64_t)INT32_MAX - 4096, "spmm_h: too many rows for the work counter");
  if (n_rows == 0) return DGC_OK;  // (an empty output tensor has a null data pointer)
  DGC_REQUIRE(out || out16, "spmm_h: no output");
  __half* o16 = static_cast<__half*>(out16);
  if (n_rows == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  switch (width) {
    case 32: return launch_h<4>(row_ptr, col, dinv, Y16, bias, out, o16, scale16, n_rows, act, work, s);
    case 64: return launch_h<8>(row_ptr, col, dinv, Y16, bias, out, o16, scale16, n_rows, act, work, s);
    case 128: return launch_h<16>(row_ptr, col, dinv, Y16, bias, out, o16, scale16, n_rows, act, work, s);
    case 256: return launch_h<32>(row_ptr, col, dinv, Y16, bias, out, o16, scale16, n_rows, act, work, s);
    default: return dgc::fail(DGC_ERR_ARG, "spmm_h: width must be 32, 64, 128 or 256");
  }
}
