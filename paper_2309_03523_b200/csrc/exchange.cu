// K6: boundary-row exchange pack/unpack for the NCCL all-to-allv.
//
// The reference bills one message per cut edge (sim.py:464-469,514-543); a
// real halo exchange moves each (source row, destination device) once. The
// send list of a peer is the ascending-global-index list of own rows that the
// peer needs (derived from MessageSet.cut_mask, costmodel.py:160-165); the
// stale filter (K5) compacts it to the keys whose decision is "send".
#include "common.cuh"

namespace {

// Order-preserving compaction in one CTA (send lists are <= ~1e5 entries).
__global__ void __launch_bounds__(1024) compact_sent_kernel(const int32_t* __restrict__ pos,
                                                           int64_t n, const uint8_t* __restrict__ send,
                                                           int32_t* __restrict__ out_idx,
                                                           int32_t* __restrict__ count) {
  __shared__ int warp_sums[32];
  __shared__ int base_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int64_t start = 0; start < n; start += blockDim.x) {
    const int64_t i = start + tid;
    const int flag = (i < n && send[pos[i]]) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int prefix = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_sums[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      warp_sums[lane] = incl - v;  // exclusive
      if (lane == 31) warp_sums[31] = incl;  // total in slot 31 after use below
    }
    __syncthreads();
    const int total = warp_sums[31];
    const int excl = (wid == 31) ? (total - __popc(bal)) : warp_sums[wid];
    if (flag) out_idx[base_s + excl + prefix] = (int32_t)i;
    __syncthreads();
    if (tid == 0) base_s += total;
    __syncthreads();
  }
  if (tid == 0) *count = base_s;
}

template <int LPR>
__global__ void gather_rows_kernel(const float4* __restrict__ Y, const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ idx, int64_t n, int w4,
                                   float4* __restrict__ out) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t i = tid / LPR; i < n; i += stride) {
    int64_t r = idx ? idx[i] : i;
    if (rows) r = rows[r];
    for (int j = lane; j < w4; j += LPR) out[i * w4 + j] = __ldg(Y + r * w4 + j);
  }
}

template <int LPR>
__global__ void scatter_rows_kernel(const float4* __restrict__ src, const int32_t* __restrict__ rows,
                                    const int32_t* __restrict__ idx, int64_t n, int w4,
                                    float4* __restrict__ dst, int add) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t i = tid / LPR; i < n; i += stride) {
    int64_t r = idx ? idx[i] : i;
    if (rows) r = rows[r];
    for (int j = lane; j < w4; j += LPR) {
      float4 v = __ldg(src + i * w4 + j);
      if (add) {
        const float4 o = dst[r * w4 + j];
        v.x += o.x;
        v.y += o.y;
        v.z += o.z;
        v.w += o.w;
      }
      dst[r * w4 + j] = v;
    }
  }
}

}  // namespace

extern "C" int dgc_compact_sent(const int32_t* pos, int64_t n, const uint8_t* send,
                                int32_t* out_idx, int32_t* count, void* stream) {
  cudaStream_t s = dgc::as_stream(stream);
  compact_sent_kernel<<<1, 1024, 0, s>>>(pos, n, send, out_idx, count);
  DGC_CHECK_LAUNCH("compact_sent_kernel");
  return DGC_OK;
}

extern "C" int dgc_gather_rows(const float* Y, const int32_t* rows, const int32_t* idx, int64_t n,
                               int32_t width, float* out, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "gather_rows: width must be a multiple of 4");
  if (n == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4, block = 256;
  const auto* y = reinterpret_cast<const float4*>(Y);
  auto* o = reinterpret_cast<float4*>(out);
  if (w4 >= 32) gather_rows_kernel<32><<<dgc::grid_for(n * 32, block), block, 0, s>>>(y, rows, idx, n, w4, o);
  else if (w4 >= 8) gather_rows_kernel<8><<<dgc::grid_for(n * 8, block), block, 0, s>>>(y, rows, idx, n, w4, o);
  else gather_rows_kernel<1><<<dgc::grid_for(n, block), block, 0, s>>>(y, rows, idx, n, w4, o);
  DGC_CHECK_LAUNCH("gather_rows_kernel");
  return DGC_OK;
}

extern "C" int dgc_scatter_rows(const float* src, const int32_t* rows, const int32_t* idx,
                                int64_t n, int32_t width, float* dst, int32_t add, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "scatter_rows: width must be a multiple of 4");
  if (n == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4, block = 256;
  const auto* sp = reinterpret_cast<const float4*>(src);
  auto* d = reinterpret_cast<float4*>(dst);
  if (w4 >= 32) scatter_rows_kernel<32><<<dgc::grid_for(n * 32, block), block, 0, s>>>(sp, rows, idx, n, w4, d, add);
  else if (w4 >= 8) scatter_rows_kernel<8><<<dgc::grid_for(n * 8, block), block, 0, s>>>(sp, rows, idx, n, w4, d, add);
  else scatter_rows_kernel<1><<<dgc::grid_for(n, block), block, 0, s>>>(sp, rows, idx, n, w4, d, add);
  DGC_CHECK_LAUNCH("scatter_rows_kernel");
  return DGC_OK;
}
