// K5: adaptive stale aggregation filter on the GPU.
//
// Restates stale.py:140-176 (filter_transmissions) and stale.py:205-212
// (max_cache_gap) for a device-resident cache: the cache holds the
// LAST-TRANSMITTED copy of every boundary key (stale.py:111-130), so the
// comparison basis is never the previous epoch (bounded staleness). The
// distance is fp32 with a fixed per-key reduction order (lane-ordered float4
// partials combined by a fixed xor tree), the maximum via an order-free
// integer atomicMax on non-negative floats -- both deterministic. The global
// D_r of one cache is the MAX all-reduce of dmax over ranks (sim.py:455-459
// uses one global cache); theta comes from threshold() on the host.
#include "common.cuh"

namespace {

template <int LPR>
__global__ void stale_distance_kernel(const float* __restrict__ Y, const int32_t* __restrict__ keys,
                                      const float* __restrict__ cache,
                                      const uint8_t* __restrict__ cached, int64_t n_keys, int width,
                                      float* __restrict__ dist, unsigned int* __restrict__ dmax) {
  // 32/LPR keys per warp and iteration; the loop bound is warp-uniform (every
  // lane of the warp runs every iteration, so the full-mask shuffles below are
  // always converged), keys past n_keys contribute acc = 0 and store nothing
  constexpr int KPW = 32 / LPR;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int lane = (int)(threadIdx.x & 31) % LPR;
  const int sub = (int)(threadIdx.x & 31) / LPR;
  const int w4 = width / 4;
  unsigned int local_max = 0u;
  for (int64_t base = warp * KPW; base < n_keys; base += nwarps * KPW) {
    const int64_t k = base + sub;
    const bool valid = k < n_keys;
    float acc = 0.f;
    if (valid) {
      const float4* y = reinterpret_cast<const float4*>(Y + (int64_t)__ldg(keys + k) * width);
      const float4* c = reinterpret_cast<const float4*>(cache + k * width);
      for (int j = lane; j < w4; j += LPR) {
        const float4 a = __ldg(y + j), b = __ldg(c + j);
        const float dx = a.x - b.x, dy = a.y - b.y, dz = a.z - b.z, dw = a.w - b.w;
        acc = fmaf(dx, dx, acc);
        acc = fmaf(dy, dy, acc);
        acc = fmaf(dz, dz, acc);
        acc = fmaf(dw, dw, acc);
      }
    }
#pragma unroll
    for (int off = LPR / 2; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    const float d = sqrtf(acc);
    if (valid && lane == 0) {
      dist[k] = d;
      if (cached[k]) local_max = max(local_max, __float_as_uint(d));
    }
  }
  // warp max then one atomic per warp (non-negative floats order like uints)
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
    local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, off));
  if ((threadIdx.x & 31) == 0 && local_max) atomicMax(dmax, local_max);
}

__global__ void stale_select_kernel(const float* __restrict__ Y, const int32_t* __restrict__ keys,
                                    const float* __restrict__ dist, double theta_host,
                                    const float* __restrict__ dmax, double coef,
                                    float* __restrict__ cache, uint8_t* __restrict__ cached,
                                    uint8_t* __restrict__ send, int64_t n_keys, int width,
                                    const int64_t* __restrict__ ncut,
                                    unsigned long long* __restrict__ billed) {
  // theta = coef * D_r (threshold(), stale.py:97-108: every mode is D_r times a
  // factor known on the host at the start of the epoch) with D_r read from
  // device memory (the MAX all-reduce result): no host round trip. The
  // comparison is in fp64 like the reference's (stale.py:169, strict >).
  const double theta = dmax ? coef * (double)*dmax : theta_host;
  // one warp per key: decision by lane 0, broadcast, then a coalesced copy
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long bill = 0;
  for (int64_t k = warp; k < n_keys; k += nwarps) {
    const bool s = (theta < 0.0) || !cached[k] || ((double)dist[k] > theta);
    if (lane == 0) {
      send[k] = s ? 1 : 0;
      if (s) cached[k] = 1;
      if (s && ncut) bill += (unsigned long long)ncut[k];
    }
    if (s) {
      const float* y = Y + (int64_t)keys[k] * width;
      float* c = cache + k * width;
      for (int j = lane; j < width; j += 32) c[j] = y[j];
    }
  }
  // reference-billed messages of the sent keys (integer atomics: exact)
  if (billed && lane == 0 && bill) atomicAdd(billed, bill);
}

}  // namespace

extern "C" int dgc_stale_distance(const float* Y, const int32_t* key_rows, const float* cache,
                                  const uint8_t* cached, int64_t n_keys, int32_t width,
                                  float* dist, float* dmax, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "stale_distance: width must be a multiple of 4");
  cudaStream_t s = dgc::as_stream(stream);
  cudaError_t e = cudaMemsetAsync(dmax, 0, sizeof(float), s);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "stale_distance memset");
  if (n_keys == 0) return DGC_OK;
  const int w4 = width / 4;
  const int block = 256;
  auto* dm = reinterpret_cast<unsigned int*>(dmax);
  if (w4 >= 32) {
    stale_distance_kernel<32><<<dgc::grid_for(n_keys * 32, block), block, 0, s>>>(
        Y, key_rows, cache, cached, n_keys, width, dist, dm);
  } else if (w4 >= 8) {
    stale_distance_kernel<8><<<dgc::grid_for(n_keys * 8, block), block, 0, s>>>(
        Y, key_rows, cache, cached, n_keys, width, dist, dm);
  } else {
    stale_distance_kernel<1><<<dgc::grid_for(n_keys, block), block, 0, s>>>(
        Y, key_rows, cache, cached, n_keys, width, dist, dm);
  }
  DGC_CHECK_LAUNCH("stale_distance_kernel");
  return DGC_OK;
}

extern "C" int dgc_stale_select2(const float* Y, const int32_t* key_rows, const float* dist,
                                 double theta, const float* dmax, double coef, float* cache,
                                 uint8_t* cached, uint8_t* send, int64_t n_keys, int32_t width,
                                 const int64_t* ncut, uint64_t* billed, void* stream) {
  if (n_keys == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int block = 256;
  stale_select_kernel<<<dgc::grid_for(n_keys * 32, block), block, 0, s>>>(
      Y, key_rows, dist, theta, dmax, coef, cache, cached, send, n_keys, width, ncut,
      reinterpret_cast<unsigned long long*>(billed));
  DGC_CHECK_LAUNCH("stale_select_kernel");
  return DGC_OK;
}

extern "C" int dgc_stale_select(const float* Y, const int32_t* key_rows, const float* dist,
                                float theta, float* cache, uint8_t* cached, uint8_t* send,
                                int64_t n_keys, int32_t width, void* stream) {
  return dgc_stale_select2(Y, key_rows, dist, (double)theta, nullptr, 0.0, cache, cached, send,
                           n_keys, width, nullptr, nullptr, stream);
}
