// Probe: TMA issue/throughput rate on B200 for small copies into shared memory.
// Each CTA (one per SM) has NW warps; lane 0..NL-1 of each warp issue copies of
// 512 B (gather4: 4 random rows x 128 B; tile: 4 consecutive rows x 128 B;
// bulk: one contiguous 512 B) into a per-warp ring of S stages (each stage =
// NL copies), waiting on the stage barrier before reuse. Reports GB/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_bar(uint64_t* b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su(b)), "r"(ph) : "memory");
}
constexpr int S = 4, NL = 16, NW = 6;
__global__ void __launch_bounds__(32 * NW, 1) probe(const __grid_constant__ CUtensorMap gmap,
                                                    const __grid_constant__ CUtensorMap tmap,
                                                    const float* src, const int* rows, int n_rows,
                                                    int iters, int mode, float* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (su(sm) & 1023)) & 1023);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* ring = base + w * S * NL * 512;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + NW * S * NL * 512) + w * S;
  if (lane == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t seed = (blockIdx.x * NW + w) * 7919u + lane * 104729u;
  float acc = 0.f;
  for (int k = 0; k < iters; ++k) {
    const int s = k % S;
    if (k >= S) {
      wait_bar(&bar[s], ((k / S) - 1) & 1);
      acc += reinterpret_cast<float*>(ring + s * NL * 512)[lane];
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[s])), "r"(NL * 512) : "memory");
    __syncwarp();
    if (lane < NL) {
      uint8_t* dst = ring + s * NL * 512 + lane * 512;
      seed = seed * 1664525u + 1013904223u;
      const int r = (int)(seed % (uint32_t)(n_rows - 4));
      if (mode == 0) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(dst)), "l"(&gmap), "r"(0),
                     "r"(r), "r"((r + 977) % n_rows), "r"((r + 3001) % n_rows), "r"((r + 50021) % n_rows), "r"(su(&bar[s])) : "memory");
      } else if (mode == 1) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                     " [%0], [%1, {%2, %3}], [%4];" ::"r"(su(dst)), "l"(&tmap), "r"(0), "r"(r), "r"(su(&bar[s])) : "memory");
      } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su(dst)), "l"(src + (size_t)r * 128), "r"(512), "r"(su(&bar[s])) : "memory");
      }
    }
  }
  for (int k = iters; k < iters + S; ++k) wait_bar(&bar[k % S], ((k / S) - 1) & 1);
  if (acc == 12345.f) sink[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 200000;  // rows of 128 floats (512 B)
  float* d; cudaMalloc(&d, (size_t)R * 128 * 4); cudaMemset(d, 0, (size_t)R * 128 * 4);
  float* sink; cudaMalloc(&sink, 4);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  CUtensorMap g, t;
  cuuint64_t dims[2] = {128, (cuuint64_t)R}, str[1] = {512};
  cuuint32_t gbox[2] = {32, 1}, tbox[2] = {32, 4}, es[2] = {1, 1};
  enc(&g, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, gbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&t, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, tbox, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const size_t smem = NW * S * NL * 512 + NW * S * 8 + 1024;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int iters = 2000;
  const char* names[3] = {"gather4 (4 rows x 128B)", "tile 4x128B", "bulk 512B"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      probe<<<148, 32 * NW, smem>>>(g, t, d, nullptr, R, iters, mode, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double bytes = 148.0 * NW * iters * NL * 512;
      if (rep) printf("%-26s R=%d: %.3f ms, %.0f GB/s, %.1f ns per copy per SM\n", names[mode], R, ms,
                      bytes / ms / 1e6, ms * 1e6 / (iters * NW * NL));
    }
  }
  cudaError_t e = cudaGetLastError(); if (e) printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
