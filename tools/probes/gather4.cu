// Probe: TMA tile::gather4 of 4 arbitrary rows x 32 fp32 columns into a
// SWIZZLE_128B shared-memory box (the A-operand layout of the tcgen05 kernels).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, const int* rows, int col0, float* out) {
  __shared__ __align__(1024) float tile[8 * 32];  // 8 rows x 128 B (one SW128 atom)
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(2 * 4 * 128) : "memory");
    for (int h = 0; h < 2; ++h)  // two gathers: rows 0-3 and 4-7 of the atom
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(tile + h * 4 * 32)),
          "l"(&map), "r"(col0), "r"(rows[4 * h]), "r"(rows[4 * h + 1]), "r"(rows[4 * h + 2]),
          "r"(rows[4 * h + 3]), "r"(smem_u32(&bar))
          : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) out[i] = tile[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

int main() {
  const int R = 1000, C = 128;
  std::vector<float> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = r * 1000 + c;
  float *d, *o; int* dr;
  cudaMalloc(&d, R * C * 4); cudaMalloc(&o, 8 * 32 * 4); cudaMalloc(&dr, 8 * 4);
  cudaMemcpy(d, h.data(), R * C * 4, cudaMemcpyHostToDevice);
  int rows[8] = {5, 77, 3, 999, 0, 500, 501, 12};
  cudaMemcpy(dr, rows, 32, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap map;
  cuuint64_t dims[2] = {C, R}, strides[1] = {C * 4};
  cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  CUresult rc = ((EncodeFn)fn)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d\n", (int)rc);
  probe<<<1, 32>>>(map, dr, 32, o);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float out[256]; cudaMemcpy(out, o, sizeof(out), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int r = 0; r < 8; ++r) {
    for (int k = 0; k < 32; ++k) {
      // SW128: element (r, k) at 16-B chunk (k/4 ^ r%8), slot k%4
      const int idx = r * 32 + (((k >> 2) ^ (r & 7)) << 2) + (k & 3);
      const float want = rows[r] * 1000 + 32 + k;
      if (out[idx] != want) ++bad;
    }
  }
  printf("row0: %g %g %g %g | row3: %g | bad=%d\n", out[0], out[1], out[2], out[3], out[3 * 32], bad);
  return 0;
}
