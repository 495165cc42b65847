// Probe: tcgen05.mma.cta_group::2 (kind::f16, M = 256, N = 128, K = 64) in a
// 2-CTA cluster: each CTA holds its 128 rows of A and half (64) of the N rows
// of B^T (K-major, SWIZZLE_128B); the leader issues; each CTA's TMEM receives
// its 128 rows x all 128 columns. Checks D against the host product.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((16 >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((1024 >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ uint32_t swz(int row, int kbyte) {  // K-major SW128 byte offset
  return (uint32_t)(row * 128 + ((((kbyte >> 4) ^ (row & 7))) << 4) + (kbyte & 15));
}
constexpr int K = 64, N = 128, NH = 64;
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const __half* A, const __half* Bt, float* D) {  // A [256 x K], Bt [N x K], D [256 x N]
  __shared__ __align__(1024) uint8_t sA[128 * 128];
  __shared__ __align__(1024) uint8_t sB[NH * 128];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int t = threadIdx.x, warp = t >> 5;
  // fill: A rows rank*128 + r, B^T rows rank*64 + n
  for (int r = t; r < 128; r += 128)
    for (int k = 0; k < K; ++k)
      *reinterpret_cast<__half*>(sA + swz(r, 2 * k)) = A[(rank * 128 + r) * K + k];
  for (int n = t; n < NH; n += 128)
    for (int k = 0; k < K; ++k)
      *reinterpret_cast<__half*>(sB + swz(n, 2 * k)) = Bt[(rank * NH + n) * K + k];
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&tslot)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tslot;
  if (rank == 0 && t == 0) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    for (int kk = 0; kk < K / 16; ++kk) {
      const uint64_t ad = sdesc(su(sA) + kk * 32), bd = sdesc(su(sB) + kk * 32);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm),
                   "l"(ad), "l"(bd), "r"(idesc), "r"(kk > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(su(&bar)), "h"((uint16_t)3) : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done) : "r"(su(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c = 0; c < N; c += 8) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) D[(rank * 128 + t) * N + c + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(128));
}

int main() {
  std::vector<__half> A(256 * K), Bt(N * K);
  std::vector<float> Af(256 * K), Bf(N * K), D(256 * N, -1.f);
  for (int i = 0; i < 256 * K; ++i) { Af[i] = (float)((i * 7919 % 17) - 8) / 8.f; A[i] = __float2half(Af[i]); }
  for (int i = 0; i < N * K; ++i) { Bf[i] = (float)((i * 104729 % 13) - 6) / 4.f; Bt[i] = __float2half(Bf[i]); }
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, Bt.size() * 2); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bt.data(), Bt.size() * 2, cudaMemcpyHostToDevice);
  probe<<<2, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < 256; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)Af[m * K + k] * Bf[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
    }
  printf("cta_group::2 M=256 N=128 K=64: max |err| = %g (D[0][0]=%f, D[200][100]=%f)\n", maxerr, D[0], D[200 * N + 100]);
  return maxerr < 1e-3 ? 0 : 2;
}
