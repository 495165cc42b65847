// Probe: register <-> (TMEM lane, column) layout of the tcgen05.ld shapes
// 16x64b, 16x128b, 16x256b (x1) for warp 0. TMEM is filled with
// tcgen05.st.32x32b (thread = lane, registers = consecutive columns) with the
// value (lane << 16) | column, then read back with each shape.
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void probe(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su(&slot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot + ((uint32_t)(warp * 32) << 16);
  const uint32_t row = warp * 32 + lane;
  for (int c = 0; c < 32; c += 4) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tm + c),
                 "r"((row << 16) | c), "r"((row << 16) | (c + 1)), "r"((row << 16) | (c + 2)), "r"((row << 16) | (c + 3)));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0) {
    uint32_t a, b, c, d;
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(a) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[0 * 128 + lane * 4] = a;
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[1 * 128 + lane * 4] = a; out[1 * 128 + lane * 4 + 1] = b;
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0, %1, %2, %3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    out[2 * 128 + lane * 4] = a; out[2 * 128 + lane * 4 + 1] = b; out[2 * 128 + lane * 4 + 2] = c; out[2 * 128 + lane * 4 + 3] = d;
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(tm + (16u << 16) + 8));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 8; ++i) out[3 * 128 + lane * 8 + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(slot), "r"(32));
}
int main() {
  uint32_t* d; cudaMalloc(&d, 5 * 128 * 4); cudaMemset(d, 0xff, 5 * 128 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  uint32_t h[640]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[4] = {"16x64b.x1", "16x128b.x1", "16x256b.x1", "16x256b.x2 @lane16 col8"};
  const int nreg[4] = {1, 2, 4, 8};
  for (int s = 0; s < 4; ++s) {
    printf("%s (thread: (lane,col) per register)\n", names[s]);
    for (int t = 0; t < 32; ++t) {
      printf(" t%02d:", t);
      for (int r = 0; r < nreg[s]; ++r) { uint32_t v = h[s * 128 + t * (s == 3 ? 8 : 4) + r]; printf(" (%u,%u)", v >> 16, v & 0xffff); }
      printf("%s", (t % 4 == 3) ? "\n" : "");
    }
  }
  return 0;
}
