// Probe: the random-row gather ceiling of one B200 (the bound of K1).
// A sub-warp of LPR lanes (16 B per lane) reads rows Y[idx[e]] for a
// contiguous range of e and folds them into registers (no reduction order, no
// dinv, no output rows: the pure gather). Indices are loaded 32 at a time by a
// coalesced load and broadcast with shuffles, and U rows are in flight per
// sub-warp. Reports gathered rows per second for row sizes 128 / 256 / 512 B
// over an L2-resident source (n rows) and an HBM-sized one.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/row_gather row_gather.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

template <int LPR, int U>
__global__ void __launch_bounds__(256) gather(const uint4* __restrict__ Y, const int* __restrict__ idx,
                                              int64_t n_idx, int per_sub, float* sink) {
  const int lane = threadIdx.x & 31, sl = lane % LPR;
  const int64_t sub = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / LPR;
  const int64_t e0 = sub * per_sub;
  uint32_t acc = 0;
  const unsigned smask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (lane & ~(LPR - 1)));
  for (int64_t b = e0; b < e0 + per_sub && b < n_idx; b += LPR) {
    const int my = (b + sl < n_idx) ? __ldg(idx + b + sl) : 0;
#pragma unroll 1
    for (int k = 0; k < LPR; k += U) {
      uint4 y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = __shfl_sync(smask, my, k + u, LPR);
        y[u] = __ldg(Y + (int64_t)c * LPR + sl);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc ^= y[u].x ^ y[u].y ^ y[u].z ^ y[u].w;
    }
  }
  if (acc == 0x12345678u) sink[0] = 1.f;
}

template <int LPR, int U>
void run(const char* tag, const uint4* Y, const int* idx, int64_t n_idx, float* sink, int occ_blocks) {
  const int per_sub = 64;  // neighbour rows per sub-warp (K1: ~9 per output row)
  const int64_t subs = (n_idx + per_sub - 1) / per_sub;
  const int64_t threads = subs * LPR;
  const int grid = (int)((threads + 255) / 256);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<LPR, U><<<grid, 256>>>(Y, idx, n_idx, per_sub, sink);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    gather<LPR, U><<<grid, 256>>>(Y, idx, n_idx, per_sub, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double rows_s = n_idx / (best * 1e-3);
  printf("%-10s row %3d B  unroll %d: %8.1f us  %6.2f G rows/s  %6.2f TB/s\n", tag, LPR * 16, U,
         best * 1e3, rows_s / 1e9, rows_s * LPR * 16 / 1e12);
  (void)occ_blocks;
}

int main() {
  const int64_t n_idx = 1 << 24;  // 16.8M gathered rows
  float* sink;
  cudaMalloc(&sink, 4);
  int* idx;
  cudaMalloc(&idx, n_idx * 4);
  for (int pass = 0; pass < 2; ++pass) {
    // pass 0: 200k source rows (L2-resident at <= 256 B); pass 1: 10M rows (HBM)
    const int64_t n_rows = pass == 0 ? 200000 : 10000000;
    std::vector<int> h(n_idx);
    std::mt19937 g(1);
    for (auto& v : h) v = (int)(g() % (uint32_t)n_rows);
    cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
    uint4* Y;
    cudaMalloc(&Y, n_rows * 512);
    cudaMemset(Y, 1, n_rows * 512);
    const char* tag = pass == 0 ? "L2 200k" : "HBM 10M";
    run<8, 1>(tag, Y, idx, n_idx, sink, 0);
    run<8, 2>(tag, Y, idx, n_idx, sink, 0);
    run<8, 4>(tag, Y, idx, n_idx, sink, 0);
    run<16, 1>(tag, Y, idx, n_idx, sink, 0);
    run<16, 2>(tag, Y, idx, n_idx, sink, 0);
    run<16, 4>(tag, Y, idx, n_idx, sink, 0);
    run<16, 8>(tag, Y, idx, n_idx, sink, 0);
    run<32, 1>(tag, Y, idx, n_idx, sink, 0);
    run<32, 2>(tag, Y, idx, n_idx, sink, 0);
    run<32, 4>(tag, Y, idx, n_idx, sink, 0);
    run<32, 8>(tag, Y, idx, n_idx, sink, 0);
    cudaFree(Y);
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
