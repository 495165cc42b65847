// Shared helpers of the B200-native DGC kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/dgc_b200.h"

namespace dgc {
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
constexpr int kNumSMs = 148;  // B200: 2 dies x 74 SMs
inline int grid_for(int64_t work_items, int block, int per_sm = 8) {
  int64_t g = (work_items + block - 1) / block;
  int64_t cap = (int64_t)kNumSMs * per_sm;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}
// Round an fp32 value to the nearest TF32 (10-bit mantissa, ties away). Outputs
// that feed the tensor cores in TF32 mode are stored pre-rounded so that the
// tcgen05 operand truncation becomes exact (unbiased errors instead of a
// systematic shrink).
__device__ __forceinline__ float rna_tf32_f(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
}  // namespace dgc

#define DGC_CHECK_LAUNCH(what)                                  \
  do {                                                          \
    cudaError_t e_ = cudaGetLastError();                        \
    if (e_ != cudaSuccess) return dgc::cuda_fail(e_, what);     \
  } while (0)

#define DGC_REQUIRE(cond, msg)                                  \
  do {                                                          \
    if (!(cond)) return dgc::fail(DGC_ERR_ARG, msg);            \
  } while (0)
