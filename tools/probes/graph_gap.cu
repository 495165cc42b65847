// Probe: per-node cost of a chain of small kernels replayed as a CUDA graph,
// with and without programmatic dependent launch (PDL: the next grid launches
// while the previous one drains; griddepcontrol.wait orders the data).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_plain(float* p, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 0.5f + 1.f;
}
__global__ void k_pdl(float* p, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 0.5f + 1.f;
  asm volatile("griddepcontrol.launch_dependents;");
}
int main() {
  const int n = 148 * 256, nodes = 64;
  float* d; cudaMalloc(&d, n * sizeof(float)); cudaMemset(d, 0, n * sizeof(float));
  cudaStream_t s; cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < nodes; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      if (pdl) cudaLaunchKernelEx(&cfg, k_pdl, d, n); else cudaLaunchKernelEx(&cfg, k_plain, d, n);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int r = 0; r < 20; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s: %.2f us per kernel node\n", pdl ? "PDL  " : "plain", ms * 1e3 / (20 * nodes));
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
