// Readout loss (K8), deterministic reductions and optimizers.
//
// The reference loss trace is synthetic (sim.py:323-324); the B200 trainer
// feeds the real mean cross-entropy into EpochLossTrace.append (stale.py:80),
// which drives threshold() unchanged. Every reduction has a fixed order.
#include <cuda_fp16.h>

#include "common.cuh"

namespace {

__global__ void __launch_bounds__(256) softmax_xent_kernel(const float* __restrict__ logits,
                                                          const int32_t* __restrict__ labels,
                                                          int64_t n, int C, float scale,
                                                          int round_out,
                                                          float* __restrict__ dlogits,
                                                          double* __restrict__ loss_partial,
                                                          float* __restrict__ dl_partial) {
  __shared__ double red[256];
  __shared__ float cred[256];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double l = 0.0;
  if (i < n) {
    const float* x = logits + i * C;
    float m = -INFINITY;
    for (int c = 0; c < C; ++c) m = fmaxf(m, x[c]);
    float s = 0.f;
    for (int c = 0; c < C; ++c) s += __expf(x[c] - m);
    const float ls = logf(s);
    const int y = labels[i];  // y < 0: padding row (no loss, no gradient)
    l = y >= 0 ? -(double)(x[y] - m - ls) : 0.0;
    const float inv = 1.f / s;
    for (int c = 0; c < C; ++c) {
      float p = __expf(x[c] - m) * inv;
      if (c == y) p -= 1.f;
      if (y < 0) p = 0.f;
      dlogits[i * C + c] = round_out ? dgc::rna_tf32_f(p * scale) : p * scale;
    }
  }
  red[threadIdx.x] = l;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss_partial[blockIdx.x] = red[0];
  if (dl_partial) {
    // per-block column sums of dlogits (readout bias gradient), fixed order
    const int64_t r0 = (int64_t)blockIdx.x * blockDim.x;
    const int64_t r1 = min(r0 + (int64_t)blockDim.x, n);
    for (int c = 0; c < C; ++c) {
      __syncthreads();
      cred[threadIdx.x] = (i < n) ? dlogits[i * C + c] : 0.f;
      __syncthreads();
      for (int off = 128; off > 0; off >>= 1) {
        if ((int)threadIdx.x < off) cred[threadIdx.x] += cred[threadIdx.x + off];
        __syncthreads();
      }
      if (threadIdx.x == 0) dl_partial[(int64_t)blockIdx.x * C + c] = (r1 > r0) ? cred[0] : 0.f;
    }
  }
}

// stage 1: block b sums rows [b*rows_per, (b+1)*rows_per) of every column.
// Threads tile (row group, float4 column); partials are combined across row
// groups in fixed order through shared memory (deterministic).
__global__ void __launch_bounds__(256) colsum_stage1(const float* __restrict__ X, int64_t n,
                                                     int width, int64_t ld, int64_t rows_per,
                                                     float* __restrict__ scratch) {
  extern __shared__ float4 red4[];
  const int w4 = width / 4;
  const int cols = w4 < 256 ? w4 : 256;
  const int groups = 256 / cols;
  const int tc = threadIdx.x % cols, tg = threadIdx.x / cols;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per;
  const int64_t r1 = min(r0 + rows_per, n);
  for (int c = tc; c < w4; c += cols) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tg < groups) {
      for (int64_t r = r0 + tg; r < r1; r += groups) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(X + r * ld) + c);
        acc.x += v.x;
        acc.y += v.y;
        acc.z += v.z;
        acc.w += v.w;
      }
    }
    __syncthreads();
    red4[threadIdx.x] = acc;
    __syncthreads();
    if (tg == 0) {
      float4 s = red4[tc];
      for (int g = 1; g < groups; ++g) {
        const float4 v = red4[g * cols + tc];
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
      reinterpret_cast<float4*>(scratch + (int64_t)blockIdx.x * width)[c] = s;
    }
  }
}

// stage 2: out[j] (+)= sum of the nblk partial rows; block = 32 columns x 8
// slab groups (each thread sums every 8th slab), combined in fixed order.
// 32 columns x 32 block groups (the order reduce_rows_batched_stage2 uses)
__global__ void __launch_bounds__(1024) colsum_stage2(const float* __restrict__ scratch, int nblk,
                                                      int width, float* __restrict__ out,
                                                      int accumulate) {
  __shared__ float red[32][33];
  const int j = blockIdx.x * 32 + threadIdx.x;
  float acc = 0.f;
  if (j < width)
#pragma unroll 4
    for (int b = threadIdx.y; b < nblk; b += 32) acc += scratch[(int64_t)b * width + j];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && j < width) {
    float s = 0.f;
    for (int g = 0; g < 32; ++g) s += red[g][threadIdx.x];
    out[j] = accumulate ? out[j] + s : s;
  }
}

// Readout softmax cross-entropy for C <= 32 classes: thread per row (logits in
// registers, 16-byte loads/stores when C % 4 == 0), per-block loss and dlogits
// column sums by warp shuffles + a fixed-order combine of the 8 warps.
template <int CM>
__global__ void __launch_bounds__(256) softmax_xent_small_kernel(
    const float* __restrict__ logits, const int32_t* __restrict__ labels, int64_t n, int C,
    float scale, int round_out, float* __restrict__ dlogits, double* __restrict__ loss_partial,
    float* __restrict__ dl_partial, __half* __restrict__ dl16, float scale16) {
  __shared__ double lred[8];
  __shared__ float cred[8][CM];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool vec = (C & 3) == 0;
  float x[CM];
  double l = 0.0;
  if (i < n) {
    const float* row = logits + i * C;
#pragma unroll
    for (int c = 0; c < CM; c += 4) {
      if (c < C) {
        if (vec) {
          const float4 v = *reinterpret_cast<const float4*>(row + c);
          x[c] = v.x; x[c + 1] = v.y; x[c + 2] = v.z; x[c + 3] = v.w;
        } else {
#pragma unroll
          for (int e = 0; e < 4; ++e) x[c + e] = (c + e < C) ? row[c + e] : 0.f;
        }
      }
    }
    float m = -INFINITY;
#pragma unroll
    for (int c = 0; c < CM; ++c) if (c < C) m = fmaxf(m, x[c]);
    const int y = labels[i];  // y < 0: padding row (no loss, no gradient)
    float zy = 0.f;
#pragma unroll
    for (int c = 0; c < CM; ++c) if (c == y) zy = x[c];
    float ssum = 0.f;
#pragma unroll
    for (int c = 0; c < CM; ++c) if (c < C) { x[c] = __expf(x[c] - m); ssum += x[c]; }
    l = y >= 0 ? -(double)(zy - m - logf(ssum)) : 0.0;
    const float inv = 1.f / ssum;
#pragma unroll
    for (int c = 0; c < CM; ++c) {
      float p = x[c] * inv;
      if (c == y) p -= 1.f;
      if (y < 0) p = 0.f;
      p *= scale;
      x[c] = round_out ? dgc::rna_tf32_f(p) : p;
    }
    if (dlogits) {
      float* drow = dlogits + i * C;
#pragma unroll
      for (int c = 0; c < CM; c += 4) {
        if (c < C) {
          if (vec) {
            *reinterpret_cast<float4*>(drow + c) = make_float4(x[c], x[c + 1], x[c + 2], x[c + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) if (c + e < C) drow[c + e] = x[c + e];
          }
        }
      }
    }
    if (dl16) {  // fp16(scale16 * dlogits): the fp16 readout GEMMs' operand (C % 8 == 0)
      __half* hrow = dl16 + i * C;
#pragma unroll
      for (int c = 0; c < CM; c += 8) {
        if (c < C) {
          uint4 v;
          __half2 h0 = __floats2half2_rn(x[c] * scale16, x[c + 1] * scale16);
          __half2 h1 = __floats2half2_rn(x[c + 2] * scale16, x[c + 3] * scale16);
          __half2 h2 = __floats2half2_rn(x[c + 4] * scale16, x[c + 5] * scale16);
          __half2 h3 = __floats2half2_rn(x[c + 6] * scale16, x[c + 7] * scale16);
          v.x = *reinterpret_cast<uint32_t*>(&h0); v.y = *reinterpret_cast<uint32_t*>(&h1);
          v.z = *reinterpret_cast<uint32_t*>(&h2); v.w = *reinterpret_cast<uint32_t*>(&h3);
          *reinterpret_cast<uint4*>(hrow + c) = v;
        }
      }
    }
  } else {
#pragma unroll
    for (int c = 0; c < CM; ++c) x[c] = 0.f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
  if (lane == 0) lred[w] = l;
  if (dl_partial) {
#pragma unroll
    for (int c = 0; c < CM; ++c) {
      if (c >= C) break;
      float v = x[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) cred[w][c] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += lred[k];
    loss_partial[blockIdx.x] = t;
  }
  if (dl_partial && (int)threadIdx.x < C) {
    float t = 0.f;
    for (int k = 0; k < 8; ++k) t += cred[k][threadIdx.x];
    dl_partial[(int64_t)blockIdx.x * C + threadIdx.x] = t;
  }
}

__global__ void relu_bwd_kernel(const float4* __restrict__ dH, const float4* __restrict__ H,
                                float4* __restrict__ dZ, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 g = dH[i], h = H[i];
    dZ[i] = make_float4(h.x > 0.f ? g.x : 0.f, h.y > 0.f ? g.y : 0.f, h.z > 0.f ? g.z : 0.f,
                        h.w > 0.f ? g.w : 0.f);
  }
}

__global__ void round_tf32_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = dgc::rna_tf32_f(in[i]);
}

// TF32 features shipped as 3 bytes per value (the host rounds to TF32 with the
// same round-to-nearest-away as cvt.rna.tf32, whose low 13 mantissa bits -- the
// whole low byte -- are zero): out = the 24-bit value << 8. Thread = 4 values
// (three 32-bit words in, one float4 out).
__global__ void unpack_tf32x24_kernel(const uint32_t* __restrict__ in, float4* __restrict__ out,
                                      int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t w0 = __ldg(in + 3 * i), w1 = __ldg(in + 3 * i + 1), w2 = __ldg(in + 3 * i + 2);
    float4 o;
    o.x = __uint_as_float((w0 & 0x00ffffffu) << 8);
    o.y = __uint_as_float(((w0 >> 24) | ((w1 & 0xffffu) << 8)) << 8);
    o.z = __uint_as_float(((w1 >> 16) | ((w2 & 0xffu) << 16)) << 8);
    o.w = __uint_as_float(w2 & 0xffffff00u);
    out[i] = o;
  }
}

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g,
                           float* __restrict__ mom, int64_t n, float lr, float mu) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float v = fmaf(mu, mom[i], g[i]);
    mom[i] = v;
    p[i] = fmaf(-lr, v, p[i]);
  }
}

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                            float b1, float b2, float eps, float c1, float c2,
                            const int32_t* __restrict__ step_dev) {
  if (step_dev) {  // step count in device memory (replayable in a CUDA graph)
    const float st = (float)*step_dev;
    c1 = 1.f - powf(b1, st);
    c2 = 1.f - powf(b2, st);
  }
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / c1) / (sqrtf(vi / c2) + eps);
  }
}

// Adam with the device step count and the step's parameter mirrors in one
// pass: p_r = rna_tf32(p) (the TF32-rounded operand copy) and p16 = fp16(p_r)
// (the fp16 GEMMs' weights), each when non-NULL.
__global__ void adam_mirror_kernel(float* __restrict__ p, const float* __restrict__ g,
                                   float* __restrict__ m, float* __restrict__ v, int64_t n,
                                   float lr, float b1, float b2, float eps,
                                   const int32_t* __restrict__ step_dev, float* __restrict__ p_r,
                                   __half* __restrict__ p16) {
  const float st = (float)*step_dev;
  const float c1 = 1.f - powf(b1, st), c2 = 1.f - powf(b2, st);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    const float pn = p[i] - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
    p[i] = pn;
    const float pr = p_r ? dgc::rna_tf32_f(pn) : pn;
    if (p_r) p_r[i] = pr;
    if (p16) p16[i] = __float2half_rn(pr);
  }
}

// End of a step: loss = sum of the per-block loss partials in a fixed order
// (one block), and the device step count advanced for the optimizer.
__global__ void __launch_bounds__(256) epoch_finish_kernel(const double* __restrict__ part, int64_t n,
                                                           double* __restrict__ out,
                                                           int32_t* __restrict__ step_dev) {
  __shared__ double red[256];
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += 256) acc += part[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = red[0];
    if (step_dev) *step_dev += 1;
  }
}

}  // namespace

extern "C" int dgc_adam_dev_mirror(float* p, const float* g, float* m, float* v, int64_t n,
                                   float lr, float beta1, float beta2, float eps,
                                   const int32_t* step_dev, float* p_r, void* p16, void* stream) {
  DGC_REQUIRE(step_dev != nullptr, "adam_dev_mirror: step_dev is NULL");
  if (n == 0) return DGC_OK;
  adam_mirror_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(
      p, g, m, v, n, lr, beta1, beta2, eps, step_dev, p_r, static_cast<__half*>(p16));
  DGC_CHECK_LAUNCH("adam_mirror_kernel");
  return DGC_OK;
}

extern "C" int dgc_epoch_finish(const double* loss_partial, int64_t n, double* loss_out,
                                int32_t* step_dev, void* stream) {
  DGC_REQUIRE(loss_out != nullptr && (n == 0 || loss_partial != nullptr),
              "epoch_finish: NULL buffer");
  epoch_finish_kernel<<<1, 256, 0, dgc::as_stream(stream)>>>(loss_partial, n, loss_out, step_dev);
  DGC_CHECK_LAUNCH("epoch_finish_kernel");
  return DGC_OK;
}

extern "C" int dgc_softmax_xent(const float* logits, const int32_t* labels, int64_t n, int32_t C,
                                float scale, int32_t flags, float* dlogits, double* loss_partial,
                                float* dl_partial, void* stream) {
  DGC_REQUIRE(C >= 1, "softmax_xent: C must be >= 1");
  if (n == 0) return DGC_OK;
  const int blocks = (int)((n + 255) / 256);
  const bool aligned = (reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(dlogits) & 15) == 0;
  if (C <= 16 && (aligned || (C & 3) != 0)) {  // (16 logits in registers: no idle guarded lanes)
    softmax_xent_small_kernel<16><<<blocks, 256, 0, dgc::as_stream(stream)>>>(
        logits, labels, n, C, scale, flags & 1, dlogits, loss_partial, dl_partial, nullptr, 1.f);
  } else if (C <= 32 && (aligned || (C & 3) != 0)) {
    softmax_xent_small_kernel<32><<<blocks, 256, 0, dgc::as_stream(stream)>>>(
        logits, labels, n, C, scale, flags & 1, dlogits, loss_partial, dl_partial, nullptr, 1.f);
  } else {
    softmax_xent_kernel<<<blocks, 256, 0, dgc::as_stream(stream)>>>(logits, labels, n, C, scale,
                                                                   flags & 1, dlogits, loss_partial,
                                                                   dl_partial);
  }
  DGC_CHECK_LAUNCH("softmax_xent_kernel");
  return DGC_OK;
}

extern "C" int dgc_softmax_xent_f16(const float* logits, const int32_t* labels, int64_t n, int32_t C,
                                    float scale, float* dlogits, double* loss_partial,
                                    float* dl_partial, void* dlogits16, float scale16, void* stream) {
  DGC_REQUIRE(C >= 1 && C <= 32 && C % 8 == 0, "softmax_xent_f16: C must be 8, 16, 24 or 32");
  DGC_REQUIRE(dlogits16 != nullptr && (reinterpret_cast<uintptr_t>(dlogits16) & 15) == 0,
              "softmax_xent_f16: dlogits16 must be 16-byte aligned");
  DGC_REQUIRE((reinterpret_cast<uintptr_t>(logits) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dlogits) & 15) == 0,
              "softmax_xent_f16: logits / dlogits must be 16-byte aligned");
  if (n == 0) return DGC_OK;
  const int blocks = (int)((n + 255) / 256);
  if (C <= 16)
    softmax_xent_small_kernel<16><<<blocks, 256, 0, dgc::as_stream(stream)>>>(
        logits, labels, n, C, scale, 0, dlogits, loss_partial, dl_partial,
        static_cast<__half*>(dlogits16), scale16);
  else
    softmax_xent_small_kernel<32><<<blocks, 256, 0, dgc::as_stream(stream)>>>(
        logits, labels, n, C, scale, 0, dlogits, loss_partial, dl_partial,
        static_cast<__half*>(dlogits16), scale16);
  DGC_CHECK_LAUNCH("softmax_xent_kernel");
  return DGC_OK;
}

extern "C" int dgc_colsum(const float* X, int64_t n, int32_t width, int64_t ld, float* out,
                          int32_t accumulate, float* scratch, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && ld % 4 == 0, "colsum: width and ld must be multiples of 4");
  cudaStream_t s = dgc::as_stream(stream);
  // ~2 blocks per SM, at least 64 rows each; scratch holds nblk*width floats
  int64_t rows_per = (n + 2 * dgc::kNumSMs - 1) / (2 * dgc::kNumSMs);
  if (rows_per < 64) rows_per = 64;
  const int nblk = (int)((n + rows_per - 1) / rows_per);
  if (nblk > 0) {
    colsum_stage1<<<nblk, 256, 256 * sizeof(float4), s>>>(X, n, width, ld, rows_per, scratch);
    DGC_CHECK_LAUNCH("colsum_stage1");
  }
  colsum_stage2<<<(width + 31) / 32, dim3(32, 32), 0, s>>>(scratch, nblk, width, out, accumulate);
  DGC_CHECK_LAUNCH("colsum_stage2");
  return DGC_OK;
}

// Two-level fixed-order row reduction: blocks (32 columns x 8 row groups)
// over a row slab each -> slab partials in scratch -> per-column sum of slabs.
__global__ void __launch_bounds__(256) reduce_rows_stage1(const float* __restrict__ in, int64_t rows,
                                                          int width, int64_t slab,
                                                          float* __restrict__ out) {
  __shared__ float red[8][33];
  const int c = blockIdx.x * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * slab, r1 = min(r0 + slab, rows);
  float acc = 0.f;
  if (c < width)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) acc += in[r * width + c];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < width) {
    float s = 0.f;
    for (int g = 0; g < 8; ++g) s += red[g][threadIdx.x];
    out[(int64_t)blockIdx.y * width + c] = s;
  }
}

// Several row reductions in two launches (the bias gradients of one step):
// stage 1 = reduce_rows_stage1 over every job's (32-column block, slab) pairs,
// stage 2 = colsum_stage2 over every job's column blocks; same fixed order as
// dgc_reduce_rows, so the results are bitwise those of separate calls.
// slabs of a row reduction: 8 rows per slab up to 2048 rows (one-row slabs made
// stage 1 a copy: 148 x 2048 dWo partials took ~11 us), 256 slabs beyond
inline int64_t rr_slabs(int64_t rows) { return rows <= 2048 ? (rows + 7) / 8 : 256; }
constexpr int kRRMaxJobs = 8;
struct RRJobs {
  const float* in[kRRMaxJobs];
  float* out[kRRMaxJobs];
  int64_t rows[kRRMaxJobs];
  int64_t slab[kRRMaxJobs];
  int64_t scr[kRRMaxJobs];   // scratch offset (floats)
  int width[kRRMaxJobs];
  int nslab[kRRMaxJobs];
  int blk1[kRRMaxJobs + 1];  // stage-1 block prefix
  int blk2[kRRMaxJobs + 1];  // stage-2 block prefix
  int n;
};

__global__ void __launch_bounds__(256) reduce_rows_batched_stage1(RRJobs J, float* __restrict__ scratch) {
  __shared__ float red[8][33];
  int j = 0;
  while (j + 1 < J.n && (int)blockIdx.x >= J.blk1[j + 1]) ++j;
  const int local = blockIdx.x - J.blk1[j];
  const int ncb = (J.width[j] + 31) / 32;
  const int cb = local % ncb, sl = local / ncb;
  const int width = J.width[j];
  const int c = cb * 32 + threadIdx.x;
  const int64_t r0 = (int64_t)sl * J.slab[j], r1 = min(r0 + J.slab[j], J.rows[j]);
  float acc = 0.f;
  if (c < width)
    for (int64_t r = r0 + threadIdx.y; r < r1; r += 8) acc += J.in[j][r * width + c];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < width) {
    float s = 0.f;
    for (int g = 0; g < 8; ++g) s += red[g][threadIdx.x];
    scratch[J.scr[j] + (int64_t)sl * width + c] = s;
  }
}

// 32 slab groups per column (<= 8 slabs per thread: the 256-slab sums were a
// latency chain of 32 loads at 8 groups)
__global__ void __launch_bounds__(1024) reduce_rows_batched_stage2(RRJobs J, const float* __restrict__ scratch) {
  __shared__ float red[32][33];
  int j = 0;
  while (j + 1 < J.n && (int)blockIdx.x >= J.blk2[j + 1]) ++j;
  const int width = J.width[j];
  const int c = (blockIdx.x - J.blk2[j]) * 32 + threadIdx.x;
  float acc = 0.f;
  if (c < width)
#pragma unroll 4
    for (int b = threadIdx.y; b < J.nslab[j]; b += 32) acc += scratch[J.scr[j] + (int64_t)b * width + c];
  red[threadIdx.y][threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.y == 0 && c < width) {
    float s = 0.f;
    for (int g = 0; g < 32; ++g) s += red[g][threadIdx.x];
    J.out[j][c] = s;
  }
}

extern "C" int dgc_reduce_rows_batched(int32_t n_jobs, const float* const* partials,
                                       const int64_t* rows, const int32_t* widths,
                                       float* const* outs, void* stream) {
  DGC_REQUIRE(n_jobs >= 1 && n_jobs <= kRRMaxJobs, "reduce_rows_batched: 1..8 jobs");
  RRJobs J{};
  J.n = n_jobs;
  int64_t scr = 0;
  J.blk1[0] = J.blk2[0] = 0;
  for (int j = 0; j < n_jobs; ++j) {
    DGC_REQUIRE(widths[j] >= 1 && rows[j] >= 1, "reduce_rows_batched: empty job");
    J.in[j] = partials[j];
    J.out[j] = outs[j];
    J.rows[j] = rows[j];
    J.width[j] = widths[j];
    int64_t slabs = rr_slabs(rows[j]);  // as dgc_reduce_rows
    const int64_t slab = (rows[j] + slabs - 1) / slabs;
    slabs = (rows[j] + slab - 1) / slab;
    J.slab[j] = slab;
    J.nslab[j] = (int)slabs;
    J.scr[j] = scr;
    scr += slabs * widths[j];
    const int ncb = (widths[j] + 31) / 32;
    J.blk1[j + 1] = J.blk1[j] + ncb * (int)slabs;
    J.blk2[j + 1] = J.blk2[j] + ncb;
  }
  // fixed-size scratch, allocated once and never freed: captured CUDA graphs
  // keep pointing at it (<= 8 jobs x 256 slabs x 4096 columns)
  constexpr int64_t kScratch = (int64_t)kRRMaxJobs * 256 * 4096;
  DGC_REQUIRE(scr <= kScratch, "reduce_rows_batched: jobs too wide");
  static float* scratch = nullptr;
  if (!scratch) {
    cudaError_t e = cudaMalloc(&scratch, kScratch * sizeof(float));
    if (e != cudaSuccess) return dgc::cuda_fail(e, "reduce_rows_batched scratch");
  }
  cudaStream_t s = dgc::as_stream(stream);
  reduce_rows_batched_stage1<<<J.blk1[n_jobs], dim3(32, 8), 0, s>>>(J, scratch);
  DGC_CHECK_LAUNCH("reduce_rows_batched_stage1");
  reduce_rows_batched_stage2<<<J.blk2[n_jobs], dim3(32, 32), 0, s>>>(J, scratch);
  DGC_CHECK_LAUNCH("reduce_rows_batched_stage2");
  return DGC_OK;
}

extern "C" int dgc_reduce_rows(const float* partial, int64_t rows, int32_t width, float* out,
                               int32_t accumulate, void* stream) {
  if (width == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  // slab partials live in a small static scratch (<= 256 slabs x 4096 columns)
  static float* scratch = nullptr;
  static size_t scratch_n = 0;
  int64_t slabs = rr_slabs(rows > 0 ? rows : 1);
  if (slabs * width > 256 * 4096) return dgc::fail(DGC_ERR_ARG, "reduce_rows: width too large");
  if (!scratch) {
    scratch_n = 256 * 4096;
    cudaError_t e = cudaMalloc(&scratch, scratch_n * sizeof(float));
    if (e != cudaSuccess) return dgc::cuda_fail(e, "reduce_rows scratch");
  }
  const int64_t slab = (rows + slabs - 1) / slabs;
  slabs = rows > 0 ? (rows + slab - 1) / slab : 0;
  if (slabs > 0) {
    dim3 grid((unsigned)((width + 31) / 32), (unsigned)slabs);
    reduce_rows_stage1<<<grid, dim3(32, 8), 0, s>>>(partial, rows, width, slab, scratch);
    DGC_CHECK_LAUNCH("reduce_rows_stage1");
  }
  colsum_stage2<<<(width + 31) / 32, dim3(32, 32), 0, s>>>(scratch, (int)slabs, width, out,
                                                         accumulate);
  DGC_CHECK_LAUNCH("reduce_rows_stage2");
  return DGC_OK;
}

extern "C" int dgc_relu_bwd(const float* dH, const float* H, float* dZ, int64_t n, void* stream) {
  DGC_REQUIRE(n % 4 == 0, "relu_bwd: n must be a multiple of 4");
  if (n == 0) return DGC_OK;
  relu_bwd_kernel<<<dgc::grid_for(n / 4, 256), 256, 0, dgc::as_stream(stream)>>>(
      reinterpret_cast<const float4*>(dH), reinterpret_cast<const float4*>(H),
      reinterpret_cast<float4*>(dZ), n / 4);
  DGC_CHECK_LAUNCH("relu_bwd_kernel");
  return DGC_OK;
}

extern "C" int dgc_unpack_tf32x24(const uint8_t* in, float* out, int64_t n, void* stream) {
  DGC_REQUIRE(n % 4 == 0, "unpack_tf32x24: n must be a multiple of 4");
  DGC_REQUIRE((reinterpret_cast<uintptr_t>(in) & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0,
              "unpack_tf32x24: misaligned buffers");
  if (n == 0) return DGC_OK;
  unpack_tf32x24_kernel<<<dgc::grid_for(n / 4, 256), 256, 0, dgc::as_stream(stream)>>>(
      reinterpret_cast<const uint32_t*>(in), reinterpret_cast<float4*>(out), n / 4);
  DGC_CHECK_LAUNCH("unpack_tf32x24_kernel");
  return DGC_OK;
}

__global__ void round_f16_kernel(const float* __restrict__ in, float* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __half2float(__float2half_rn(in[i]));
}

// fp16 features shipped from the host (2 bytes per value): thread = 8 values
// (one 16-B load, two float4 stores)
__global__ void unpack_f16_kernel(const uint4* __restrict__ in, float4* __restrict__ out,
                                  int64_t n8) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 u = __ldg(in + i);
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    const float2 c = __half22float2(*reinterpret_cast<const __half2*>(&u.z));
    const float2 d = __half22float2(*reinterpret_cast<const __half2*>(&u.w));
    out[2 * i] = make_float4(a.x, a.y, b.x, b.y);
    out[2 * i + 1] = make_float4(c.x, c.y, d.x, d.y);
  }
}

extern "C" int dgc_round_f16(const float* in, float* out, int64_t n, void* stream) {
  if (n == 0) return DGC_OK;
  round_f16_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(in, out, n);
  DGC_CHECK_LAUNCH("round_f16_kernel");
  return DGC_OK;
}

extern "C" int dgc_unpack_f16(const void* in, float* out, int64_t n, void* stream) {
  DGC_REQUIRE(n % 8 == 0, "unpack_f16: n must be a multiple of 8");
  DGC_REQUIRE((reinterpret_cast<uintptr_t>(in) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0,
              "unpack_f16: misaligned buffers");
  if (n == 0) return DGC_OK;
  unpack_f16_kernel<<<dgc::grid_for(n / 8, 256), 256, 0, dgc::as_stream(stream)>>>(
      static_cast<const uint4*>(in), reinterpret_cast<float4*>(out), n / 8);
  DGC_CHECK_LAUNCH("unpack_f16_kernel");
  return DGC_OK;
}

__global__ void to_f16_kernel(const float* __restrict__ in, __half* __restrict__ out, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2half_rn(in[i]);
}

extern "C" int dgc_to_f16(const float* in, void* out, int64_t n, void* stream) {
  if (n == 0) return DGC_OK;
  to_f16_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(
      in, static_cast<__half*>(out), n);
  DGC_CHECK_LAUNCH("to_f16_kernel");
  return DGC_OK;
}

extern "C" int dgc_round_tf32(const float* in, float* out, int64_t n, void* stream) {
  if (n == 0) return DGC_OK;
  round_tf32_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(in, out, n);
  DGC_CHECK_LAUNCH("round_tf32_kernel");
  return DGC_OK;
}

extern "C" int dgc_sgd(float* p, const float* g, float* mom, int64_t n, float lr, float momentum,
                       void* stream) {
  if (n == 0) return DGC_OK;
  sgd_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(p, g, mom, n, lr, momentum);
  DGC_CHECK_LAUNCH("sgd_kernel");
  return DGC_OK;
}

extern "C" int dgc_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                        float beta1, float beta2, float eps, int32_t step, void* stream) {
  if (n == 0) return DGC_OK;
  const float c1 = 1.f - powf(beta1, (float)step), c2 = 1.f - powf(beta2, (float)step);
  adam_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(p, g, m, v, n, lr, beta1,
                                                                       beta2, eps, c1, c2, nullptr);
  DGC_CHECK_LAUNCH("adam_kernel");
  return DGC_OK;
}

extern "C" int dgc_adam_dev(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                            float beta1, float beta2, float eps, const int32_t* step_dev,
                            void* stream) {
  DGC_REQUIRE(step_dev != nullptr, "adam_dev: step_dev is NULL");
  if (n == 0) return DGC_OK;
  adam_kernel<<<dgc::grid_for(n, 256), 256, 0, dgc::as_stream(stream)>>>(p, g, m, v, n, lr, beta1,
                                                                       beta2, eps, 1.f, 1.f, step_dev);
  DGC_CHECK_LAUNCH("adam_kernel");
  return DGC_OK;
}

extern "C" int dgc_zero_async(void* ptr, int64_t bytes, void* stream) {
  DGC_REQUIRE(bytes >= 0, "zero_async: negative size");
  if (bytes == 0) return DGC_OK;
  cudaError_t e = cudaMemsetAsync(ptr, 0, (size_t)bytes, dgc::as_stream(stream));
  return e == cudaSuccess ? DGC_OK : dgc::cuda_fail(e, "zero_async");
}
