// K8+K2 fused: the fp16 readout of the LSTM model in ONE persistent tcgen05
// kernel (sm_100a). Per 128-instance tile of the last LSTM layer's fp16 h:
//
//   logits  = h16 Wo16 + bo                     MMA 1 (K = H)        -> TMEM
//   loss, dlogits = softmax-xent(logits, y)     epilogue, thread per instance
//   S dh    = (S dlogits16) Wo16^T              MMA 2 (K = C)        -> TMEM -> fp16 dh
//   S dWo  += h16^T (S dlogits16)               MMA 3 (K = 128 rows) -> TMEM, whole launch
//
// h16 is read ONCE (TMA, SWIZZLE_128B boxes); the same shared-memory tile is the
// K-major A operand of MMA 1 and, read MN-major, the A operand of MMA 3. The
// epilogue writes S dlogits16 twice into shared memory: row-major (K-major A of
// MMA 2) and transposed (K-major B of MMA 3). It replaces four launches of the
// unfused path (logits GEMM, dgc_softmax_xent_f16, the dWo split-K GEMM and the
// dh GEMM) and their round trips of logits / dlogits through HBM. The loss and
// the dlogits column sums (the bo gradient) leave as partials per (tile, TMEM
// lane quadrant) and the dWo accumulator as one partial per CTA;
// dgc_epoch_finish / dgc_reduce_rows reduce them in fixed order (deterministic).
//
// Replaces: the synthetic readout + loss of the reference's simulated epoch
// (sim.py:323-324, restated in oracle/dgnn.py); S = 2^e is the trainer's
// power-of-two gradient scale, removed exactly from dWo here
// and from dh by the BPTT that consumes it (dgc_rnn_bwd_tc bit 25).
//
// Roles (448 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer, warps 2-5 = softmax group (logits -> loss, dlogits operands, partials),
// warps 6-13 = dh group (two per TMEM lane quadrant, 64 columns each, double-
// buffered accumulator: tile i's dh leaves while tile i+1's softmax runs).
// Warp w reads TMEM lanes 32 (w % 4) .. 32 (w % 4) + 31.
#include <cuda_fp16.h>

#include "tc_common.cuh"

namespace {

using namespace dgc::tc;

constexpr int kH = 128;               // hidden width (K of MMA 1, N of MMA 2, M of MMA 3)
constexpr int kStages = 3;            // h16 tiles in flight
constexpr int kTileBytes = BM * kH * 2;  // 32 KB: two [128 x 64] SWIZZLE_128B boxes
constexpr int kStgStride = 144;       // dh staging row stride (bytes): conflict-free 16-B accesses
constexpr int kThreads = 64 + 128 + 256;
constexpr int kStgStrideEvo = 272;    // fp32 dZ2 staging: 32 rows x 64 floats + 16 B

// byte offset of fp16 element (row, k) (k < 64) in a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t sw128_h(int row, int k) {
  return (uint32_t)row * 128u + ((((uint32_t)k >> 3) ^ ((uint32_t)row & 7u)) << 4) +
         (((uint32_t)k & 7u) << 1);
}
__device__ __forceinline__ void sts_b16(uint32_t addr, __half v) {
  asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(__half_as_ushort(v)) : "memory");
}

// one level of a butterfly column-sum over the warp: keep W/2 of the lane's W
// column partials, exchange the other half with lane ^ OFF; once a lane holds
// one column, the remaining levels sum it plainly
template <int W, int OFF>
__device__ __forceinline__ void butterfly_colsum(float* v, int lane, int& col) {
  if constexpr (OFF >= 1) {
    if constexpr (W > 1) {
      const bool up = (lane & OFF) != 0;
#pragma unroll
      for (int j = 0; j < W / 2; ++j) {
        const float send = up ? v[j] : v[j + W / 2];
        const float keep = up ? v[j + W / 2] : v[j];
        v[j] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
      }
      col += up ? W / 2 : 0;
      butterfly_colsum<W / 2, OFF / 2>(v, lane, col);
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], OFF);
      butterfly_colsum<1, OFF / 2>(v, lane, col);
    }
  }
}

// EVO (EvolveGCN-O, whose readout input is H2 = relu(.)): the dh group writes
// dZ2 = dh * (H2 > 0) as fp32 (the mask is the h tile itself, held in shared
// memory until the group has read it) and the dZ2 column sums (the b2 gradient)
// per (tile, quadrant); else S dh as fp16.
template <int C, bool EVO>
__global__ void __launch_bounds__(kThreads, 1)
    readout_f16_kernel(const __grid_constant__ CUtensorMap tmH, const __half* __restrict__ Wo16,
                       const float* __restrict__ bo, const int32_t* __restrict__ labels, int64_t n,
                       int m_tiles, float scale, float scale16, __half* __restrict__ dh16,
                       double* __restrict__ loss_partial, float* __restrict__ dl_partial,
                       float* __restrict__ dwo_partial, float* __restrict__ dz2,
                       float* __restrict__ b2_partial) {
  constexpr int kStg = EVO ? kStgStrideEvo : kStgStride;
  static_assert(C == 16 || C == 32, "readout_f16: C must be 16 or 32");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sH = smem;                                   // [kStages][2 boxes][128 rows][128 B]
  uint8_t* sWoT = sH + kStages * kTileBytes;            // MMA 1 B: [2 k-blocks][C rows][128 B]
  uint8_t* sWo = sWoT + 2 * C * 128;                    // MMA 2 B: [H rows][128 B] (k < C used)
  uint8_t* sDlA = sWo + kH * 128;                       // MMA 2 A: [128 rows][128 B] (k < C used)
  uint8_t* sDlT = sDlA + BM * 128;                      // MMA 3 B: [2 k-blocks][C rows][128 B]
  uint8_t* sStg = sDlT + 2 * C * 128;                   // dh staging [8 warps][32 rows][144 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(sStg + 8 * 32 * kStg);
  uint64_t* empty = full + kStages;
  uint64_t* acc1_full = empty + kStages;
  uint64_t* acc1_empty = acc1_full + 1;
  uint64_t* dl_ready = acc1_empty + 1;
  uint64_t* dl_free = dl_ready + 1;
  uint64_t* acc2_full = dl_free + 1;    // [2]
  uint64_t* acc2_empty = acc2_full + 2;  // [2]
  uint64_t* dwo_full = acc2_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dwo_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // TMEM columns: logits [0, C), S dWo [32, 32 + C), S dh [128, 256) and [256, 384)
  constexpr uint32_t kAcc1 = 0, kAcc3 = 32, kAcc2 = 128, kTmemCols = 512;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], EVO ? 9 : 1);  // EVO: + the 8 dh warps (the mask)
    }
    mbar_init(acc1_full, 1);
    mbar_init(acc1_empty, 4);
    mbar_init(dl_ready, 4);
    mbar_init(dl_free, 1);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc2_full[a], 1);
      mbar_init(&acc2_empty[a], 8);
    }
    mbar_init(dwo_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmH) : "memory");
  }
  // resident B operands from Wo16 [H][C] (row-major): Wo^T for MMA 1 (row c holds
  // Wo[:, c] over two 64-wide k-blocks) and Wo for MMA 2 (row h holds Wo[h, :])
  for (int e = threadIdx.x; e < kH * C; e += blockDim.x) {
    const int h = e / C, c = e % C;
    const __half v = Wo16[e];
    sts_b16(smem_u32(sWoT) + (uint32_t)((h >> 6) * C * 128) + sw128_h(c, h & 63), v);
    sts_b16(smem_u32(sWo) + sw128_h(h, c), v);
  }
  fence_async_smem();
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int i = 0;
      for (int t = blockIdx.x; t < m_tiles; t += gridDim.x, ++i) {
        const int s = i % kStages;
        mbar_wait(&empty[s], ((i / kStages) & 1) ^ 1);
        mbar_expect_tx(&full[s], (uint32_t)kTileBytes);
        uint8_t* dst = sH + s * kTileBytes;
        tma_load_2d(dst, &tmH, 0, t * BM, &full[s]);
        tma_load_2d(dst + BM * 128, &tmH, 64, t * BM, &full[s]);
      }
    }
  } else if (warp == 1) {
    const uint32_t id1 = idesc_f16(C);                 // [128 x C] = h (K-major) x WoT
    const uint32_t id2 = idesc_f16(kH);                // [128 x H] = dl (K-major) x Wo
    const uint32_t id3 = idesc_f16mn(C, true, false);  // [H x C] = h^T (MN-major) x dl^T
    const uint32_t woT = smem_u32(sWoT), wo = smem_u32(sWo);
    const uint32_t dlA = smem_u32(sDlA), dlT = smem_u32(sDlT);
    // logits of tile j (MMA 1): issued one tile ahead, so tile j+1's product runs
    // under tile j's softmax (acc1 is released as soon as the epilogue read it)
    auto mma1 = [&](int j) {
      const int s = j % kStages;
      const uint32_t hs = smem_u32(sH + s * kTileBytes);
      mbar_wait(&full[s], (j / kStages) & 1);
      mbar_wait(acc1_empty, (j & 1) ^ 1);
      fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kb = 0; kb < 2; ++kb)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16(tmem_base + kAcc1, kdesc(hs + kb * BM * 128 + kk * 32),
                    kdesc(woT + kb * C * 128 + kk * 32), id1, (kb | kk) ? 1u : 0u);
        mma_commit(acc1_full);
      }
      __syncwarp();
    };
    const int my_tiles = blockIdx.x < m_tiles ? (m_tiles - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;
    if (my_tiles > 0) mma1(0);
    for (int i = 0; i < my_tiles; ++i) {
      const int s = i % kStages;
      const uint32_t hs = smem_u32(sH + s * kTileBytes);
      if (i + 1 < my_tiles) mma1(i + 1);
      const int a2 = i & 1;
      mbar_wait(dl_ready, i & 1);
      mbar_wait(&acc2_empty[a2], ((i >> 1) & 1) ^ 1);
      fence_after();
      if (lane == 0) {
#pragma unroll
        for (int kk = 0; kk < C / 16; ++kk)
          mma_f16(tmem_base + kAcc2 + a2 * 128, kdesc(dlA + kk * 32), kdesc(wo + kk * 32), id2,
                  kk ? 1u : 0u);
        // S dWo += h^T dl: A = the h tile read MN-major (64-unit chunks are the
        // two boxes, 16 KB apart; 16 instance rows = 2 KB per MMA), B = dl^T
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_f16(tmem_base + kAcc3, sdesc(hs + kk * 2048, BM * 128, 1024, 2),
                  kdesc(dlT + (kk >> 2) * C * 128 + (kk & 3) * 32), id3, (i | kk) ? 1u : 0u);
        mma_commit(&acc2_full[a2]);
        mma_commit(&empty[s]);
        mma_commit(dl_free);
      }
      __syncwarp();
    }
    if (lane == 0) mma_commit(dwo_full);
    __syncwarp();
  } else if (warp < 6) {
    const int q = warp & 3;  // TMEM lane quadrant
    const int rl = 32 * q + lane;  // this thread's instance row in the tile
    const uint32_t tq = tmem_base + ((uint32_t)(32 * q) << 16);
    const uint32_t dlA = smem_u32(sDlA), dlT = smem_u32(sDlT);
    float bov[C];
#pragma unroll
    for (int c = 0; c < C; ++c) bov[c] = __ldg(bo + c);
    int i = 0;
    // labels one tile ahead (their load latency was exposed before every softmax)
    int y_next = (int64_t)blockIdx.x * BM + rl < n ? __ldg(labels + (int64_t)blockIdx.x * BM + rl) : -1;
    for (int t = blockIdx.x; t < m_tiles; t += gridDim.x, ++i) {
      const int64_t row = (int64_t)t * BM + rl;
      const int y = y_next;  // y < 0: padding (no loss, no gradient)
      {
        const int64_t nrow = row + (int64_t)gridDim.x * BM;
        y_next = (t + (int)gridDim.x < m_tiles && nrow < n) ? __ldg(labels + nrow) : -1;
      }
      mbar_wait(acc1_full, i & 1);
      fence_after();
      float x[C];
      tmem_ld16(tq + kAcc1, x);
      if (C == 32) tmem_ld16(tq + kAcc1 + 16, x + 16);
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc1_empty);
      // softmax cross-entropy of this row (dgc_softmax_xent_f16's arithmetic)
      float m = -INFINITY, zy = 0.f;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        x[c] += bov[c];
        m = fmaxf(m, x[c]);
        if (c == y) zy = x[c];
      }
      float ssum = 0.f;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        x[c] = __expf(x[c] - m);
        ssum += x[c];
      }
      double l = (y >= 0 && row < n) ? -(double)(zy - m - logf(ssum)) : 0.0;
      const float inv = 1.f / ssum;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        float p = x[c] * inv;
        if (c == y) p -= 1.f;
        if (y < 0) p = 0.f;
        x[c] = p * scale;
      }
      // S dlogits16 into both MMA operand layouts (after the previous tile's
      // MMAs 2 / 3 have read them)
      if (i > 0) mbar_wait(dl_free, (i - 1) & 1);
      {
        uint32_t hv[C / 2];
#pragma unroll
        for (int c = 0; c < C / 2; ++c) {
          const __half2 h2 = __floats2half2_rn(x[2 * c] * scale16, x[2 * c + 1] * scale16);
          hv[c] = *reinterpret_cast<const uint32_t*>(&h2);
        }
#pragma unroll
        for (int c8 = 0; c8 < C / 8; ++c8)
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dlA + sw128_h(rl, 8 * c8)),
                       "r"(hv[4 * c8]), "r"(hv[4 * c8 + 1]), "r"(hv[4 * c8 + 2]), "r"(hv[4 * c8 + 3])
                       : "memory");
        const uint32_t tb = dlT + (uint32_t)((rl >> 6) * C * 128);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const uint32_t w = hv[c >> 1];
          asm volatile("st.shared.b16 [%0], %1;" ::"r"(tb + sw128_h(c, rl & 63)),
                       "h"((unsigned short)((c & 1) ? (w >> 16) : (w & 0xffffu)))
                       : "memory");
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(dl_ready);
      // loss and dlogits column sums (the bo gradient) per (tile, lane quadrant):
      // no barrier among the softmax warps; the partial rows are reduced in fixed order
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      if (lane == 0) loss_partial[4 * (int64_t)t + q] = l;
      {
        // butterfly: each level halves the columns a lane keeps (C - 1 shuffles
        // for C <= 32 instead of 5 C); the lane ends with column col
        float v[C];
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = x[c];
        int col = 0;
        butterfly_colsum<C, 16>(v, lane, col);
        if (C == 32 || (lane & 1) == 0) dl_partial[(4 * (int64_t)t + q) * C + col] = v[0];
      }
    }
    // the launch's S dWo accumulator: lane = hidden unit, C columns -> partial / S
    if (i > 0) {
      mbar_wait(dwo_full, 0);
      fence_after();
      float v[C];
      tmem_ld16(tq + kAcc3, v);
      if (C == 32) tmem_ld16(tq + kAcc3 + 16, v + 16);
      const float inv16 = 1.f / scale16;
      float* dst = dwo_partial + (int64_t)blockIdx.x * kH * C + (int64_t)rl * C;
#pragma unroll
      for (int c = 0; c < C; c += 4)
        *reinterpret_cast<float4*>(dst + c) =
            make_float4(v[c] * inv16, v[c + 1] * inv16, v[c + 2] * inv16, v[c + 3] * inv16);
    }
  } else {
    // dh group: S dh of 32 rows x 64 columns per warp: TMEM -> fp16 -> staging ->
    // coalesced 128-B row segments
    const int q = warp & 3, half = (warp - 6) >> 2;
    const float inv16 = 1.f / scale16;
    const uint32_t tq = tmem_base + ((uint32_t)(32 * q) << 16) + kAcc2 + 64 * half;
    const uint32_t stg = smem_u32(sStg) + (uint32_t)((warp - 6) * 32 * kStg);
    const int rl = 32 * q + lane;
    int i = 0;
    for (int t = blockIdx.x; t < m_tiles; t += gridDim.x, ++i) {
      const int a2 = i & 1;
      mbar_wait(&acc2_full[a2], (i >> 1) & 1);
      fence_after();
      if constexpr (EVO) {
        // dZ2 = (S dh / S) * (H2 > 0), H2 = this tile's h (stage i % kStages, box = half)
        const uint32_t hb = smem_u32(sH + (i % kStages) * kTileBytes) + (uint32_t)(half * BM * 128 + rl * 128);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          float v[32];
          tmem_ld32(tq + a2 * 128 + 32 * ch, v);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) {
            uint4 m;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(m.x), "=r"(m.y), "=r"(m.z), "=r"(m.w)
                         : "r"(hb + ((((uint32_t)(4 * ch + jj)) ^ ((uint32_t)rl & 7u)) << 4)));
            const uint32_t mq[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&mq[k]));
              v[8 * jj + 2 * k] = f.x > 0.f ? v[8 * jj + 2 * k] * inv16 : 0.f;
              v[8 * jj + 2 * k + 1] = f.y > 0.f ? v[8 * jj + 2 * k + 1] * inv16 : 0.f;
            }
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg + (uint32_t)(lane * kStg + (ch * 8 + j) * 16)),
                         "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]), "f"(v[4 * j + 3])
                         : "memory");
          // column sums of the warp's 32 rows (lane ends with column lane)
          int col = 0;
          butterfly_colsum<32, 16>(v, lane, col);
          b2_partial[(4 * (int64_t)t + q) * kH + 64 * half + 32 * ch + col] = v[0];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[i % kStages]);  // the mask tile is read
      } else {
  #pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          float v[32];
          tmem_ld32(tq + a2 * 128 + 32 * ch, v);
  #pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t p[4];
  #pragma unroll
            for (int e = 0; e < 4; ++e) {
              const __half2 h2 = __floats2half2_rn(v[8 * j + 2 * e], v[8 * j + 2 * e + 1]);
              p[e] = *reinterpret_cast<const uint32_t*>(&h2);
            }
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(
                             stg + (uint32_t)(lane * kStgStride + (ch * 4 + j) * 16)),
                         "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3])
                         : "memory");
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc2_empty[a2]);
      const int64_t wrow0 = (int64_t)t * BM + 32 * q;
      if constexpr (EVO) {
#pragma unroll 4
        for (int it = 0; it < 16; ++it) {
          const int r = 2 * it + (lane >> 4), c16 = lane & 15;
          uint4 v;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "r"(stg + (uint32_t)(r * kStg + c16 * 16)));
          if (wrow0 + r < n) reinterpret_cast<uint4*>(dz2 + (wrow0 + r) * kH + 64 * half)[c16] = v;
        }
      } else {
  #pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int r = 4 * it + (lane >> 3), ch = lane & 7;
          uint4 v;
          asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                       : "r"(stg + (uint32_t)(r * kStgStride + ch * 16)));
          if (wrow0 + r < n) reinterpret_cast<uint4*>(dh16 + (wrow0 + r) * kH + 64 * half)[ch] = v;
        }
      }
      __syncwarp();
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

template <int C, bool EVO>
int launch_readout(const void* h16, const void* Wo16, const float* bo, const int32_t* labels,
                   int64_t n, float scale, float scale16, void* dh16, double* loss_partial,
                   float* dl_partial, float* dwo_partial, float* dz2, float* b2_partial, int grid,
                   cudaStream_t s) {
  CUtensorMap tmH;
  int rc = dgc::make_map_f16(&tmH, h16, n, kH, kH, 64, BM);
  if (rc != DGC_OK) return rc;
  const int m_tiles = (int)((n + BM - 1) / BM);
  const size_t smem = 1024 + (size_t)kStages * kTileBytes + 2 * C * 128 + kH * 128 + BM * 128 +
                      2 * C * 128 + 8 * 32 * (EVO ? kStgStrideEvo : kStgStride) + 16 * 8 + 16;
  auto kern = readout_f16_kernel<C, EVO>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "readout_f16: set smem");
  kern<<<grid, kThreads, smem, s>>>(tmH, static_cast<const __half*>(Wo16), bo, labels, n, m_tiles, scale,
                                    scale16, static_cast<__half*>(dh16), loss_partial, dl_partial,
                                    dwo_partial, dz2, b2_partial);
  DGC_CHECK_LAUNCH("readout_f16_kernel");
  return DGC_OK;
}

}  // namespace

extern "C" int32_t dgc_readout_f16_grid(int64_t n) {
  const int64_t m_tiles = (n + BM - 1) / BM;
  return (int32_t)(m_tiles < dgc::kNumSMs ? (m_tiles < 1 ? 1 : m_tiles) : dgc::kNumSMs);
}

extern "C" int dgc_readout_f16(const void* h16, const void* Wo16, const float* bo,
                               const int32_t* labels, int64_t n, int32_t H, int32_t C, float scale,
                               float scale16, void* dh16, double* loss_partial, float* dl_partial,
                               float* dwo_partial, void* stream) {
  DGC_REQUIRE(H == kH, "readout_f16: H must be 128");
  DGC_REQUIRE(C == 16 || C == 32, "readout_f16: C must be 16 or 32");
  DGC_REQUIRE(n > 0 && n < (int64_t)INT32_MAX / 2, "readout_f16: bad row count");
  DGC_REQUIRE((reinterpret_cast<uintptr_t>(dh16) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dwo_partial) & 15) == 0,
              "readout_f16: dh16 / dwo_partial must be 16-byte aligned");
  cudaStream_t s = dgc::as_stream(stream);
  const int grid = dgc_readout_f16_grid(n);
  return C == 16 ? launch_readout<16, false>(h16, Wo16, bo, labels, n, scale, scale16, dh16, loss_partial,
                                             dl_partial, dwo_partial, nullptr, nullptr, grid, s)
                 : launch_readout<32, false>(h16, Wo16, bo, labels, n, scale, scale16, dh16, loss_partial,
                                             dl_partial, dwo_partial, nullptr, nullptr, grid, s);
}

extern "C" int dgc_readout_f16_evolve(const void* h2_16, const void* Wo16, const float* bo,
                                      const int32_t* labels, int64_t n, int32_t H, int32_t C,
                                      float scale, float scale16, float* dz2, float* b2_partial,
                                      double* loss_partial, float* dl_partial, float* dwo_partial,
                                      void* stream) {
  DGC_REQUIRE(H == kH, "readout_f16_evolve: H must be 128");
  DGC_REQUIRE(C == 16 || C == 32, "readout_f16_evolve: C must be 16 or 32");
  DGC_REQUIRE(n > 0 && n < (int64_t)INT32_MAX / 2, "readout_f16_evolve: bad row count");
  DGC_REQUIRE((reinterpret_cast<uintptr_t>(dz2) & 15) == 0 &&
                  (reinterpret_cast<uintptr_t>(dwo_partial) & 15) == 0,
              "readout_f16_evolve: dz2 / dwo_partial must be 16-byte aligned");
  cudaStream_t s = dgc::as_stream(stream);
  const int grid = dgc_readout_f16_grid(n);
  return C == 16 ? launch_readout<16, true>(h2_16, Wo16, bo, labels, n, scale, scale16, nullptr,
                                            loss_partial, dl_partial, dwo_partial, dz2, b2_partial, grid, s)
                 : launch_readout<32, true>(h2_16, Wo16, bo, labels, n, scale, scale16, nullptr,
                                            loss_partial, dl_partial, dwo_partial, dz2, b2_partial, grid, s);
}
