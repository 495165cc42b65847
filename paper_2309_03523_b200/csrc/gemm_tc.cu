// K2: tcgen05 TF32 GEMM for the DGNN's dense contractions (sm_100a).
//
// C[M,N] = op(A) op(B) with fp32 storage, TF32 tensor-core math and fp32
// accumulation in TMEM; "3xTF32" (hi*hi + hi*lo + lo*hi) gives fp32-level
// accuracy for the parity mode. The shapes of this workload are tall-skinny
// (M = instances per device, K and N = feature widths <= 512), so the kernel
// streams 128-row M tiles of A through a multi-stage TMA -> SMEM pipeline
// (SWIZZLE_128B, K-major or MN-major), one elected thread issues
// tcgen05.mma.cta_group::1.kind::tf32 into a TMEM accumulator of up to 256
// columns, and four epilogue warps drain TMEM (tcgen05.ld 32x32b) with fused
// bias / ReLU-mask / accumulate epilogues. Weight gradients (K = instances)
// split K over CTAs and reduce the partials in fixed order (deterministic).
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer, warps 2-5 = 3xTF32 hi/lo converters, then epilogue. Every mbarrier
// wait carries a watchdog (trap after ~4 s) so a bad descriptor can never
// hang the GPU.

#include <cuda_fp16.h>

#include "tc_common.cuh"

namespace {

using namespace dgc::tc;
using dgc::make_map;
using dgc::make_map_f16;
using dgc::make_map_f16_sw64;
constexpr int kEpiWarps = 8;  // 2 per TMEM lane quadrant, round-robin 32-column chunks
constexpr int kThreads = 64 + 32 * kEpiWarps;
constexpr int kABytes = BM * BK * 4;  // 16 KiB

template <bool A_MN, bool B_MN, bool SPLIT3, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, int tma_store, int64_t c_rows_per_z,
                     const __grid_constant__ CUtensorMap tmR, int mask_boxes,
                     const __grid_constant__ CUtensorMap tmA2, int64_t a2_row0,
                     float* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int bn, int stages,
                     int kb_total, int kb_per_split, int m_tiles, int n_tiles, int splits,
                     const float* __restrict__ bias, const float* __restrict__ relu_src,
                     int accumulate, float* __restrict__ partial,
                     float* __restrict__ colsum_partial, int b_res,
                     const int32_t* __restrict__ seg_of_mtile, int b_seg_rows,
                     const int32_t* __restrict__ kitems, float alpha, __half* __restrict__ C16,
                     int64_t ldc16, float c16_scale, const __half* __restrict__ relu16,
                     int64_t ldr16) {
  // C16: fp16(c16_scale * C) of the final tile (the next fp16 GEMM's / SpMM's
  // operand); with C == nullptr it is the only output. relu16: an fp16 ReLU-mask
  // source (the fp16 activation the forward consumed).
  // F16: fp16 operands (kind::f16, 64 elements per 128-B k-block row; MN-major
  // boxes of 64 MN elements x 64 k-rows), C = alpha * A B (alpha undoes an
  // operand's power-of-two scale exactly); else fp32 storage, TF32 math
  constexpr int KE = F16 ? 64 : BK;
  // Persistent: CTA c owns tiles c, c+G, ... of the (split, m-tile, n-tile)
  // space, n fastest. With G a multiple of n_tiles every CTA keeps ONE n-tile,
  // so (b_res) its whole B panel is loaded into shared memory once and only A
  // streams; the n_tiles CTAs sharing an A tile run together (L2 dedups A).
  // Two TMEM accumulators let the epilogue drain tile i while the MMA runs i+1.
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived from the __shared__ array (keeps shared-space
  // addressing: STS/LDS instead of generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  // accumulate: bit 0 add into C; output activation bits: 1 ReLU, 2 round to TF32
  const int out_act = accumulate >> 1;
  accumulate &= 1;
  const int b_bytes = bn * BK * 4;
  const int ab_bytes = kABytes + b_bytes;
  const int ld_bytes = b_res ? kABytes : ab_bytes;  // bytes TMA-loaded per stage
  const int stage_bytes = ab_bytes * (SPLIT3 ? 2 : 1);
  uint8_t* bres = smem + (size_t)stages * (b_res ? kABytes : stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(bres + (b_res ? (size_t)kb_total * b_bytes : 0));
  uint64_t* empty = full + stages;
  uint64_t* conv = empty + stages;
  uint64_t* tfull = conv + stages;   // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint64_t* bres_full = tempty + 2;  // [1]
  uint64_t* mfull = bres_full + 1;   // [kEpiWarps] fp16 ReLU-mask boxes landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mfull + kEpiWarps);
  // epilogue staging (transpose buffers, or 4 KB SWIZZLE_128B boxes), 1024-B aligned
  uint8_t* stg_raw = reinterpret_cast<uint8_t*>(tmem_slot + 4);
  float* stg_base = reinterpret_cast<float*>(stg_raw + ((1024u - (smem_u32(stg_raw) & 1023u)) & 1023u));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_total = m_tiles * n_tiles * splits;
  const uint32_t acc_cols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
  const uint32_t tmem_cols = 2 * acc_cols;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 32 * kEpiWarps);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 32 * kEpiWarps);
    }
    mbar_init(bres_full, 1);
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(&mfull[w], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    if (a2_row0 < M) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA2) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  auto tile_coords = [&](int t, int64_t& m0, int64_t& n0, int& z, int& kb0, int& nkb) {
    const int nt = t % n_tiles;
    const int rest = t / n_tiles;
    const int mt = rest % m_tiles;
    z = rest / m_tiles;
    m0 = (int64_t)mt * BM;
    n0 = (int64_t)nt * bn;
    if (kitems) {  // K-segmented work items (per-snapshot weight gradients)
      kb0 = kitems[2 * z];
      nkb = kitems[2 * z + 1];
    } else {
      kb0 = z * kb_per_split;
      nkb = min(kb_total, kb0 + kb_per_split) - kb0;
    }
  };

  if (warp == 0) {
    if (lane == 0) {
      if (b_res && (int)blockIdx.x < n_tiles_total) {
        // the CTA's fixed n-tile: its whole B panel once
        const int64_t n0 = (int64_t)(blockIdx.x % n_tiles) * bn;
        mbar_expect_tx(bres_full, (uint32_t)(kb_total * b_bytes));
        for (int kb = 0; kb < kb_total; ++kb) {
          uint8_t* sb = bres + (size_t)kb * b_bytes;
          if (!B_MN) {
            tma_load_2d(sb, &tmB, kb * KE, (int)n0, bres_full);
          } else if (F16) {
            for (int i = 0; i < bn / 64; ++i)
              tma_load_2d(sb + i * 8192, &tmB, (int)n0 + 64 * i, kb * KE, bres_full);
          } else {
            for (int i = 0; i < bn / 32; ++i)
              tma_load_2d(sb + i * 4096, &tmB, (int)n0 + 32 * i, kb * BK, bres_full);
          }
        }
      }
      int g = 0;
      for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        int64_t m0, n0;
        int z, kb0, nkb;
        tile_coords(t, m0, n0, z, kb0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + (size_t)s * (b_res ? kABytes : stage_bytes);
          uint8_t* sb = sa + kABytes;
          mbar_expect_tx(&full[s], (uint32_t)ld_bytes);
          const int k0 = (kb0 + kb) * KE;
          // row-segmented B (one weight matrix per snapshot block of 128-row tiles)
          const int boff = seg_of_mtile ? seg_of_mtile[m0 / BM] * b_seg_rows : 0;
          // stacked A: rows >= a2_row0 come from the second operand
          const CUtensorMap* mA = m0 >= a2_row0 ? &tmA2 : &tmA;
          const int am0 = (int)(m0 >= a2_row0 ? m0 - a2_row0 : m0);
          if (!A_MN) {
            tma_load_2d(sa, mA, k0, am0, &full[s]);
          } else if (F16) {
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_2d(sa + i * 8192, mA, am0 + 64 * i, k0, &full[s]);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 32; ++i)
              tma_load_2d(sa + i * 4096, mA, am0 + 32 * i, k0, &full[s]);
          }
          if (!b_res) {
            if (!B_MN) {
              tma_load_2d(sb, &tmB, k0, (int)n0 + boff, &full[s]);
            } else if (F16) {
              for (int i = 0; i < bn / 64; ++i)
                tma_load_2d(sb + i * 8192, &tmB, (int)n0 + 64 * i, k0 + boff, &full[s]);
            } else {
              for (int i = 0; i < bn / 32; ++i)
                tma_load_2d(sb + i * 4096, &tmB, (int)n0 + 32 * i, k0 + boff, &full[s]);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = F16 ? idesc_f16mn(bn, A_MN, B_MN) : idesc_tf32(bn, A_MN, B_MN);
    if (b_res) {
      mbar_wait(bres_full, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    int g = 0, i = 0;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++i) {
      int64_t m0, n0;
      int z, kb0, nkb;
      tile_coords(t, m0, n0, z, kb0, nkb);
      const int a = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      mbar_wait(&tempty[a], aph ^ 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t tacc = tmem_base + (uint32_t)a * acc_cols;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int s = g % stages;
        const uint32_t ph = (g / stages) & 1;
        mbar_wait(SPLIT3 ? &conv[s] : &full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (lane == 0) {
          const uint32_t sa = smem_u32(smem + (size_t)s * (b_res ? kABytes : stage_bytes));
          const uint32_t sb = b_res ? smem_u32(bres + (size_t)(kb0 + kb) * b_bytes) : sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            if (F16) {
              // K = 16 per MMA: K-major 32 B inside the 128-B swizzle row;
              // MN-major 16 k-rows (two 1-KB SWIZZLE_128B atoms) per MMA, 64-element
              // MN chunks 8 KB apart
              const uint32_t ao = A_MN ? kk * 2048 : kk * 32;
              const uint32_t bo = B_MN ? kk * 2048 : kk * 32;
              const uint64_t ad = A_MN ? sdesc(sa + ao, 8192, 1024, 2) : kdesc(sa + ao);
              const uint64_t bd = B_MN ? sdesc(sb + bo, 8192, 1024, 2) : kdesc(sb + bo);
              mma_f16(tacc, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
              continue;
            }
            // K-major: advance 32 B inside the 128-B swizzle row; MN-major: eight
            // k-rows (two 512-B atoms, 1024 B) per MMA, MN chunks 4096 B apart.
            const uint32_t ao = A_MN ? kk * 1024 : kk * 32;
            const uint32_t bo = B_MN ? kk * 1024 : kk * 32;
            const uint64_t ad = A_MN ? mndesc(sa + ao) : kdesc(sa + ao);
            const uint64_t bd = B_MN ? mndesc(sb + bo) : kdesc(sb + bo);
            mma_tf32(tacc, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
            if (SPLIT3) {
              const uint64_t adl = A_MN ? mndesc(sa + ab_bytes + ao) : kdesc(sa + ab_bytes + ao);
              const uint64_t bdl = B_MN ? mndesc(sb + ab_bytes + bo) : kdesc(sb + ab_bytes + bo);
              mma_tf32(tacc, ad, bdl, idesc, 1u);
              mma_tf32(tacc, adl, bd, idesc, 1u);
            }
          }
          mma_commit(&empty[s]);
          if (kb == nkb - 1) mma_commit(&tfull[a]);
        }
        __syncwarp();
      }
    }
  } else {
    const int tq = threadIdx.x - 64;  // 0..32*kEpiWarps-1
    const int chalf = (warp - 2) >> 2;  // first 32-column chunk of this warp
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    float* stg = stg_base + (warp - 2) * 32 * 33;
    int g = 0, i = 0;
    int box_seq = 0;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++i) {
      int64_t m0, n0;
      int z, kb0, nkb;
      tile_coords(t, m0, n0, z, kb0, nkb);
      if (SPLIT3) {
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&full[s], ph);
          float4* hi = reinterpret_cast<float4*>(smem + (size_t)s * stage_bytes);
          float4* lo = reinterpret_cast<float4*>(smem + (size_t)s * stage_bytes + ab_bytes);
          for (int e = tq; e < ab_bytes / 16; e += 32 * kEpiWarps) {
            const float4 x = hi[e];
            float4 h, l;
            h.x = __uint_as_float(to_tf32(x.x));
            h.y = __uint_as_float(to_tf32(x.y));
            h.z = __uint_as_float(to_tf32(x.z));
            h.w = __uint_as_float(to_tf32(x.w));
            l.x = x.x - h.x;
            l.y = x.y - h.y;
            l.z = x.z - h.z;
            l.w = x.w - h.w;
            hi[e] = h;
            lo[e] = l;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&conv[s]);
        }
      }
      const int a = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      // mask_boxes: the fp16 ReLU mask of this warp's chunks arrives by TMA
      // ([32 rows x 32 cols] SWIZZLE_64B boxes, the output boxes' layout) under
      // the accumulator wait; thread-per-row loads of it cost ~18 us per
      // 200000 x 128 launch (32 row segments per warp load)
      uint8_t* mbox = reinterpret_cast<uint8_t*>(stg_base) + (size_t)kEpiWarps * tma_store * 4096 +
                      (size_t)(warp - 2) * mask_boxes * 2048;
      if (relu16 && mask_boxes) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();  // the previous tile's mask reads are done
        if (lane == 0) {
          int nbx = 0;
          for (int c = 32 * chalf; c < bn; c += 32 * (kEpiWarps / 4)) ++nbx;
          mbar_arrive_expect_tx(&mfull[warp - 2], (uint32_t)nbx * 2048u);
          int ci = 0;
          for (int c = 32 * chalf; c < bn; c += 32 * (kEpiWarps / 4), ++ci)
            tma_load_2d(mbox + ci * 2048, &tmR, (int)(n0 + c), (int)(m0 + q * 32), &mfull[warp - 2]);
        }
      }
      if ((relu_src || (relu16 && !mask_boxes)) && tma_store) {
        // this thread's row of the ReLU mask streams into L1 while the tile's
        // MMAs finish (thread = row; its chunks of the tile's columns)
        const int64_t row = m0 + q * 32 + lane;
        if (row < M)
          for (int c = 32 * chalf; c < bn; c += 32 * (kEpiWarps / 4))
            if (n0 + c < N) {
              if (relu_src) asm volatile("prefetch.global.L1 [%0];" ::"l"(relu_src + row * ldc + n0 + c));
              else asm volatile("prefetch.global.L1 [%0];" ::"l"(relu16 + row * ldr16 + n0 + c));
            }
      }
      mbar_wait(&tfull[a], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (tma_store) {
        // TMEM -> registers (thread = row) [+ bias] -> this warp's SWIZZLE_128B
        // staging box [32 rows x 32 cols] -> one TMA store per chunk (the copy
        // engine writes the tile; the epilogue never issues global stores).
        // tma_store = number of 4 KB boxes per warp (2: ping-pong, a chunk never
        // waits for the previous chunk's store to leave shared memory)
        for (int c = 32 * chalf; c < bn; c += 32 * (kEpiWarps / 4), ++box_seq) {
          uint8_t* box = reinterpret_cast<uint8_t*>(
              stg_base + ((warp - 2) * tma_store + (box_seq % tma_store)) * 1024);
          float v[32];
          tmem_ld32(tmem_base + (uint32_t)a * acc_cols + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
          if (F16) {
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] *= alpha;
          }
          const int64_t nb = n0 + c;
          if (bias) {
            if (nb + 32 <= N && (reinterpret_cast<uintptr_t>(bias + nb) & 15) == 0) {
              // 8 broadcast 16-B loads (every lane reads the same 32 values)
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias + nb) + j);
                v[4 * j] += b4.x; v[4 * j + 1] += b4.y; v[4 * j + 2] += b4.z; v[4 * j + 3] += b4.w;
              }
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u) v[u] += (nb + u < N) ? __ldg(bias + nb + u) : 0.f;
            }
          }
          if (out_act & 1) {
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = fmaxf(v[u], 0.f);
          }
          if (out_act & 2) {
#pragma unroll
            for (int u = 0; u < 32; ++u) v[u] = dgc::rna_tf32_f(v[u]);
          }
          const int64_t row = m0 + q * 32 + lane;
          if (relu16 && mask_boxes) {  // this chunk's box (zero-filled outside the matrix)
            if (c == 32 * chalf) mbar_wait(&mfull[warp - 2], (uint32_t)(i & 1));
            const uint8_t* mb = mbox + ((c - 32 * chalf) / (32 * (kEpiWarps / 4))) * 2048;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 m = *reinterpret_cast<const uint4*>(mb + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4));
              const uint32_t q4[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&q4[k]));
                if (!(f.x > 0.f)) v[8 * j + 2 * k] = 0.f;
                if (!(f.y > 0.f)) v[8 * j + 2 * k + 1] = 0.f;
              }
            }
          } else if (relu16 && row < M) {  // fp16 mask source: 64-B row segment
            const uint4* rs = reinterpret_cast<const uint4*>(relu16 + row * ldr16 + nb);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const uint4 m = (nb + 8 * j < N) ? __ldg(rs + j) : make_uint4(0u, 0u, 0u, 0u);
              const uint32_t q[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&q[k]));
                if (!(f.x > 0.f)) v[8 * j + 2 * k] = 0.f;
                if (!(f.y > 0.f)) v[8 * j + 2 * k + 1] = 0.f;
              }
            }
          }
          if (relu_src || colsum_partial) {
            // ReLU mask from the forward activation (thread = row, 128-B row segment)
            const bool rok = row < M;
            if (relu_src) {
              const float4* rs = reinterpret_cast<const float4*>(relu_src + row * ldc + nb);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 m = (rok && nb + 4 * j < N) ? __ldg(rs + j) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (!(m.x > 0.f)) v[4 * j] = 0.f;
                if (!(m.y > 0.f)) v[4 * j + 1] = 0.f;
                if (!(m.z > 0.f)) v[4 * j + 2] = 0.f;
                if (!(m.w > 0.f)) v[4 * j + 3] = 0.f;
              }
            }
            if (colsum_partial) {
              // column sums of this warp's 32 rows: butterfly transpose-reduction
              // (31 shuffles; lane u ends with column u), fixed order
              float x[32];
#pragma unroll
              for (int u = 0; u < 32; ++u) x[u] = rok ? v[u] : 0.f;
#pragma unroll
              for (int sft = 16; sft >= 1; sft >>= 1) {
                const bool up = (lane & sft) != 0;
#pragma unroll
                for (int i = 0; i < sft; ++i) {
                  const float send = up ? x[i] : x[i + sft];
                  const float keep = up ? x[i + sft] : x[i];
                  x[i] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
                }
              }
              if (nb + lane < N) colsum_partial[((m0 / BM) * 4 + q) * N + nb + lane] = x[0];
            }
          }
          if (C16 && C && row < M) {  // fp16 copy beside C (thread = row, direct stores)
            __half* o = C16 + row * ldc16 + nb;
            if (nb + 32 <= N) {
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                __half2 h[4];
#pragma unroll
                for (int k = 0; k < 4; ++k)
                  h[k] = __floats2half2_rn(v[8 * j + 2 * k] * c16_scale, v[8 * j + 2 * k + 1] * c16_scale);
                *reinterpret_cast<uint4*>(o + 8 * j) = *reinterpret_cast<const uint4*>(h);
              }
            } else {
#pragma unroll
              for (int u = 0; u < 32; ++u)  // (unrolled: v stays in registers)
                if (nb + u < N) o[u] = __float2half_rn(v[u] * c16_scale);
            }
          }
          if (lane == 0) {  // the store that last used this box has read it
            if (tma_store == 2) bulk_wait_read<1>();
            else bulk_wait_read<0>();
          }
          __syncwarp();
          if (!C) {  // fp16-only output: a [32 rows x 64 B] SWIZZLE_64B box, one TMA store
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              __half2 h[4];
#pragma unroll
              for (int k = 0; k < 4; ++k)
                h[k] = __floats2half2_rn(v[8 * j + 2 * k] * c16_scale, v[8 * j + 2 * k + 1] * c16_scale);
              *reinterpret_cast<uint4*>(box + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
                  *reinterpret_cast<const uint4*>(h);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(&tmC, box, (int)(n0 + c), (int)(m0 + q * 32));
              bulk_commit();
            }
            continue;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(box + sw128_offset(lane, 4 * j)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            // split-K / K-segmented partials: tile z writes rows z*M + m (M % 128 == 0)
            tma_store_2d(&tmC, box, (int)(n0 + c), (int)(z * c_rows_per_z + m0 + q * 32));
            bulk_commit();
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&tempty[a]);
        continue;
      }
      // TMEM -> registers (thread = row) -> padded smem transpose -> coalesced
      // 128-byte row stores (lane = column), epilogue fused into the store pass.
      for (int c = 32 * chalf; c < bn; c += 32 * (kEpiWarps / 4)) {
        float v[32];
        tmem_ld32(tmem_base + (uint32_t)a * acc_cols + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
#pragma unroll
        for (int u = 0; u < 32; ++u) stg[lane * 33 + u] = F16 ? v[u] * alpha : v[u];
        __syncwarp();
        const int64_t n = n0 + c + lane;
        const bool col_ok = (c + lane < bn) && (n < N);
        const float bn_v = (bias && col_ok) ? __ldg(bias + n) : 0.f;
        float csum = 0.f;  // this warp's 32 rows of column n (bias gradients)
#pragma unroll 1
        for (int r0 = 0; r0 < 32; r0 += 8) {
          float x[8], aux[8], acc_in[8];
          bool ok[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int64_t row = m0 + q * 32 + r0 + u;
            ok[u] = col_ok && row < M;
            x[u] = stg[(r0 + u) * 33 + lane];
            aux[u] = (ok[u] && relu_src) ? relu_src[row * ldc + n] : 1.f;
            acc_in[u] = (ok[u] && accumulate && !partial) ? C[row * ldc + n] : 0.f;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (!ok[u]) continue;
            const int64_t row = m0 + q * 32 + r0 + u;
            if (partial) {
              partial[((int64_t)z * M + row) * N + n] = x[u];
            } else {
              float y = x[u] + acc_in[u] + bn_v;
              if (relu_src && !(aux[u] > 0.f)) y = 0.f;
              if (out_act & 1) y = fmaxf(y, 0.f);
              if (out_act & 2) y = dgc::rna_tf32_f(y);
              C[row * ldc + n] = y;
              if (C16) C16[row * ldc16 + n] = __float2half_rn(y * c16_scale);
              csum += y;
            }
          }
        }
        if (colsum_partial && col_ok)
          colsum_partial[((m0 / BM) * 4 + q) * N + n] = csum;
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[a]);
    }
  }
  if (tma_store && warp >= 2 && lane == 0) bulk_wait<0>();  // stores complete before exit
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
  }
}

// Split-K reduction, fixed order. Block = 64 float4 column groups x 16 split
// slices: thread (g, s) sums splits s, s+16, ... of 4 consecutive elements
// (16-B loads, unrolled by 4), the 16 slices are then combined in order through
// shared memory. The small weight gradients (128 x 16, 128 x 128 over ~143
// splits) were latency-bound at 4 slices (13-14 us per launch). Needs N % 4 == 0.
constexpr int kRedSlices = 16;  // split slices per element quad (one 64 x 16 block)
__global__ void __launch_bounds__(64 * kRedSlices) splitk_reduce4_kernel(
    const float* __restrict__ partial, int splits, int64_t M, int64_t N, float* __restrict__ C,
    int64_t ldc, const float* __restrict__ bias, const float* __restrict__ relu_src,
    int accumulate) {
  __shared__ float4 red[kRedSlices][64];
  const int64_t total4 = M * N / 4;
  const int64_t e4 = (int64_t)blockIdx.x * 64 + threadIdx.x;
  const int sl = threadIdx.y;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e4 < total4) {
    const float4* p4 = reinterpret_cast<const float4*>(partial);
    // unrolled: the loads of 4 splits are in flight together (the sums keep
    // their sequential order)
#pragma unroll 4
    for (int z = sl; z < splits; z += kRedSlices) {
      const float4 v = __ldg(p4 + (int64_t)z * total4 + e4);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
  }
  red[sl][threadIdx.x] = acc;
  __syncthreads();
  if (sl != 0 || e4 >= total4) return;
  float4 t = red[0][threadIdx.x];
  for (int k = 1; k < kRedSlices; ++k) {
    const float4 v = red[k][threadIdx.x];
    t.x += v.x; t.y += v.y; t.z += v.z; t.w += v.w;
  }
  const int64_t e = e4 * 4, r = e / N, n = e % N;  // 4 elements of one row (N % 4 == 0)
  float o[4] = {t.x, t.y, t.z, t.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    float* dst = C + r * ldc + n + k;
    float a = o[k];
    if (accumulate) a += *dst;
    if (bias) a += bias[n + k];
    if (relu_src && !(relu_src[r * ldc + n + k] > 0.f)) a = 0.f;
    *dst = a;
  }
}

__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int splits, int64_t M,
                                     int64_t N, float* __restrict__ C, int64_t ldc,
                                     const float* __restrict__ bias,
                                     const float* __restrict__ relu_src, int accumulate) {
  const int64_t total = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, n = i % N;
    float acc = 0.f;
    for (int zz = 0; zz < splits; ++zz) acc += partial[(int64_t)zz * total + i];
    float* dst = C + r * ldc + n;
    if (accumulate) acc += *dst;
    if (bias) acc += bias[n];
    if (relu_src && !(relu_src[r * ldc + n] > 0.f)) acc = 0.f;
    *dst = acc;
  }
}

// out[s] = sum of the partials of segment s's work items, fixed order.
__global__ void seg_reduce_kernel(const float* __restrict__ partial, const int32_t* __restrict__ item_ptr,
                                  int n_seg, int64_t M, int64_t N, float* __restrict__ C,
                                  int64_t ldc) {
  const int64_t per = M * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < per * n_seg;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int sg = (int)(i / per);
    const int64_t e = i % per, r = e / N, n = e % N;
    float acc = 0.f;
    for (int z = item_ptr[sg]; z < item_ptr[sg + 1]; ++z) acc += partial[(int64_t)z * per + e];
    C[((int64_t)sg * M + r) * ldc + n] = acc;
  }
}

struct SegOpts {
  const int32_t* seg_of_mtile = nullptr;  // row-segmented B
  int b_seg_rows = 0;
  int b_nseg = 1;
  const int32_t* kitems = nullptr;        // K-segmented items (kb0, nkb)
  int n_kitems = 0;
  const int32_t* item_ptr = nullptr;      // items of each segment
  int n_seg = 0;
  const float* a2 = nullptr;              // stacked A: rows [a2_row0, M) of op(A)
  int64_t lda2 = 0;
  int64_t a2_row0 = 0;
};

int g_max_ctas = 0;  // 0: every SM (dgc_gemm_max_ctas)

template <bool A_MN, bool B_MN, bool SPLIT3, bool F16 = false>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc, int tma_store,
                int64_t c_rows_per_z, const CUtensorMap& ma2, int64_t a2_row0,
                float* C, int64_t ldc, int64_t M,
                int64_t N, int bn, int ntiles, int kb_total, int splits, int kb_per,
                const float* bias, const float* relu_src, int accumulate, float* partial,
                float* colsum_partial, const SegOpts& so, cudaStream_t s, float alpha = 1.f,
                __half* C16 = nullptr, int64_t ldc16 = 0, float c16_scale = 1.f,
                const __half* relu16 = nullptr, int64_t ldr16 = 0) {
  const int ab = kABytes + bn * BK * 4;
  const int stage_bytes = ab * (SPLIT3 ? 2 : 1);
  // shared memory: pipeline stages (+ resident B panel) + the epilogue staging
  // (8 x 4 KB TMA-store boxes, or 8 padded 32x33 transpose tiles) + alignment
  // and barriers, within the 227 KB per-CTA limit
  int stg_bytes = tma_store ? kEpiWarps * 4096 : kEpiWarps * 32 * 33 * 4;
  // fp16 ReLU mask by TMA: one 2 KB box per 32-column chunk of each epilogue warp
  const int mask_boxes = (relu16 && tma_store && !getenv("DGC_GEMM_NO_MASK_TMA")) ? (bn + 63) / 64 : 0;
  const int mask_bytes = kEpiWarps * mask_boxes * 2048;
  CUtensorMap mr = mc;
  if (mask_boxes) {
    const int rc = make_map_f16_sw64(&mr, relu16, M, N, ldr16, 32, 32);
    if (rc) return rc;
  }
  const int budget = 232448 - 1024 - 512 - 1024 - stg_bytes - mask_bytes;
  // B panel resident in shared memory when one CTA keeps one n-tile and it fits
  const int bres_bytes = kb_total * bn * BK * 4;
  int bres_max = 96 * 1024;
  if (const char* env = getenv("DGC_GEMM_BRES_KB")) bres_max = atoi(env) * 1024;
  const int b_res = (!SPLIT3 && splits == 1 && bres_bytes <= bres_max && bres_bytes + 2 * kABytes <= budget &&
                     !so.seg_of_mtile &&
                     !so.kitems && !getenv("DGC_GEMM_NO_BRES")) ? 1 : 0;
  int stages = b_res ? (budget - bres_bytes) / kABytes : budget / stage_bytes;
  int max_stages = 4;
  if (const char* env = getenv("DGC_GEMM_MAX_STAGES")) {
    const int cap = atoi(env);
    if (cap >= 1) max_stages = cap;
  }
  stages = stages > max_stages ? max_stages : stages;
  if (stages < 1) return dgc::fail(DGC_ERR_ARG, "gemm: tile does not fit shared memory");
  const size_t pipe = (size_t)stages * (b_res ? kABytes : stage_bytes) + (b_res ? (size_t)bres_bytes : 0);
  // a second TMA-store box per warp when it fits beside the pipeline
  if (tma_store && pipe + 1024 + 512 + 1024 + 2 * stg_bytes + mask_bytes <= 232448 &&
      !getenv("DGC_GEMM_ONE_BOX")) {
    tma_store = 2;
    stg_bytes *= 2;
  }
  const size_t smem = pipe + 1024 + 512 + 1024 + stg_bytes + mask_bytes;
  auto kern = gemm_tf32_kernel<A_MN, B_MN, SPLIT3, F16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "gemm: set smem");
  const int m_tiles = (int)((M + BM - 1) / BM);
  const int total = m_tiles * ntiles * splits;
  // multiple of n_tiles: fixed n per CTA; g_max_ctas caps it for GEMMs that
  // run concurrently with another one (dgc_gemm_max_ctas)
  const int sms = g_max_ctas > 0 && g_max_ctas < dgc::kNumSMs ? g_max_ctas : dgc::kNumSMs;
  int grid = (sms / ntiles) * ntiles;
  if (grid < ntiles) grid = ntiles;
  if (grid > total) grid = total;
  kern<<<grid, kThreads, smem, s>>>(ma, mb, mc, tma_store, c_rows_per_z, mr, mask_boxes, ma2, a2_row0, C, ldc, M, N, bn, stages, kb_total, kb_per, m_tiles,
                                    ntiles, splits, bias, relu_src, accumulate, partial,
                                    colsum_partial, b_res, so.seg_of_mtile, so.b_seg_rows,
                                    so.kitems, alpha, C16, ldc16, c16_scale, relu16, ldr16);
  DGC_CHECK_LAUNCH("gemm_tf32_kernel");
  return DGC_OK;
}

}  // namespace

extern "C" int32_t dgc_gemm_max_ctas(int32_t n) {
  const int32_t prev = g_max_ctas;
  g_max_ctas = n > 0 ? n : 0;
  return prev;
}

extern "C" int dgc_gemm_splits(int64_t K, int32_t precision, int32_t k_splits) {
  const int KE = precision == 2 ? 64 : BK;
  const int kb_total = (int)((K + KE - 1) / KE);
  if (k_splits < 1) k_splits = 1;
  int kb_per = (kb_total + k_splits - 1) / k_splits;
  if (precision == 3 && kb_per > 16) kb_per = 16;
  return kb_per > 0 ? (kb_total + kb_per - 1) / kb_per : 1;
}

// K == 0 (a device that owns no rows: its weight-gradient contractions are
// empty): C = (accumulate ? C : 0) + bias, then the epilogue's ReLU mask /
// output activation, exactly as the tensor-core epilogue would apply them.
__global__ void gemm_k0_kernel(float* C, int64_t ldc, int64_t M, int64_t N, const float* bias,
                               const float* relu_src, int accumulate, int out_act) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < M * N;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / N, c = i % N;
    float v = accumulate ? C[r * ldc + c] : 0.f;
    if (bias) v += bias[c];
    if (relu_src && !(relu_src[r * N + c] > 0.f)) v = 0.f;
    if (out_act & 1) v = fmaxf(v, 0.f);
    if (out_act & 2) v = dgc::rna_tf32_f(v);
    C[r * ldc + c] = v;
  }
}

static int gemm_impl(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                     int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn, int32_t b_mn,
                     int32_t precision, const float* bias, const float* relu_src,
                     int32_t accumulate, int32_t k_splits, float* partial, float* colsum_partial,
                     const SegOpts& so, void* stream, float alpha = 1.f, void* C16 = nullptr,
                     int64_t ldc16 = 0, float c16_scale = 1.f, const void* relu16 = nullptr,
                     int64_t ldr16 = 0) {
  DGC_REQUIRE(M >= 0 && N >= 0 && K >= 0, "gemm: bad shape");
  const int out_act = (accumulate >> 1) & 3;  // bit 1 ReLU, bit 2 TF32-round the output
  accumulate &= 1;
  if (K == 0) {
    if (M == 0 || N == 0) return DGC_OK;
    DGC_REQUIRE(colsum_partial == nullptr && so.seg_of_mtile == nullptr && so.kitems == nullptr,
                "gemm: K == 0 supports plain / bias / ReLU-mask epilogues only");
    gemm_k0_kernel<<<dgc::grid_for(M * N, 256), 256, 0, dgc::as_stream(stream)>>>(
        C, ldc, M, N, bias, relu_src, accumulate, out_act);
    DGC_CHECK_LAUNCH("gemm_k0_kernel");
    return DGC_OK;
  }
  DGC_REQUIRE(precision >= 1 && precision <= 3,
              "gemm: precision must be 1 (TF32), 2 (fp16 operands) or 3 (3xTF32)");
  const bool f16 = precision == 2;  // A, B are fp16 (the pointers' element type)
  const int KE = f16 ? 64 : BK;     // elements per k-block
  DGC_REQUIRE(!f16 || (!so.seg_of_mtile && !so.kitems), "gemm: fp16 operands: plain / stacked-A only");
  DGC_REQUIRE(k_splits >= 1, "gemm: k_splits >= 1");
  if (M == 0 || N == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int align = b_mn ? (f16 ? 64 : 32) : 16;
  const int ntiles = (int)((N + 255) / 256);
  int bn = (int)((N + ntiles - 1) / ntiles);
  bn = (bn + align - 1) / align * align;
  if (bn > 256) bn = 256;
  const int kb_total = (int)((K + KE - 1) / KE);
  // split-K only to fill the machine: ~one wave of (m-tile, n-tile, split) work
  // items (the split-K partials cost 2 x splits x M x N x 4 bytes of traffic)
  {
    const int64_t tiles = ((M + BM - 1) / BM) * ntiles;
    const int64_t cap = tiles >= dgc::kNumSMs ? 1 : dgc::kNumSMs / tiles;
    if (k_splits > cap) k_splits = (int)cap;
  }
  int kb_per = (kb_total + k_splits - 1) / k_splits;
  // The tcgen05 fp32 accumulator truncates (measured: a systematic -1.2e-4
  // relative bias after 625 k-blocks of 3xTF32, tools/debug_gemm.py), so the
  // fp32-parity mode caps every TMEM accumulation chain at kMaxChainKb k-blocks
  // and finishes the sum in the round-to-nearest split-K reduction.
  constexpr int kMaxChainKb = 16;
  if (precision == 3 && kb_per > kMaxChainKb) kb_per = kMaxChainKb;
  const int splits = so.kitems ? so.n_kitems : (kb_total + kb_per - 1) / kb_per;
  if (splits > 1 || so.kitems)
    DGC_REQUIRE(partial != nullptr, "gemm: split-K / K-segmented items need a partial buffer");
  if (splits > 1) DGC_REQUIRE(colsum_partial == nullptr, "gemm: column sums need k_splits == 1");
  CUtensorMap ma, mb;
  // A / A2 / B maps: fp32 (TF32) or fp16 boxes
  auto map_a = [&](CUtensorMap* m, const float* p, int64_t rows, int64_t ld) {
    if (f16)
      return a_mn ? make_map_f16(m, p, K, rows, ld, 64, 64) : make_map_f16(m, p, rows, K, ld, 64, BM);
    return a_mn ? make_map(m, p, K, rows, ld, 32, 32, true) : make_map(m, p, rows, K, ld, 32, BM, false);
  };
  int rc = map_a(&ma, A, M, lda);
  if (rc) return rc;
  CUtensorMap ma2 = ma;
  int64_t a2_row0 = INT64_MAX;
  if (so.a2) {
    DGC_REQUIRE(so.a2_row0 > 0 && so.a2_row0 % BM == 0 && so.a2_row0 < M,
                "gemm: stacked A needs a 128-aligned split row inside M");
    a2_row0 = so.a2_row0;
    rc = map_a(&ma2, so.a2, M - a2_row0, so.lda2);
    if (rc) return rc;
    rc = map_a(&ma, A, a2_row0, lda);
    if (rc) return rc;
  }
  const int64_t nseg = so.b_nseg > 0 ? so.b_nseg : 1;
  rc = f16 ? (b_mn ? make_map_f16(&mb, B, K * nseg, N, ldb, 64, 64)
                   : make_map_f16(&mb, B, N * nseg, K, ldb, 64, (uint32_t)bn))
           : b_mn ? make_map(&mb, B, K * nseg, N, ldb, 32, 32, true)
                  : make_map(&mb, B, N * nseg, K, ldb, 32, (uint32_t)bn, false);
  if (rc) return rc;
  float* part = (splits > 1 || so.kitems) ? partial : nullptr;
  DGC_REQUIRE(!(part && out_act), "gemm: an output activation needs an unsplit K");
  DGC_REQUIRE(!(part && (C16 || relu16)), "gemm: fp16 outputs / masks need an unsplit K");
  DGC_REQUIRE(C || C16 || M == 0 || N == 0, "gemm: no output");
  DGC_REQUIRE(!C16 || (ldc16 % 8 == 0 && (reinterpret_cast<uintptr_t>(C16) & 15) == 0),
              "gemm: the fp16 output needs 16-byte aligned rows");
  DGC_REQUIRE(!relu16 || (ldr16 % 8 == 0 && (reinterpret_cast<uintptr_t>(relu16) & 15) == 0 &&
                          !relu_src && !accumulate),
              "gemm: the fp16 ReLU mask needs 16-byte aligned rows (and no fp32 mask / accumulate)");
  const bool s3 = precision == 3;
  // plain / bias-only outputs leave through TMA stores (box 32 cols x 32 rows)
  CUtensorMap mc;
  int tma_store = 0;
  int64_t c_rows_per_z = 0;
  if (!part && !C) {
    // fp16-only output: the row path (thread = row) and TMA stores of
    // [32 x 32] fp16 boxes (SWIZZLE_64B) from the per-warp staging box
    rc = make_map_f16_sw64(&mc, C16, M, N, ldc16, 32, 32);
    if (rc) return rc;
    tma_store = 1;
  } else if (relu16) {
    DGC_REQUIRE(!part, "gemm: the fp16 ReLU mask needs an unsplit K");
    tma_store = make_map(&mc, C, M, N, ldc, 32, 32, false) == DGC_OK ? 1 : 0;
    DGC_REQUIRE(tma_store, "gemm: the fp16 ReLU mask needs a TMA-storable C");
  } else if (!getenv("DGC_GEMM_NO_TMA_STORE")) {
    if (!part) {
      tma_store = (!accumulate && ((ldc * 4) % 16 == 0) && (!relu_src || N % 4 == 0)) ? 1 : 0;
      if (tma_store && make_map(&mc, C, M, N, ldc, 32, 32, false) != DGC_OK) tma_store = 0;
    } else if (M % BM == 0 && N % 4 == 0) {
      // partial tiles [items x M, N]: a tile never crosses into the next item
      const int64_t items = so.kitems ? so.n_kitems : splits;
      tma_store = make_map(&mc, part, items * M, N, N, 32, 32, false) == DGC_OK ? 1 : 0;
      c_rows_per_z = M;
    }
  }
  if (so.kitems && splits == 0) {
    rc = DGC_OK;
  } else {
#define DGC_GEMM_CASE4(AM, BMN, S3, F)                                                           \
  if ((bool)a_mn == AM && (bool)b_mn == BMN && s3 == S3 && f16 == F)                              \
    rc = launch_gemm<AM, BMN, S3, F>(ma, mb, mc, tma_store, c_rows_per_z, ma2, a2_row0, C, ldc,  \
                                     M, N, bn, ntiles,                                           \
                                     kb_total,                                                   \
                                     splits, kb_per,                                             \
                                     part ? nullptr : bias, part ? nullptr : relu_src,           \
                                     part ? 0 : (accumulate | (out_act << 1)), part,             \
                                     colsum_partial, so, s, alpha, static_cast<__half*>(C16), ldc16,  \
                                     c16_scale, static_cast<const __half*>(relu16), ldr16);
#define DGC_GEMM_CASE(AM, BMN, S3) DGC_GEMM_CASE4(AM, BMN, S3, false)
    DGC_GEMM_CASE4(false, false, false, true)
    DGC_GEMM_CASE4(false, true, false, true)
    DGC_GEMM_CASE4(true, false, false, true)
    DGC_GEMM_CASE4(true, true, false, true)
    DGC_GEMM_CASE(false, false, false)
    DGC_GEMM_CASE(false, true, false)
    DGC_GEMM_CASE(true, false, false)
    DGC_GEMM_CASE(true, true, false)
    DGC_GEMM_CASE(false, false, true)
    DGC_GEMM_CASE(false, true, true)
    DGC_GEMM_CASE(true, false, true)
    DGC_GEMM_CASE(true, true, true)
#undef DGC_GEMM_CASE
#undef DGC_GEMM_CASE4
  }
  if (rc) return rc;
  if (so.kitems) {
    seg_reduce_kernel<<<dgc::grid_for(M * N * so.n_seg, 256), 256, 0, s>>>(
        part, so.item_ptr, so.n_seg, M, N, C, ldc);
    DGC_CHECK_LAUNCH("seg_reduce_kernel");
  } else if (part) {
    if (N % 4 == 0 && (reinterpret_cast<uintptr_t>(part) & 15) == 0) {
      const int64_t total4 = M * N / 4;
      splitk_reduce4_kernel<<<(unsigned)((total4 + 63) / 64), dim3(64, kRedSlices), 0, s>>>(
          part, splits, M, N, C, ldc, bias, relu_src, accumulate);
    } else {
      splitk_reduce_kernel<<<dgc::grid_for(M * N, 256), 256, 0, s>>>(part, splits, M, N, C, ldc,
                                                                     bias, relu_src, accumulate);
    }
    DGC_CHECK_LAUNCH("splitk_reduce_kernel");
  }
  return DGC_OK;
}

extern "C" int dgc_gemm_tf32(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                             int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn,
                             int32_t b_mn, int32_t precision, const float* bias,
                             const float* relu_src, int32_t accumulate, int32_t k_splits,
                             float* partial, float* colsum_partial, void* stream) {
  return gemm_impl(A, lda, B, ldb, C, ldc, M, N, K, a_mn, b_mn, precision, bias, relu_src,
                   accumulate, k_splits, partial, colsum_partial, SegOpts{}, stream);
}

extern "C" int dgc_gemm_tf32_segmented(const float* A, int64_t lda, const float* B, int64_t ldb,
                                       float* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                                       int32_t a_mn, int32_t b_mn, int32_t precision,
                                       const float* bias, const float* relu_src,
                                       const int32_t* seg_of_mtile, int32_t b_nseg,
                                       const int32_t* kitems, int32_t n_kitems,
                                       const int32_t* item_ptr, int32_t n_seg, float* partial,
                                       float* colsum_partial, int32_t act, void* stream) {
  DGC_REQUIRE(!(seg_of_mtile && kitems), "gemm_segmented: row- and K-segmentation are exclusive");
  // stacked per-segment B: a 32-row TMA box must not run into the next matrix
  DGC_REQUIRE(!seg_of_mtile || (b_mn ? K % 32 == 0 : N % 16 == 0),
              "gemm_segmented: row-segmented B needs K % 32 == 0 (MN-major) / N % 16 == 0");
  SegOpts so;
  so.seg_of_mtile = seg_of_mtile;
  so.b_nseg = b_nseg > 0 ? b_nseg : 1;
  so.b_seg_rows = seg_of_mtile ? (int)(b_mn ? K : N) : 0;
  so.kitems = kitems;
  so.n_kitems = n_kitems;
  so.item_ptr = item_ptr;
  so.n_seg = n_seg;
  return gemm_impl(A, lda, B, ldb, C, ldc, M, N, K, a_mn, b_mn, precision, bias, relu_src,
                   (act & 3) << 1, 1, partial, colsum_partial, so, stream);
}

extern "C" int dgc_gemm_tf32_stacked_a(const float* A0, int64_t lda0, const float* A1, int64_t lda1,
                                       int64_t M0, const float* B, int64_t ldb, float* C,
                                       int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn,
                                       int32_t b_mn, int32_t precision, int32_t k_splits,
                                       float* partial, void* stream) {
  SegOpts so;
  so.a2 = A1;
  so.lda2 = lda1;
  so.a2_row0 = M0;
  return gemm_impl(A0, lda0, B, ldb, C, ldc, M, N, K, a_mn, b_mn, precision, nullptr, nullptr, 0,
                   k_splits, partial, nullptr, so, stream);
}

extern "C" int dgc_gemm_f16(const void* A, int64_t lda, const void* B, int64_t ldb, float* C,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn, int32_t b_mn,
                            float alpha, const float* bias, const float* relu_src, int32_t accumulate,
                            int32_t k_splits, float* partial, float* colsum_partial, void* C16,
                            int64_t ldc16, float c16_scale, const void* relu16, int64_t ldr16,
                            void* stream) {
  return gemm_impl(static_cast<const float*>(A), lda, static_cast<const float*>(B), ldb, C, ldc, M,
                   N, K, a_mn, b_mn, 2, bias, relu_src, accumulate, k_splits, partial,
                   colsum_partial, SegOpts{}, stream, alpha, C16, ldc16, c16_scale, relu16, ldr16);
}

extern "C" int dgc_gemm_f16_stacked_a(const void* A0, int64_t lda0, const void* A1, int64_t lda1,
                                      int64_t M0, const void* B, int64_t ldb, float* C, int64_t ldc,
                                      int64_t M, int64_t N, int64_t K, int32_t a_mn, int32_t b_mn,
                                      float alpha, int32_t k_splits, float* partial, void* stream) {
  SegOpts so;
  so.a2 = static_cast<const float*>(A1);
  so.lda2 = lda1;
  so.a2_row0 = M0;
  return gemm_impl(static_cast<const float*>(A0), lda0, static_cast<const float*>(B), ldb, C, ldc, M,
                   N, K, a_mn, b_mn, 2, nullptr, nullptr, 0, k_splits, partial, nullptr, so, stream,
                   alpha);
}
