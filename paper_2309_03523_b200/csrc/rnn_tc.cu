// K3/K4 on tensor cores: persistent tcgen05 masked LSTM forward (TF32).
//
// Same semantics as dgc_rnn_fwd (rnn.cu, the reference form of
// gru_forward_masked, fusion.py:428-469, carried to the LSTM): a CTA owns a tile
// of 128 FFD-packed rows for all L positions. Per position p:
//   MMA   : acc[128, 4H] = h_in[128, H] x U[H, 4H]  (tcgen05.mma.kind::tf32, A =
//           the h tile in shared memory (K-major SWIZZLE_128B, written by the
//           epilogue), B = U^T streamed by TMA through a 2-stage ring, fp32 TMEM
//           accumulator of 4H <= 512 columns);
//   epi   : 4 warps (thread = packed row = TMEM lane) read the gates 16 units at a
//           time (tcgen05.ld 32x32b.x16), add the precomputed x Wx + b row of the
//           slot's instance, update c/h, store h|c / the backward save, and write
//           the NEXT position's masked h_in (carry mask, or the cross-device carry
//           at a run start) straight into the swizzled A tile.
// The input projection x Wx + b of all slots is one K2 GEMM ahead of this kernel.
#include <cuda_fp16.h>

#include <type_traits>

#include "tc_common.cuh"

namespace {

// Compact save row of the H = 128 cluster kernels (forward writes, BPTT and
// the weight-gradient GEMM read), all fp16: [h_in (H) | c_in (H) | i, f, g, o
// interleaved per unit (4 H: unit j at halves 2H + 4j .. +3)] = 3 H floats
// per instance (1536 B at H = 128). fp16 keeps the 10 explicit mantissa bits of
// the TF32 path's operands (h_in is fp16-exact by construction, gates in (0,1)
// / (-1,1), |c| <= L); h_in is the fp16 A operand of [dWx; dU] = [x; h_in]^T
// dgx, and interleaving the gates makes a BPTT lane's four units one 32-B load
// and the forward's one 32-B store.
template <int H> __host__ __device__ constexpr int tc_save_floats() {
  return H == 128 ? 3 * H : 7 * H;
}
__device__ __forceinline__ uint32_t h2u(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void sth4(__half* p, float4 v) {
  *reinterpret_cast<uint2*>(p) = make_uint2(h2u(v.x, v.y), h2u(v.z, v.w));
}
// the gates of 4 consecutive units, interleaved: 32 B at p (16-B aligned)
__device__ __forceinline__ void st_ifgo(__half* p, float4 i, float4 f, float4 g, float4 o) {
  uint4* q = reinterpret_cast<uint4*>(p);
  q[0] = make_uint4(h2u(i.x, f.x), h2u(g.x, o.x), h2u(i.y, f.y), h2u(g.y, o.y));
  q[1] = make_uint4(h2u(i.z, f.z), h2u(g.z, o.z), h2u(i.w, f.w), h2u(g.w, o.w));
}
// round to the nearest fp16 (exactly representable in TF32 too, in range)
__device__ __forceinline__ float f16r(float x) { return __half2float(__float2half_rn(x)); }
__device__ __forceinline__ float2 u2h(uint32_t u) {
  return __half22float2(*reinterpret_cast<const __half2*>(&u));
}

using namespace dgc::tc;
using dgc::make_map;
using dgc::make_gather_map;
using dgc::make_gather_map_f16;

// warp 0 TMA, warp 1 MMA + TMEM, warps 2..9 epilogue: 2 warps per TMEM lane
// quadrant (32 packed rows), each owning H/2 hidden units.
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;
constexpr int kStages = 2;     // B ring: one (k-block, 256-column part) of U^T per stage
constexpr int kChunk = 16;     // units per TMEM load / smem transpose
constexpr int kStgStride = 17; // padded row stride of the transpose buffer (floats)
constexpr int kStgFloats = 4 * 32 * kStgStride;  // 4 gates x 32 rows per warp
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// sigmoid(x) = 0.5 * tanh(x/2) + 0.5 (one MUFU op)
__device__ __forceinline__ float sigm(float x) { return fmaf(0.5f, tanh_fast(0.5f * x), 0.5f); }
__device__ __forceinline__ float rna_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Per-position timestamps of CTA 0 (ns, globaltimer) for tools/time_lstm_*.py:
// [p][0] MMA issue start, [p][1] accumulator ready, [p][2] epilogue done.
// Compiled in only with -DDGC_LSTM_TIMESTAMPS (make DGC_TS=1): the production
// kernels carry no probe.
__device__ unsigned long long g_lstm_ts[256][8];
__device__ unsigned long long g_lstm_ts2[256][8];  // forward chunk-0 internals
__device__ unsigned long long g_lstm_ts3[256][32];  // BPTT: each epilogue warp's last chunk done
#ifdef DGC_LSTM_TIMESTAMPS
#define DGC_TS(cond, p, k) \
  do {                     \
    if (cond) g_lstm_ts[p][k] = globaltimer(); \
  } while (0)
#define DGC_TS2(cond, p, k) \
  do {                      \
    if (cond) g_lstm_ts2[p][k] = globaltimer(); \
  } while (0)
#define DGC_TS3(cond, p, k) \
  do {                      \
    if (cond) g_lstm_ts3[p][k] = globaltimer(); \
  } while (0)
#else
#define DGC_TS3(cond, p, k) \
  do {                      \
  } while (0)
#define DGC_TS(cond, p, k) \
  do {                     \
  } while (0)
#define DGC_TS2(cond, p, k) \
  do {                      \
  } while (0)
#endif

template <int H>
__global__ void __launch_bounds__(kThreads, 1)
    lstm_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmUt, const float* __restrict__ gx,
                       const int32_t* __restrict__ slot_row, const uint8_t* __restrict__ slot_mask,
                       const int32_t* __restrict__ slot_carry, const float* __restrict__ carry,
                       int64_t R, int L, int64_t ld, float* __restrict__ h_out,
                       float* __restrict__ c_out, float* __restrict__ save) {
  constexpr int G4 = 4 * H;
  constexpr int KB = H / BK;                 // k-blocks of the h operand
  constexpr int kABytes = KB * BM * 128;     // h tile (K-major SWIZZLE_128B)
  constexpr int kNPart = G4 > 256 ? 256 : G4;
  constexpr int kNParts = G4 / kNPart;
  constexpr int kBStage = kNPart * 128;      // kNPart rows of U^T x 32 k
  constexpr int kUnits = H / 2;              // units per epilogue warp
  constexpr uint32_t kTmemCols = G4 <= 128 ? 128 : G4 <= 256 ? 256 : 512;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived from the __shared__ array (keeps shared-space
  // addressing: STS/LDS instead of generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + kABytes;
  float* stg_all = reinterpret_cast<float*>(sB + kStages * kBStage);
  uint64_t* b_full = reinterpret_cast<uint64_t*>(stg_all + kEpiWarps * kStgFloats);
  uint64_t* b_empty = b_full + kStages;
  uint64_t* a_full = b_empty + kStages;
  uint64_t* acc_full = a_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    mbar_init(a_full, kEpiThreads);
    mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmUt) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  constexpr int kUnitsPerStep = KB * kNParts;  // B stages per position

  if (warp == 0) {
    if (lane == 0) {
      for (int g = 0; g < L * kUnitsPerStep; ++g) {
        const int s = g % kStages;
        mbar_wait(&b_empty[s], ((g / kStages) & 1) ^ 1);
        const int kb = (g % kUnitsPerStep) / kNParts, part = g % kNParts;
        mbar_expect_tx(&b_full[s], (uint32_t)kBStage);
        tma_load_2d(sB + s * kBStage, &tmUt, kb * BK, part * kNPart, &b_full[s]);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_tf32(kNPart, false, false);
    const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
    for (int p = 0; p < L; ++p) {
      mbar_wait(a_full, p & 1);
      fence_after();
      DGC_TS(blockIdx.x == 0 && lane == 0 && p < 256, p, 0);
      for (int u = 0; u < kUnitsPerStep; ++u) {
        const int g = p * kUnitsPerStep + u;
        const int s = g % kStages;
        const int kb = u / kNParts, part = u % kNParts;
        mbar_wait(&b_full[s], (g / kStages) & 1);
        fence_after();
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t ad = kdesc(a_base + kb * BM * 128 + kk * 32);
            const uint64_t bd = kdesc(b_base + s * kBStage + kk * 32);
            mma_tf32(tmem_base + part * kNPart, ad, bd, idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit(&b_empty[s]);
          if (u == kUnitsPerStep - 1) mma_commit(acc_full);
        }
        __syncwarp();
      }
    }
  } else {
    // Epilogue. TMEM rows are packed rows (thread = row for tcgen05.ld); every
    // 16-unit chunk is transposed through shared memory so that global traffic
    // runs with lanes = (2 rows x 16 units): each gx / h / c / save access is a
    // contiguous 64-byte row segment instead of 32 scattered rows.
    const int ew = warp - 2;
    const int q = warp & 3;                 // TMEM lane quadrant
    const int u_lo = (ew >> 2) * kUnits;    // this warp's unit range
    float* stg = stg_all + ew * kStgFloats;
    const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
    const int uu = lane & 15, rr = lane >> 4;  // lane -> (row parity, unit)
    auto a_ptr = [&](int r, int k) {
      return reinterpret_cast<float*>(sA + (k / BK) * BM * 128 + sw128_offset(r, k % BK));
    };
    // prologue: h_in of position 0 (run start: carry or zero)
    for (int it = 0; it < 16; ++it) {
      const int r = q * 32 + it * 2 + rr;
      const int64_t row = row0 + r;
      const int ci = row < R ? slot_carry[row * L] : -1;
      for (int j = u_lo + uu; j < u_lo + kUnits; j += 16)
        *a_ptr(r, j) = ci >= 0 ? rna_tf32(carry[(int64_t)ci * 2 * H + j]) : 0.f;
    }
    fence_async_smem();
    mbar_arrive(a_full);
    for (int p = 0; p < L; ++p) {
      const bool has_next = p + 1 < L;
      // per-row slot info of this warp's 32 rows, one row per lane (issued before
      // the accumulator wait so the loads overlap the MMA); broadcast by shuffle
      const int64_t my_row = row0 + q * 32 + lane;
      const bool my_ok = my_row < R;
      const int64_t my_s = my_row * L + p;
      const int my_inst = my_ok ? slot_row[my_s] : -1;
      const bool my_mk = my_ok && slot_mask[my_s];
      const int my_ci = my_ok ? slot_carry[my_s] : -1;
      const int my_prev = (p > 0 && my_mk) ? slot_row[my_s - 1] : -1;
      const float my_mnext = (has_next && my_ok) ? (float)slot_mask[my_s + 1] : 0.f;
      const int my_cnext = (has_next && my_ok) ? slot_carry[my_s + 1] : -1;
      mbar_wait(acc_full, p & 1);
      fence_after();
      DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 1);
#pragma unroll 1
      for (int j0 = u_lo; j0 < u_lo + kUnits; j0 += kChunk) {
        // TMEM (thread = row) -> smem [gate][row][unit]
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) {
          float a[16];
          tmem_ld16(tl + gi * H + j0, a);
#pragma unroll
          for (int u = 0; u < 16; ++u) stg[(gi * 32 + lane) * kStgStride + u] = a[u];
        }
        __syncwarp();
        const int j = j0 + uu;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          // issue every global load of 8 row pairs first (memory-level parallelism)
          float xg[8][4], cin[8];
          int inst[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int rl = (half * 8 + t) * 2 + rr;
            inst[t] = __shfl_sync(0xffffffffu, my_inst, rl);
            const int ci = __shfl_sync(0xffffffffu, my_ci, rl);
            const int prev = __shfl_sync(0xffffffffu, my_prev, rl);
            const float* gr = gx + (int64_t)max(inst[t], 0) * G4 + j;
#pragma unroll
            for (int gi = 0; gi < 4; ++gi) xg[t][gi] = inst[t] >= 0 ? __ldg(gr + gi * H) : 0.f;
            cin[t] = ci >= 0 ? carry[(int64_t)ci * 2 * H + H + j]
                             : (prev >= 0 ? c_out[(int64_t)prev * ld + j] : 0.f);
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int rl = (half * 8 + t) * 2 + rr;
            const int r = q * 32 + rl;
            const float m_next = __shfl_sync(0xffffffffu, my_mnext, rl);
            const int c_next = __shfl_sync(0xffffffffu, my_cnext, rl);
            const float hin = *a_ptr(r, j);
            float hn = 0.f;
            if (inst[t] >= 0) {
              const float ig = sigm(stg[(0 * 32 + rl) * kStgStride + uu] + xg[t][0]);
              const float fg = sigm(stg[(1 * 32 + rl) * kStgStride + uu] + xg[t][1]);
              const float gg = tanh_fast(stg[(2 * 32 + rl) * kStgStride + uu] + xg[t][2]);
              const float og = sigm(stg[(3 * 32 + rl) * kStgStride + uu] + xg[t][3]);
              const float cn = fg * cin[t] + ig * gg;
              const float tc = tanh_fast(cn);
              hn = rna_tf32(og * tc);
              float* sv = save + (int64_t)inst[t] * 7 * H + j;
              sv[0] = hin;
              sv[H] = cin[t];
              sv[2 * H] = ig;
              sv[3 * H] = fg;
              sv[4 * H] = gg;
              sv[5 * H] = og;
              sv[6 * H] = tc;
              h_out[(int64_t)inst[t] * ld + j] = hn;
              c_out[(int64_t)inst[t] * ld + j] = cn;
            }
            if (has_next)
              *a_ptr(r, j) = c_next >= 0 ? rna_tf32(carry[(int64_t)c_next * 2 * H + j]) : hn * m_next;
          }
        }
        __syncwarp();
      }
      DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 2);
      if (has_next) {
        fence_before();
        fence_async_smem();
        mbar_arrive(a_full);
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

// Forward, 2-CTA cluster, vectorised epilogue (16 warps = 4 per TMEM lane
// quadrant, 8 rows each). A lane owns one row and 4 consecutive units of a
// 16-unit chunk (lane = 8 rows x 4 unit quads), so every global / shared / DSMEM
// access is a 16-byte vector and the per-row slot info is loaded per lane (no
// shuffles). The carried c stays in shared memory per lane (same cells at every
// position); the next chunk's gx loads are issued before the current chunk's math.
constexpr int kVEW = 16;
// Row tiling of the 2-CTA cluster kernels: a cluster owns 4 x rq packed rows
// (rq per TMEM lane quadrant, rows q*32 + [0, rq) of its 128-row MMA tile) with
// rq = ceil(R / (4 * 74)) <= 32, so R rows spread over <= 74 clusters = 148 SMs.
inline int cluster_rows_per_quadrant(int64_t R) {
  const int64_t per = (R + 4 * (dgc::kNumSMs / 2) - 1) / (4 * (dgc::kNumSMs / 2));
  return (int)(per < 1 ? 1 : per > 32 ? 32 : per);
}
inline int64_t cluster_tiles(int64_t R) {
  const int64_t rows = 4 * (int64_t)cluster_rows_per_quadrant(R);
  return (R + rows - 1) / rows;
}
__device__ __forceinline__ float4 f4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ float4 zero4() { return make_float4(0.f, 0.f, 0.f, 0.f); }

// FX (fused input projection): the gate pre-activations x Wx + h U + b are
// accumulated in TMEM from two operand pairs per position -- the x rows of the
// position's packed slots, gathered by TMA (tile::gather4, rows given by
// slot_row) against Wx^T, then the h tile against U^T -- into double-buffered
// accumulators (2 x 256 columns), so the x part of position p+1 runs while the
// epilogue drains position p. The gx GEMM and every per-position global load of
// the epilogue disappear; the bias is added from L1.
// FX accumulator column order: inside each 16-unit chunk, TMEM column k holds
// unit 4 (k/2 % 4) + 2 (k >= 8) + (k & 1), so the 16x256b TMEM load hands lane
// (row r, unit quad uq) exactly units 4 uq .. 4 uq + 3 of its row (columns
// 2 uq, 2 uq + 1, 8 + 2 uq, 9 + 2 uq): the epilogue reads its gates straight
// from TMEM, with no shared-memory staging. Applied to both B operands (U^T, Wx^T).
__host__ __device__ constexpr int fx_unit(int col) {
  return (col & ~15) + 4 * ((col & 7) >> 1) + ((col & 8) ? 2 : 0) + (col & 1);
}
template <int H, int kVEW, bool FX>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * kVEW, 1)
    lstm_fwd_tc2v_kernel(const __grid_constant__ CUtensorMap tmUt,
                         const __grid_constant__ CUtensorMap tmWxT,
                         const __grid_constant__ CUtensorMap tmX, const float* __restrict__ bias,
                         const float* __restrict__ gx,
                         const int32_t* __restrict__ slot_row, const uint8_t* __restrict__ slot_mask,
                         const int32_t* __restrict__ slot_carry, const float* __restrict__ carry,
                         int64_t R, int L, int64_t ld, float* __restrict__ h_out,
                         float* __restrict__ c_out, float* __restrict__ save, int rq,
                         const float* __restrict__ Uw, const float* __restrict__ Wxw,
                         __half* __restrict__ h16, int hends) {
  constexpr int kEpiT = 32 * kVEW;
  constexpr int G4 = 4 * H;
  constexpr int HU = H / 2;
  constexpr int NCH = HU / 16;               // 16-unit chunks per CTA
  constexpr int NP = 4 * HU;
  constexpr int KB = H / BK;
  // FX (F = H = 128): every operand of the gate product is fp16 (kind::f16,
  // the same 10-bit mantissa as TF32): the h tile (2 k-blocks of 64 units), the
  // x rows TMA-gathered from an fp16 copy of the layer input, and this CTA's
  // halves of U^T and Wx^T, resident in shared memory for the whole launch --
  // no weight bytes move per position (streaming them was the recurrence's
  // critical path: all 148 SMs re-read the same 256 KB every position).
  constexpr int kABytes = FX ? 2 * BM * 128 : KB * BM * 128;
  constexpr int kWBytes = FX ? 2 * NP * 128 : 0;  // one resident fp16 weight half: 2 k-blocks
  constexpr int kBStages = FX ? 0 : kStages;
  constexpr int kBStage = NP * 128;
  constexpr int kXStages = FX ? 1 : kStages;
  // staging [gate][8 rows][16 units] per warp, all 4 gates at once or (the
  // 16-warp fp16 variant, to fit its shared memory) 2 at a time
  constexpr int kStgGates = (FX && kVEW > 12) ? 2 : 4;
  constexpr int kStgW = kStgGates * 8 * 16;
  constexpr uint32_t kAccCols = NP <= 128 ? 128 : 256;
  constexpr uint32_t kTmemCols = FX ? 2 * kAccCols : kAccCols;
  constexpr int kXStage = BM * 128;          // one x k-block: 128 rows x 128 B
  static_assert(!FX || H == 128, "fused input projection: F = H = 128");
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived from the __shared__ array (keeps shared-space
  // addressing: STS/LDS instead of generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sU = smem + kABytes;              // FX: resident U^T half (fp16)
  uint8_t* sW = sU + kWBytes;                // FX: resident Wx^T half (fp16)
  uint8_t* sB = sW + kWBytes;
  uint8_t* sX = sB + kBStages * kBStage;     // FX: x k-block ring
  float* stg_all = reinterpret_cast<float*>(sX + (FX ? kXStages * kXStage : 0));
  float* c_all = stg_all + kVEW * kStgW;     // carried c: [warp][chunk][lane] float4
  uint64_t* b_full = reinterpret_cast<uint64_t*>(c_all + kVEW * NCH * 32 * 4);
  uint64_t* b_empty = b_full + kStages;
  // h-tile readiness: FX (double-buffered accumulators) splits it into two
  // halves -- units {0-31, 64-95} (both CTAs' first 32 units) and {32-63,
  // 96-127} -- so the h U^T MMA of p+1 starts on the first half while the
  // epilogues of p finish
  constexpr int kHalves = (FX && KB == 4) ? 2 : 1;
  uint64_t* a_full = b_empty + kStages;      // [2]
  uint64_t* acc_full = a_full + 2;           // [2] (FX: per accumulator)
  uint64_t* acc_empty = acc_full + 2;        // [2] FX
  uint64_t* x_full = acc_empty + 2;          // [kStages] FX
  uint64_t* x_empty = x_full + kStages;      // [kStages] FX
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(x_empty + kStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank(), peer = crank ^ 1u;
  // the cluster's packed rows: rq per TMEM lane quadrant (rq <= 32), so the
  // recurrence spreads over ~all SMs instead of R/128 tiles
  const int64_t row0 = (int64_t)(blockIdx.x >> 1) * 4 * rq;
  const int u0 = (int)crank * HU;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    // local epilogue threads arrive (CTA scope); the peer's half of the h tile
    // lands by st.async (complete_tx), expected by one local arrive.expect_tx
    // one arrival per epilogue warp (lane 0 after the warp's proxy fences and a
    // __syncwarp): 384 per-thread arrivals on one mbarrier serialise for ~0.4 us
    mbar_init(&a_full[0], kVEW);
    mbar_init(&a_full[1], kVEW);
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 2);  // both CTAs' MMAs (multicast commit)
      mbar_init(&acc_empty[a], kVEW);
    }
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&x_full[st], 1);
      mbar_init(&x_empty[st], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmUt) : "memory");
    if (FX) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmWxT) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&tmX) : "memory");
    }
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  fence_before();
  __syncthreads();
  cluster_sync_all();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  DGC_TS3(blockIdx.x == 0 && threadIdx.x == 64, 2, 30);

  if (warp == 0) {
    if (!FX) {
      if (lane == 0) {
        for (int g = 0; g < L * KB; ++g) {
          const int s = g % kStages;
          mbar_wait(&b_empty[s], ((g / kStages) & 1) ^ 1);
          const int kb = g % KB;
          mbar_expect_tx(&b_full[s], (uint32_t)kBStage);
#pragma unroll
          for (int gi = 0; gi < 4; ++gi)
            tma_load_2d(sB + s * kBStage + gi * HU * 128, &tmUt, kb * BK, gi * H + u0, &b_full[s]);
        }
      }
    } else {
      // per position: 4 x k-blocks (x rows gathered, Wx^T), then 4 h k-blocks (U^T).
      // Lane g < 4 * ceil(rq/4) gathers rows [4i, 4i+4) of lane quadrant g / ceil(rq/4).
      const int gpq = (rq + 3) / 4;                // gathers per lane quadrant
      const int n_g = 4 * gpq;
      const uint32_t x_bytes = (uint32_t)n_g * 4u * 128u;
      const int gq = lane / gpq, gi0 = (lane % gpq) * 4;
      int gxs = 0;                                 // x-ring sequence number
      for (int p = 0; p < L; ++p) {
        int idx[4] = {0, 0, 0, 0};
        if (lane < n_g) {
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = gi0 + e;
            const int64_t prow = row0 + (int64_t)gq * rq + i;
            const int inst = (i < rq && prow < R) ? slot_row[prow * L + p] : -1;
            idx[e] = inst >= 0 ? inst : 0;  // padding slots read row 0 (result unused)
          }
        }
        // the position's x rows: 2 fp16 k-blocks of 64 units (weights are resident)
        for (int kb = 0; kb < 2; ++kb, ++gxs) {
          const int sx = gxs % kXStages;
          if (lane == 0) {
            mbar_wait(&x_empty[sx], ((gxs / kXStages) & 1) ^ 1);
            mbar_expect_tx(&x_full[sx], x_bytes);
          }
          __syncwarp();
          if (lane < n_g)
            tma_gather4(sX + sx * kXStage + (gq * 32 + gi0) * 128, &tmX, kb * 64, idx[0], idx[1],
                        idx[2], idx[3], &x_full[sx]);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_tf32(NP, false, false);
    const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB), x_base = smem_u32(sX);
    int g = 0, gxs = 0;
    for (int p = 0; p < L; ++p) {
      const int ab = FX ? (p & 1) : 0;
      const uint32_t tacc = tmem_base + ab * kAccCols;
      if (FX) {
        mbar_wait(&acc_empty[ab], ((p >> 1) & 1) ^ 1);  // epilogue of p-2 drained it
        fence_after();
        if (p == 0) {  // the resident weights were written by the epilogue warps
          mbar_wait(&a_full[0], 0);
          fence_after();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        const uint32_t w_base = smem_u32(sW), idesc16 = idesc_f16(NP);
        for (int kb = 0; kb < 2; ++kb, ++gxs) {
          const int sx = gxs % kXStages;
          mbar_wait(&x_full[sx], (gxs / kXStages) & 1);
          fence_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_f16(tacc, kdesc(x_base + sx * kXStage + kk * 32),
                      kdesc(w_base + kb * NP * 128 + kk * 32), idesc16, (kb > 0 || kk > 0) ? 1u : 0u);
            mma_commit(&x_empty[sx]);
          }
          __syncwarp();
        }
        DGC_TS(blockIdx.x == 0 && lane == 0 && p < 256, p, 6);
      }
      if (FX) {
        // h part: fp16 h tile x resident fp16 U^T; half h = the 16-unit slices
        // kk = 2h, 2h+1 of both 64-unit k-blocks
        const uint32_t u_base = smem_u32(sU);
        const uint32_t idesc16 = idesc_f16(NP);
        for (int h = 0; h < 2; ++h) {
          mbar_wait(&a_full[h], p & 1);
          fence_after();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          DGC_TS(h == 0 && blockIdx.x == 0 && lane == 0 && p < 256, p, 0);
          if (lane == 0) {
#pragma unroll
            for (int kb16 = 0; kb16 < 2; ++kb16)
#pragma unroll
              for (int kk = 2 * h; kk < 2 * h + 2; ++kk)
                mma_f16(tacc, kdesc(a_base + kb16 * BM * 128 + kk * 32),
                        kdesc(u_base + kb16 * NP * 128 + kk * 32), idesc16, 1u);
            if (h == 1) mma_commit_mc(&acc_full[ab], (uint16_t)0x3);
          }
          __syncwarp();
        }
        continue;
      }
      for (int i = 0; i < KB; ++i, ++g) {
        const int kb = kHalves == 2 ? (i >> 1) + 2 * (i & 1) : i;  // 0, 2, 1, 3
        if (i % (KB / kHalves) == 0) {
          mbar_wait(&a_full[i / (KB / kHalves)], p & 1);
          fence_after();
          // generic-proxy writes (local st.shared, peer st.async) -> async proxy (MMA)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          DGC_TS(i == 0 && blockIdx.x == 0 && lane == 0 && p < 256, p, 0);
        }
        const int s = g % kStages;
        mbar_wait(&b_full[s], (g / kStages) & 1);
        fence_after();
        DGC_TS(i == 2 && blockIdx.x == 0 && lane == 0 && p < 256, p, 7);
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk)
            mma_tf32(tacc, kdesc(a_base + kb * BM * 128 + kk * 32),
                     kdesc(b_base + s * kBStage + kk * 32), idesc,
                     (FX || i > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&b_empty[s]);
          if (i == KB - 1) mma_commit_mc(&acc_full[ab], (uint16_t)0x3);
        }
        __syncwarp();
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;                  // TMEM lane quadrant (warp id % 4)
    const int rb = (ew >> 2) * 8;            // first quadrant row of this warp
    const int r8 = lane >> 2, uq = lane & 3;
    const int r = q * 32 + rb + r8;          // tile (TMEM lane / A) row of this lane
    const int64_t grow = row0 + q * rq + rb + r8;
    const bool ok = rb + r8 < rq && grow < R;
    const bool active = rb < rq;             // warps with no rows only keep the protocol
    const uint32_t stg = smem_u32(stg_all + ew * kStgW);             // byte addresses
    const uint32_t creg = smem_u32(c_all + (ew * NCH * 32 + lane) * 4);  // + ch * 512
    const uint32_t sA_s = smem_u32(sA);
    const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
    const uint32_t sA_peer = map_peer(sA, peer);
    const uint32_t afull_peer = map_peer(a_full, peer);
    // h-tile address of unit k of this lane's row: fp32 k-blocks of 32 units,
    // or (FX) fp16 k-blocks of 64 units; both K-major SWIZZLE_128B
    auto a_off = [&](int k) {
      if (FX)
        return (uint32_t)((k >> 6) * BM * 128 + r * 128 + ((((k & 63) >> 3) ^ (r & 7)) << 4) +
                          (k & 7) * 2);
      return (uint32_t)((k / BK) * BM * 128) + sw128_offset(r, k % BK);
    };
    // unit k of this CTA lies in h-tile half (k - u0) / 32 (kHalves == 2)
    auto put_h = [&](int k, float4 v) {
      const uint32_t off = a_off(k);
      const uint32_t half = kHalves == 2 ? (uint32_t)((k - u0) >> 5) : 0u;
      if (FX) {
        const uint2 hv = make_uint2(h2u(v.x, v.y), h2u(v.z, v.w));
        asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(sA_s + off), "r"(hv.x), "r"(hv.y)
                     : "memory");
        st_async_v2(sA_peer + off, hv, afull_peer + half * 8u);
      } else {
        sts4(sA_s + off, v);
        st_async_v4(sA_peer + off, v, afull_peer + half * 8u);
      }
    };
    auto get_h = [&](int k) {  // this lane's 4 units of the h tile (as the MMA reads them)
      if (FX) {
        uint32_t a, b;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(sA_s + a_off(k)));
        const float2 lo = u2h(a), hi = u2h(b);
        return make_float4(lo.x, lo.y, hi.x, hi.y);
      }
      return lds4(sA_s + a_off(k));
    };
    // bytes of the peer's half of the h tile it writes into ours: 8 rows x HU
    // units per active warp (4 quadrants x ceil(rq / 8) warps)
    const uint32_t kPeerBytes = 4u * (uint32_t)((rq + 7) / 8) * 8u * HU * (FX ? 2u : 4u);
    if (FX) {
      // this CTA's halves of U^T and Wx^T (B row n = gate column (n / HU) * H +
      // u0 + fx_unit(n % HU), K = the H input units) as fp16, K-major
      // SWIZZLE_128B, read straight from U and Wx [H, 4H]: an item is 8 input
      // units x 4 consecutive gate columns (eight 16-B loads, coalesced across
      // the warp), transposed in registers into four 16-B B-row segments;
      // resident for the whole launch, ordered before the first MMA by the
      // prologue's a_full arrival
      constexpr int kQuads = NP / 4;  // gate-column quads of this CTA
#pragma unroll 2
      for (int c = threadIdx.x - 64; c < 2 * (H / 8) * kQuads; c += kEpiT) {
        const int qd = c % kQuads, kg = (c / kQuads) % (H / 8), mat = c / (kQuads * (H / 8));
        const int g = qd / (HU / 4), j0 = 4 * (qd % (HU / 4));  // gate, first own unit
        const int k0 = kg * 8;
        const float* src = (mat ? Wxw : Uw) + (int64_t)k0 * G4 + g * H + u0 + j0;
        float4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = ldg4(src + (int64_t)i * G4);
        // units j0 + e sit in B rows g HU + (j0 & ~15) + {2p, 2p+1, 8+2p, 9+2p} (fx_unit)
        const int p4 = (j0 & 15) >> 2, nb = g * HU + (j0 & ~15);
        const int rows[4] = {nb + 2 * p4, nb + 2 * p4 + 1, nb + 8 + 2 * p4, nb + 9 + 2 * p4};
        const uint32_t base = smem_u32(mat ? sW : sU) + (uint32_t)((k0 >> 6) * NP * 128);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          auto el = [&](const float4& f) { return e == 0 ? f.x : e == 1 ? f.y : e == 2 ? f.z : f.w; };
          const int n = rows[e];
          const uint32_t dst = base + (uint32_t)(n * 128 + ((((k0 & 63) >> 3) ^ (n & 7)) << 4));
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst),
                       "r"(h2u(el(v[0]), el(v[1]))), "r"(h2u(el(v[2]), el(v[3]))),
                       "r"(h2u(el(v[4]), el(v[5]))), "r"(h2u(el(v[6]), el(v[7])))
                       : "memory");
        }
      }
    }
    auto publish = [&](int half) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (ew == 0) mbar_arrive_expect_tx(&a_full[half], kPeerBytes / kHalves);
        else mbar_arrive(&a_full[half]);
      }
    };
    auto drained = [&](int ab) {  // this warp has read accumulator ab
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
    };
    auto publish_all = [&]() {
      for (int h = 0; h < kHalves; ++h) publish(h);
    };
    // prologue: h_in of position 0 (run start: carry or zero)
    if (active) {
      const int ci = ok ? slot_carry[grow * L] : -1;
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        const int j = u0 + ch * 16 + uq * 4;
        float4 v = zero4();
        if (ci >= 0) {
          v = f4(carry + (int64_t)ci * 2 * H + j);
          if (!FX) v = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
        }
        put_h(j, v);
        sts4(creg + ch * 512, zero4());
      }
    }
    publish_all();
    DGC_TS3(blockIdx.x == 0 && threadIdx.x == 64, 2, 31);
    int n_inst = ok ? slot_row[grow * L] : -1, n_mk = 0, n_ci = ok ? slot_carry[grow * L] : -1;
    for (int p = 0; p < L; ++p) {
      const bool has_next = p + 1 < L;
      const int inst = n_inst, mk = n_mk, ci = n_ci;
      if (has_next && ok) {
        const int64_t s1 = grow * L + p + 1;
        n_inst = slot_row[s1];
        n_mk = slot_mask[s1];
        n_ci = slot_carry[s1];
      } else {
        n_inst = -1; n_mk = 0; n_ci = -1;
      }
      const float m_next = (float)n_mk;
      const int ab = FX ? (p & 1) : 0;
      const uint32_t acc_par = FX ? ((p >> 1) & 1) : (p & 1);
      if (!active) {  // keep the a_full / acc_empty phase order: step p's MMA done first
        mbar_wait(&acc_full[ab], acc_par);
        if (FX) drained(ab);
        if (has_next) publish_all();
        continue;
      }
      const float* gxr = gx + (int64_t)max(inst, 0) * G4 + u0 + uq * 4;
      float4 xg[4];
#pragma unroll
      for (int gi = 0; gi < 4; ++gi)
        xg[gi] = FX ? ldg4(bias + gi * H + u0 + uq * 4) : (inst >= 0 ? ldg4(gxr + gi * H) : zero4());
      mbar_wait(&acc_full[ab], acc_par);
      fence_after();
      DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 1);
#pragma unroll (FX ? 2 : 1)
      for (int ch = 0; ch < NCH; ++ch) {
        const int c0 = ch * 16;
        const int j = u0 + c0 + uq * 4;
        float4 pre[4];
        const uint32_t ta = tl + ab * kAccCols + c0;
        DGC_TS2(ch == 0 && blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 0);
        // staging row k (64 B) holds its 16-B quads XOR-swizzled by (k >> 1) & 3:
        // the 8 writing lanes and the 8 lanes of every read phase hit 8
        // distinct bank quads (conflict-free both ways)
        auto stage = [&](const float* a, int ng) {
          if (lane >= rb && lane < rb + 8) {
            const int k = lane - rb;
#pragma unroll
            for (int gi = 0; gi < ng; ++gi) {
              const uint32_t d = stg + (gi * 8 + k) * 64;
#pragma unroll
              for (int u = 0; u < 16; u += 4)
                sts4(d + ((((u >> 2) ^ (k >> 1)) & 3) << 4),
                     make_float4(a[gi * 16 + u], a[gi * 16 + u + 1], a[gi * 16 + u + 2],
                                 a[gi * 16 + u + 3]));
            }
          }
          __syncwarp();
        };
        if (FX) {
          // lanes q*32 + (rb & 16) .. +15 of the quadrant; this warp's 8 rows are
          // the lane-L or lane-L+8 half
          float a[16];
          const uint32_t t16 = ta + ((uint32_t)(rb & 16) << 16);
          tmem_ld16x256x4(t16, t16 + HU, t16 + 2 * HU, t16 + 3 * HU, (rb & 8) != 0, a);
#pragma unroll
          for (int gi = 0; gi < 4; ++gi)
            pre[gi] = make_float4(a[4 * gi], a[4 * gi + 1], a[4 * gi + 2], a[4 * gi + 3]);
        } else if (kStgGates == 4) {
          float a[64];
          tmem_ld16x4(ta, ta + HU, ta + 2 * HU, ta + 3 * HU, a);
          DGC_TS2(ch == 0 && blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 1);
          stage(a, 4);
#pragma unroll
          for (int gi = 0; gi < 4; ++gi)
            pre[gi] = lds4(stg + (gi * 8 + r8) * 64 + (((uq ^ (r8 >> 1)) & 3) << 4));
        } else {  // two gates at a time (the 16-warp fp16 variant's shared memory)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float a[32];
            tmem_ld16(ta + (2 * h) * HU, a);
            tmem_ld16(ta + (2 * h + 1) * HU, a + 16);
            stage(a, 2);
#pragma unroll
            for (int gi = 0; gi < 2; ++gi)
              pre[2 * h + gi] = lds4(stg + (gi * 8 + r8) * 64 + (((uq ^ (r8 >> 1)) & 3) << 4));
            __syncwarp();
          }
        }
        DGC_TS2(ch == 0 && blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 2);
        // next chunk's gx in flight while this chunk computes
        float4 xn[4];
#pragma unroll
        for (int gi = 0; gi < 4; ++gi)
          xn[gi] = ch + 1 >= NCH ? zero4()
                   : FX ? ldg4(bias + gi * H + u0 + c0 + 16 + uq * 4)
                        : (inst >= 0 ? ldg4(gxr + gi * H + c0 + 16) : zero4());
        float4 cin = zero4();
        if (ci >= 0) cin = f4(carry + (int64_t)ci * 2 * H + H + j);
        else if (mk) cin = lds4(creg + ch * 512);
        const float4 hin = get_h(j);
        float4 hn = zero4(), cn = zero4();
        if (inst >= 0) {
          float4 ig, fg, gg, og, tc;
#define DGC_LSTM_CELL(c)                                          \
  ig.c = sigm(pre[0].c + xg[0].c);                                \
  fg.c = sigm(pre[1].c + xg[1].c);                                \
  gg.c = tanh_fast(pre[2].c + xg[2].c);                           \
  og.c = sigm(pre[3].c + xg[3].c);                                \
  cn.c = fg.c * cin.c + ig.c * gg.c;                              \
  tc.c = tanh_fast(cn.c);                                         \
  hn.c = FX ? f16r(og.c * tc.c) : rna_tf32(og.c * tc.c);
          DGC_LSTM_CELL(x) DGC_LSTM_CELL(y) DGC_LSTM_CELL(z) DGC_LSTM_CELL(w)
#undef DGC_LSTM_CELL
          DGC_TS2(ch == 0 && blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 3);
          constexpr int kSF = tc_save_floats<H>();
          float* sv = save + (int64_t)inst * kSF + j;
          if (H == 128) {  // compact fp16 row: h_in, c_in, i, f, g, o (the BPTT recomputes tanh(c))
            __half* sh = reinterpret_cast<__half*>(save + (int64_t)inst * kSF);
            sth4(sh + j, hin);
            sth4(sh + H + j, cin);
            st_ifgo(sh + 2 * H + 4 * j, ig, fg, gg, og);
          } else {
            st4(sv, hin);
            st4(sv + H, cin);
            st4(sv + 2 * H, ig);
            st4(sv + 3 * H, fg);
            st4(sv + 4 * H, gg);
            st4(sv + 5 * H, og);
            st4(sv + 6 * H, tc);
          }
          // hends: the fp16 copy is the layer's output; fp32 h only where a run
          // ends (the carries other devices read), like c
          if (!hends || !(has_next && n_mk)) st4(h_out + (int64_t)inst * ld + j, hn);
          if (FX && h16) sth4(h16 + (int64_t)inst * H + j, hn);  // the next layer's fp16 x
          // c leaves the kernel only where a run ends (the carries other devices
          // read); inside a run it lives in creg and in the successor's c_in save
          if (!(has_next && n_mk)) st4(c_out + (int64_t)inst * ld + j, cn);
        }
        DGC_TS2(ch == 0 && blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 4);
        sts4(creg + ch * 512, cn);
        if (has_next) {
          float4 v;
          if (n_ci >= 0) {
            v = f4(carry + (int64_t)n_ci * 2 * H + j);
            if (!FX) v = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
          } else {
            v = make_float4(hn.x * m_next, hn.y * m_next, hn.z * m_next, hn.w * m_next);
          }
          put_h(j, v);
        }
        DGC_TS2(ch == 0 && blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 5);
        // first half of this CTA's units done: the MMA of p+1 may start on it
        if (kHalves == 2 && has_next && ch == NCH / 2 - 1) publish(0);
#pragma unroll
        for (int gi = 0; gi < 4; ++gi) xg[gi] = xn[gi];
        __syncwarp();
        DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && p < 256 && ch < 3, p, 3 + ch);
      }
      DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && p < 256, p, 2);
      if (FX) drained(ab);  // this accumulator is drained
      if (has_next) publish(kHalves - 1);
    }
  }
  DGC_TS3(blockIdx.x == 0 && threadIdx.x == 64, 3, 30);
  fence_before();
  __syncthreads();
  cluster_sync_all();
  DGC_TS3(blockIdx.x == 0 && threadIdx.x == 64, 3, 31);
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

template <int H, int EW, bool FX>
int launch_lstm_tc2v_ew(const CUtensorMap& m, const CUtensorMap& mwx, const CUtensorMap& mx,
                        const float* bias, const float* gx, const int32_t* slot_row,
                        const uint8_t* slot_mask, const int32_t* slot_carry, const float* carry,
                        int64_t R, int L, int64_t ld, float* h_out, float* c_out, float* save,
                        int rq, cudaStream_t s, const float* Uw = nullptr,
                        const float* Wxw = nullptr, __half* h16 = nullptr, int hends = 0) {
  // FX: fp16 h tile + resident fp16 U^T / Wx^T halves + one x stage
  const size_t smem = (FX ? (size_t)2 * BM * 128 + (size_t)2 * 2 * 2 * H * 128 + (size_t)BM * 128
                         : (size_t)(H / BK) * BM * 128 + (size_t)kStages * 2 * H * 128) +
                      (size_t)EW * ((FX && EW > 12) ? 2 : 4) * 8 * 16 * 4 +
                      (size_t)EW * (H / 32) * 32 * 16 + 1024 + 256;
  auto kern = lstm_fwd_tc2v_kernel<H, EW, FX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "lstm_fwd_tc2v: set smem");
  const int grid = 2 * (int)cluster_tiles(R);
  kern<<<grid, 64 + 32 * EW, smem, s>>>(m, mwx, mx, bias, gx, slot_row, slot_mask, slot_carry,
                                        carry, R, L, ld, h_out, c_out, save, rq, Uw, Wxw, h16, hends);
  DGC_CHECK_LAUNCH("lstm_fwd_tc2v_kernel");
  return DGC_OK;
}

// 12 epilogue warps (3 per lane quadrant = 24 rows) when rq <= 24: the idle
// fourth warp's registers go to the others (128 instead of 96 per thread)
template <int H>
int launch_lstm_tc2v(const float* gx, const float* Ut, const int32_t* slot_row,
                     const uint8_t* slot_mask, const int32_t* slot_carry, const float* carry,
                     int64_t R, int L, int64_t ld, float* h_out, float* c_out, float* save,
                     cudaStream_t s) {
  CUtensorMap m;
  int rc = make_map(&m, Ut, 4 * H, H, H, 32, H / 2, false);
  if (rc) return rc;
  const int rq = cluster_rows_per_quadrant(R);
  if (rq <= 24 && !getenv("DGC_RNN_EW16"))
    return launch_lstm_tc2v_ew<H, 12, false>(m, m, m, nullptr, gx, slot_row, slot_mask, slot_carry,
                                             carry, R, L, ld, h_out, c_out, save, rq, s);
  return launch_lstm_tc2v_ew<H, 16, false>(m, m, m, nullptr, gx, slot_row, slot_mask, slot_carry,
                                           carry, R, L, ld, h_out, c_out, save, rq, s);
}

// Fused input projection (H = F = 128): x [n, F] (row stride ldx), WxT [4H, F],
// Ut [4H, H], bias [4H]; no gx.
int launch_lstm_tc2x(const void* x16, int64_t n_x, const float* Wx, const float* U,
                     const float* bias, const int32_t* slot_row, const uint8_t* slot_mask,
                     const int32_t* slot_carry, const float* carry, int64_t R, int L, int64_t ld,
                     float* h_out, float* c_out, float* save, __half* h16, int hends, cudaStream_t s) {
  constexpr int H = 128;
  CUtensorMap mx;  // (the fp32 weight maps of the other instantiations are unused here)
  int rc = make_gather_map_f16(&mx, x16, n_x, H, H);
  if (rc) return rc;
  const int rq = cluster_rows_per_quadrant(R);
  if (rq <= 24 && !getenv("DGC_RNN_EW16"))
    return launch_lstm_tc2v_ew<H, 12, true>(mx, mx, mx, bias, nullptr, slot_row, slot_mask,
                                            slot_carry, carry, R, L, ld, h_out, c_out, save, rq, s,
                                            U, Wx, h16, hends);
  return launch_lstm_tc2v_ew<H, 16, true>(mx, mx, mx, bias, nullptr, slot_row, slot_mask,
                                          slot_carry, carry, R, L, ld, h_out, c_out, save, rq, s, U,
                                          Wx, h16, hends);
}

// ---------------------------------------------------------------------------
// Backward (BPTT) on tensor cores. Per position p, from the last to the first:
//   epi : dh = m(p+1) * acc[(p+1)%2] + dh_out[inst], dc = dc carried (global
//         scratch, per tile row x unit); saved gates -> da (4 gates) -> dgx,
//         bias partial sums, carried dc = dcn * f * m(p); da is written straight
//         into a ring of K-major SWIZZLE_128B A k-blocks (32 gate columns each);
//   MMA : acc[p%2] = da[128, 4H] x U^T  (B = U itself, [H, 4H] K-major, TMA ring)
//         = the gradient w.r.t. h_in(p), consumed by the epilogue of p-1.
// Two TMEM accumulators + an acc_empty barrier let the MMA of p-1 start on the
// first da k-blocks while the epilogue of p is still reading acc[(p+1)%2].
constexpr int kBwdEpiWarps = 8;
constexpr int kBwdEpiThreads = 32 * kBwdEpiWarps;
constexpr int kBwdThreads = 64 + kBwdEpiThreads;
constexpr int kBwdAStages = 8;
constexpr int kBwdBStages = 4;

template <int H>
__global__ void __launch_bounds__(kBwdThreads, 1)
    lstm_bwd_tc_kernel(const __grid_constant__ CUtensorMap tmU, const int32_t* __restrict__ slot_row,
                       const uint8_t* __restrict__ slot_mask, int64_t R, int L,
                       const float* __restrict__ save, const float* __restrict__ dh_out,
                       float* __restrict__ dgx, float* __restrict__ dc_scr, int rnd,
                       float* __restrict__ bias_partial) {
  constexpr int G4 = 4 * H;
  constexpr int NC = H / 32;                 // 32-unit chunks
  constexpr int KB = G4 / BK;                // k-blocks of da per position (= 4*NC)
  constexpr int kAStage = BM * 128;          // 16 KB
  constexpr int kBStage = H * 128;           // H rows of U x 32 k
  constexpr uint32_t kTmemCols = 2 * H <= 32 ? 32 : 2 * H <= 64 ? 64 : 2 * H <= 128 ? 128 : 256;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived from the __shared__ array (keeps shared-space
  // addressing: STS/LDS instead of generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + kBwdAStages * kAStage;
  float* stg_all = reinterpret_cast<float*>(sB + kBwdBStages * kBStage);
  uint64_t* a_full = reinterpret_cast<uint64_t*>(stg_all + kBwdEpiWarps * 32 * 33);
  uint64_t* a_empty = a_full + kBwdAStages;
  uint64_t* b_full = a_empty + kBwdAStages;
  uint64_t* b_empty = b_full + kBwdBStages;
  uint64_t* acc_full = b_empty + kBwdBStages;   // [2]
  uint64_t* acc_empty = acc_full + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = (int64_t)blockIdx.x * BM;
  if (warp == 0 && lane == 0) {
    // a k-block (gate, chunk) is written by the 4 quadrant warps of one half
    for (int s = 0; s < kBwdAStages; ++s) {
      mbar_init(&a_full[s], 128);
      mbar_init(&a_empty[s], 1);
    }
    for (int s = 0; s < kBwdBStages; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], kBwdEpiThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmU) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // k-block sequence per position: i = c*4 + g  (chunk c, gate g), K offset g*H + 32c
  if (warp == 0) {
    if (lane == 0) {
      for (int seq = 0; seq < L * KB; ++seq) {
        const int s = seq % kBwdBStages;
        mbar_wait(&b_empty[s], ((seq / kBwdBStages) & 1) ^ 1);
        const int i = seq % KB, c = i >> 2, g = i & 3;
        mbar_expect_tx(&b_full[s], (uint32_t)kBStage);
        tma_load_2d(sB + s * kBStage, &tmU, g * H + 32 * c, 0, &b_full[s]);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_tf32(H, false, false);
    const uint32_t a_base = smem_u32(sA), b_base = smem_u32(sB);
    for (int t = 0; t < L; ++t) {  // t = L-1-p
      const int p = L - 1 - t;
      const int a = p & 1;
      mbar_wait(&acc_empty[a], ((t >> 1) & 1) ^ 1);
      fence_after();
      for (int i = 0; i < KB; ++i) {
        const int seq = t * KB + i;
        const int sa = seq % kBwdAStages, sb = seq % kBwdBStages;
        mbar_wait(&a_full[sa], (seq / kBwdAStages) & 1);
        mbar_wait(&b_full[sb], (seq / kBwdBStages) & 1);
        fence_after();
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk)
            mma_tf32(tmem_base + a * H, kdesc(a_base + sa * kAStage + kk * 32),
                     kdesc(b_base + sb * kBStage + kk * 32), idesc, (i > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&a_empty[sa]);
          mma_commit(&b_empty[sb]);
          if (i == KB - 1) mma_commit(&acc_full[a]);
        }
        __syncwarp();
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;            // TMEM lane quadrant = rows q*32..q*32+31
    const int half = ew >> 2;          // chunks c with c % 2 == half
    float* stg = stg_all + ew * 32 * 33;
    const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
    const int64_t my_row = row0 + q * 32 + lane;
    const bool my_ok = my_row < R;
    float bsum[(NC + 1) / 2][4];
#pragma unroll
    for (int cc = 0; cc < (NC + 1) / 2; ++cc)
#pragma unroll
      for (int g = 0; g < 4; ++g) bsum[cc][g] = 0.f;
    for (int t = 0; t < L; ++t) {
      const int p = L - 1 - t;
      const bool has_next = p + 1 < L;
      const int64_t my_s = my_row * L + p;
      const int my_inst = my_ok ? slot_row[my_s] : -1;
      const float my_m = my_ok ? (float)slot_mask[my_s] : 0.f;
      const float my_mnext = (has_next && my_ok) ? (float)slot_mask[my_s + 1] : 0.f;
      if (has_next) {
        mbar_wait(&acc_full[(p + 1) & 1], ((t - 1) >> 1) & 1);
        fence_after();
      }
#pragma unroll 1
      for (int c = half, cc = 0; c < NC; c += 2, ++cc) {
        const int j = 32 * c + lane;  // this lane's hidden unit
        if (has_next) {
          float v[32];
          tmem_ld32(tl + ((p + 1) & 1) * H + 32 * c, v);
#pragma unroll
          for (int u = 0; u < 32; ++u) stg[lane * 33 + u] = v[u];
        }
        __syncwarp();
        // acquire the 4 A k-blocks (c, g) of this position
        const int seq0 = t * KB + c * 4;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int seq = seq0 + g;
          mbar_wait(&a_empty[seq % kBwdAStages], ((seq / kBwdAStages) & 1) ^ 1);
        }
#pragma unroll 1
        for (int r0 = 0; r0 < 32; r0 += 8) {
          float ld[8][6], dhv[8], dcv[8];
          int inst[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rl = r0 + u;
            inst[u] = __shfl_sync(0xffffffffu, my_inst, rl);
            const float mn = __shfl_sync(0xffffffffu, my_mnext, rl);
            const int64_t trow = (int64_t)blockIdx.x * BM + q * 32 + rl;
            dhv[u] = has_next ? mn * stg[rl * 33 + lane] : 0.f;
            dcv[u] = has_next ? dc_scr[trow * H + j] : 0.f;
            if (inst[u] >= 0) {
              dhv[u] += dh_out[(int64_t)inst[u] * H + j];
              const float* sv = save + (int64_t)inst[u] * 7 * H + j;
#pragma unroll
              for (int k = 0; k < 6; ++k) ld[u][k] = sv[(k + 1) * H];  // c_in,i,f,g,o,tc
            } else {
#pragma unroll
              for (int k = 0; k < 6; ++k) ld[u][k] = 0.f;
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rl = r0 + u;
            const int r = q * 32 + rl;
            const float mp = __shfl_sync(0xffffffffu, my_m, rl);
            const int64_t trow = (int64_t)blockIdx.x * BM + r;
            float da[4] = {0.f, 0.f, 0.f, 0.f};
            float dcp = 0.f;
            if (inst[u] >= 0) {
              const float c_in = ld[u][0], ig = ld[u][1], fg = ld[u][2], gg = ld[u][3],
                          og = ld[u][4], tc = ld[u][5];
              const float g_ = dhv[u];
              const float d_o = g_ * tc;
              const float dcn = dcv[u] + g_ * og * (1.f - tc * tc);
              da[0] = dcn * gg * ig * (1.f - ig);
              da[1] = dcn * c_in * fg * (1.f - fg);
              da[2] = dcn * ig * (1.f - gg * gg);
              da[3] = d_o * og * (1.f - og);
              dcp = dcn * fg * mp;
              float* o = dgx + (int64_t)inst[u] * G4 + j;
#pragma unroll
              for (int g = 0; g < 4; ++g) {
                if (rnd) da[g] = rna_tf32(da[g]);
                o[g * H] = da[g];
                bsum[cc][g] += da[g];
              }
            }
            if (row0 + r < R) dc_scr[trow * H + j] = dcp;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const int seq = seq0 + g;
              *reinterpret_cast<float*>(sA + (seq % kBwdAStages) * kAStage + sw128_offset(r, lane)) = da[g];
            }
          }
        }
        fence_async_smem();
#pragma unroll
        for (int g = 0; g < 4; ++g) mbar_arrive(&a_full[(seq0 + g) % kBwdAStages]);
        __syncwarp();
      }
      if (has_next) {  // release the accumulator this position read
        fence_before();
        mbar_arrive(&acc_empty[(p + 1) & 1]);
      }
    }
    // bias partials: combine the 4 quadrant warps of each half in fixed order
    if (bias_partial) {
      __syncwarp();
      for (int cc = 0; cc < (NC + 1) / 2; ++cc) {  // uniform trip count for bar.sync
        const int c = half + 2 * cc;
        for (int g = 0; g < 4; ++g) {
          stg[lane] = bsum[cc][g];
          asm volatile("bar.sync 1, %0;" ::"r"(kBwdEpiThreads));
          if (q == 0 && c < NC) {
            float acc = 0.f;
            for (int qq = 0; qq < 4; ++qq)
              acc += stg_all[((qq + 4 * half) - 0) * 32 * 33 + lane];
            bias_partial[(int64_t)blockIdx.x * G4 + g * H + 32 * c + lane] = acc;
          }
          asm volatile("bar.sync 1, %0;" ::"r"(kBwdEpiThreads));
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

// Backward, 2-CTA cluster, K-split (H = 128). CTA c owns hidden units
// [c*H/2, (c+1)*H/2) and the 8 da k-blocks (4 gates x 2 chunks of 32 units) of
// them. Its MMA forms a PARTIAL dh for ALL H units from its own k-blocks only
// (M = 128 rows, N = H, K = 2H; B = the matching 32-column blocks of U), so the
// A ring stays CTA-local (local arrivals, no cluster-scope fences). The two
// CTAs then swap the halves that belong to the other CTA's units: 8 rows x H/2
// floats per epilogue warp through st.async + complete_tx into the peer's
// double-buffered receive tile, and each CTA adds its own half (TMEM, staged in
// shared memory) and the received half. rq rows per lane quadrant as the
// forward; 8 rows per epilogue warp (12 warps when rq <= 24, else 16).
// Vectorised epilogue: a lane owns 4 consecutive units of 2 rows per 32-unit
// chunk (lane = 4 rows x 8 unit quads), so its saved gates are one 32-B load
// (the interleaved compact row), c_in 8 B, dh_out / dgx / the da A-tile 16-B
// vectors; in the 12-warp variant every load of a position is issued at its
// start, under the wait for the position's dh partials. Carried dc in registers.
// A-ring depth and receive-tile rows per lane quadrant: the 12-warp variant
// (rq <= 24) sizes the receive tiles for 24 rows and spends the freed shared
// memory on 6 A stages, so the second chunk's da rarely waits for the MMA to
// drain the first chunk's stages.
template <int kVEW> __host__ __device__ constexpr int ks_a_stages() { return kVEW <= 12 ? 5 : 3; }
template <int kVEW> __host__ __device__ constexpr int ks_recv_rq() { return kVEW <= 12 ? 24 : 32; }
constexpr int kKsStgStride = 64 + 16;  // own-half staging row stride (floats): conflict-free
                                        // for the (row, unit quad) writes and the (r4, u8) reads
template <int H, int kVEW, bool DH16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * kVEW, 1)
    lstm_bwd_tc2k_kernel(const float* __restrict__ U, const int32_t* __restrict__ slot_row,
                         const uint8_t* __restrict__ slot_mask, int64_t R, int L,
                         const float* __restrict__ save, const float* __restrict__ dh_out,
                         float* __restrict__ dgx, int rnd, float* __restrict__ bias_partial,
                         int rq, float da_scale, int dgx16, uint32_t recv_bytes) {
  static_assert(H == 128, "K-split cluster BPTT is specialised for H = 128");
  constexpr int EW = kVEW;
  constexpr int kEpiT = 32 * EW;
  constexpr int RPW = 8;                     // rows per warp
  constexpr bool kHoist = EW <= 12;          // chunk 0's loads issued at the position start
  constexpr int G4 = 4 * H;
  constexpr int HU = H / 2;
  constexpr int KBO = 4;                     // own fp16 da k-blocks (64 gate columns) per position
  constexpr int kAStage = BM * 128;          // 128 rows x 64 fp16 gate columns
  constexpr int kUBytes = KBO * H * 128;     // resident fp16 B: H units x 256 own gate columns
  constexpr int kS = kKsStgStride;
  constexpr int kStgW = RPW * kS;
  static_assert(kStgW >= 8 * 32, "staging must hold the warp's bias partials");
  constexpr int kKsAStages = ks_a_stages<kVEW>();
  constexpr int kRQ = ks_recv_rq<kVEW>();    // receive-tile rows per lane quadrant
  constexpr int kRecv = 4 * kRQ * HU;        // floats per receive tile
  // two N = H accumulators + the epilogue's carried dc (thread-private words
  // at columns 2H + 16 * (warp's row group): 16 floats per lane)
  constexpr uint32_t kTmemCols = 4 * H;
  constexpr int kSF = tc_save_floats<H>();   // compact save row (floats)
  using DhoT = typename std::conditional<DH16, uint2, float4>::type;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B aligned base, derived from the __shared__ array (keeps shared-space
  // addressing: STS/LDS instead of generic ST/LD)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sU = sA + kKsAStages * kAStage;
  float* recv = reinterpret_cast<float*>(sU + kUBytes);  // [2][4 kRQ][HU]
  float* stg_all = recv + 2 * kRecv;
  uint64_t* a_full = reinterpret_cast<uint64_t*>(stg_all + EW * kStgW);
  uint64_t* a_empty = a_full + kKsAStages;
  uint64_t* acc_full = a_empty + kKsAStages;    // [2]
  uint64_t* acc_empty = acc_full + 2;           // [2]
  uint64_t* recv_full = acc_empty + 2;          // [2]
  uint64_t* u_ready = recv_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(u_ready + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank(), peer = crank ^ 1u;
  const int64_t tile = blockIdx.x >> 1;
  const int64_t row0 = tile * 4 * rq;
  const int u0 = (int)crank * HU, pu0 = (int)peer * HU;
  if (warp == 0 && lane == 0) {
    // one arrival per epilogue warp (lane 0 after the warp's fences and a
    // __syncwarp): 384 per-thread arrivals on one mbarrier serialise for ~0.4 us
    for (int s = 0; s < kKsAStages; ++s) {
      mbar_init(&a_full[s], EW);
      mbar_init(&a_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], EW);
      mbar_init(&recv_full[a], 1);  // local arrive.expect_tx + the peer's st.async bytes
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    // the MMA's B operand, resident for the launch: U's 256 own gate columns for
    // all H units as fp16, K-major SWIZZLE_128B ([4 k-blocks][H rows][128 B]),
    // written by every thread (one warp took ~20 us, the first MMA's wait)
#pragma unroll 4
    for (int c = threadIdx.x; c < H * (4 * HU / 8); c += 64 + 32 * EW) {
      const int n = c % H, k0 = (c / H) * 8;
      const int i = k0 >> 5, gcol = (i & 3) * H + 32 * (2 * (int)crank + (i >> 2)) + (k0 & 31);
      const float* src = U + (int64_t)fx_unit(n) * G4 + gcol;  // N order: see fx_unit
      const float4 a = ldg4(src), b = ldg4(src + 4);
      const uint32_t dst = smem_u32(sU) + (uint32_t)((k0 >> 6) * H * 128 + n * 128 +
                                                     ((((k0 & 63) >> 3) ^ (n & 7)) << 4));
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(h2u(a.x, a.y)),
                   "r"(h2u(a.z, a.w)), "r"(h2u(b.x, b.y)), "r"(h2u(b.z, b.w))
                   : "memory");
    }
    fence_async_smem();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised before any st.async
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // own gate column k (0..255) of a position: 32-column block i = k >> 5 =
  // 4 lc + g (chunk lc: global chunk 2*crank + lc, gate g); fp16 k-block k >> 6

  if (warp == 0) {
    // idle after the prologue
  } else if (warp == 1) {
    // dh partial = (S da)[128, own 256] x U_own^T -> TMEM (kind::f16, fp32 accumulate)
    const uint32_t idesc16 = idesc_f16(H);
    const uint32_t a_base = smem_u32(sA), u_base = smem_u32(sU);
    for (int t = 0; t < L; ++t) {
      const int p = L - 1 - t;
      const int a = p & 1;
      mbar_wait(&acc_empty[a], ((t >> 1) & 1) ^ 1);
      fence_after();
      for (int i = 0; i < KBO; ++i) {
        const int seq = t * KBO + i;
        const int sa = seq % kKsAStages;
        mbar_wait(&a_full[sa], (seq / kKsAStages) & 1);
        fence_after();
        DGC_TS(i == KBO - 1 && blockIdx.x == 0 && lane == 0 && t < 256, t, 7);
        if (lane == 0) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_f16(tmem_base + a * H, kdesc(a_base + sa * kAStage + kk * 32),
                    kdesc(u_base + i * H * 128 + kk * 32), idesc16, (i > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&a_empty[sa]);
          if (i == KBO - 1) mma_commit(&acc_full[a]);
        }
        __syncwarp();
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;                 // TMEM lane quadrant (warp id % 4)
    const int rb = (ew >> 2) * RPW;         // first quadrant row of this warp
    const int r4 = lane >> 3, u8 = lane & 7;  // vector lane: rows rb + 4 it + r4, units 4 u8 .. +3
    const uint32_t stg_s = smem_u32(stg_all + ew * kStgW);
    const uint32_t sA_s = smem_u32(sA), recv_s = smem_u32(recv);
    // the TMEM base and the peer's receive-tile addresses are re-derived where
    // they are used (a shared-memory load / one mapa): held in registers across
    // the position loop they were spilled to local memory and reloaded on the
    // critical path
    const uint32_t tslot_s = smem_u32(tmem_slot);
    const bool active = rb < rq;
    const float inv_scale = 1.f / da_scale;  // da_scale: a power of two
    int sbase[2];  // first slot of each of this lane's rows (R * L < 2^31), -1: no row
    int inst[2];
    // slot masks as bits: bit it = this position's mask of row it, bit 2 + it =
    // the mask of its successor slot (mnext)
    uint32_t mbits = 0;
#pragma unroll
    for (int it = 0; it < 2; ++it) {
      const int rl = rb + 4 * it + r4;
      const int64_t vrow = row0 + q * rq + rl;
      sbase[it] = (rl < rq && vrow < R) ? (int)(vrow * L) : -1;
      inst[it] = sbase[it] >= 0 ? slot_row[sbase[it] + L - 1] : -1;
      mbits |= (sbase[it] >= 0 && slot_mask[sbase[it] + L - 1]) ? (1u << it) : 0u;
    }
    // thread-private TMEM words next to the accumulators (kept out of the
    // register file, where they were spilled to local memory): the carried dc
    // of (chunk lc, row it) at tdc + 8 lc + 4 it, and the bias partial sums of
    // (chunk lc, gate g) at tbs + 16 lc + 4 g
    const uint32_t tq = tmem_base + ((uint32_t)(q * 32) << 16);
    const uint32_t tdc = tq + 2 * H + 16 * (uint32_t)(ew >> 2);
    const uint32_t tbs = tq + 2 * H + 64 + 32 * (uint32_t)(ew >> 2);
    {
      const float z[16] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      tmem_st16(tdc, z);
      tmem_st16(tbs, z);
      tmem_st16(tbs + 16, z);
    }
    // this lane's saved fields of (chunk lc, row it): dh_out (4 units), c_in, i/f/g/o.
    // DH16: dh_out is S-scaled fp16 (8 B per lane, kept raw until its use)
    auto load_fields = [&](int lc, int it, DhoT& dho, uint2& cv, uint4& g0, uint4& g1) {
      const int j = u0 + 32 * lc + 4 * u8;
      if (inst[it] >= 0) {
        if constexpr (DH16)
          dho = __ldg(reinterpret_cast<const uint2*>(dh_out) + (((int64_t)inst[it] * H + j) >> 2));
        else
          dho = ldg4(dh_out + (int64_t)inst[it] * H + j);
        const __half* sv = reinterpret_cast<const __half*>(save + (int64_t)inst[it] * kSF) + H;
        cv = __ldg(reinterpret_cast<const uint2*>(sv + j));
        g0 = __ldg(reinterpret_cast<const uint4*>(sv + H + 4 * j));
        g1 = __ldg(reinterpret_cast<const uint4*>(sv + H + 4 * j + 8));
      } else {
        if constexpr (DH16)
          dho = make_uint2(0u, 0u);
        else
          dho = zero4();
        cv = make_uint2(0u, 0u);
        g0 = g1 = make_uint4(0u, 0u, 0u, 0u);
      }
    };
    for (int t = 0; t < L; ++t) {
      const int p = L - 1 - t;
      const bool has_next = p + 1 < L;
      DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 0);
      DhoT dho[2][2];
      uint2 cvv[2][2];
      uint4 gv0[2][2], gv1[2][2];
      if (kHoist) {  // chunk 0 now; chunk 1's lines into L2 (loaded before chunk 1's math)
#pragma unroll
        for (int it = 0; it < 2; ++it) {
          load_fields(0, it, dho[0][it], cvv[0][it], gv0[0][it], gv1[0][it]);
          if (inst[it] >= 0) {
            const int j = u0 + 32 + 4 * u8;
            const __half* sv = reinterpret_cast<const __half*>(save + (int64_t)inst[it] * kSF) + H;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(sv + H + 4 * j));
            if (u8 == 0) {
              asm volatile("prefetch.global.L2 [%0];" ::"l"(sv + j));
              asm volatile("prefetch.global.L2 [%0];" ::"l"(dh_out + (int64_t)inst[it] * H + j));
            }
          }
        }
      }
      // the next position's slots (consumed one position later)
      int n_inst[2];
      uint32_t n_mbits = 0;
#pragma unroll
      for (int it = 0; it < 2; ++it) {
        const bool ok = sbase[it] >= 0 && p > 0;
        n_inst[it] = ok ? slot_row[sbase[it] + p - 1] : -1;
        n_mbits |= (ok && slot_mask[sbase[it] + p - 1]) ? (1u << it) : 0u;
      }
      DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 6);
      if (has_next) {
        // recv_bytes: what the peer sends into our receive tile per position
        // (8 rows x HU per active peer warp); a kernel parameter, so it is not
        // held in (spilled) registers across the loop
        if (ew == 0 && lane == 0) mbar_arrive_expect_tx(&recv_full[t & 1], recv_bytes);
        mbar_wait(&acc_full[(p + 1) & 1], ((t - 1) >> 1) & 1);
        fence_after();
        DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 1);
        if (active) {
          // partial dh of this warp's 8 rows: 16x256b TMEM loads of lanes
          // q*32 + (rb & 16) .. +15 hand lane (r8, uq) units 16 i + 4 uq .. +3 of
          // row rb + r8 (U's rows are in fx_unit order): own units -> staging,
          // the peer's units -> the peer's receive tile, all lanes storing
          uint32_t tbase;
          asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tbase) : "r"(tslot_s));
          const uint32_t ta = tbase + ((uint32_t)(q * 32 + (rb & 16)) << 16) + ((p + 1) & 1) * H;
          const bool hi = (rb & 8) != 0;
          const int r8 = lane >> 2, uq = lane & 3;
          float v[16];
          tmem_ld16x256x4(ta + u0, ta + u0 + 16, ta + u0 + 32, ta + u0 + 48, hi, v);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            sts4(stg_s + (uint32_t)((r8 * kS + 16 * i + 4 * uq) * 4),
                 make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
          tmem_ld16x256x4(ta + pu0, ta + pu0 + 16, ta + pu0 + 32, ta + pu0 + 48, hi, v);
          const uint32_t dst = map_peer(recv, peer) +
                               (uint32_t)(((t & 1) * kRecv + (q * kRQ + rb + r8) * HU + 4 * uq) * 4);
          const uint32_t rfull = map_peer(recv_full, peer) + (uint32_t)((t & 1) * 8);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            st_async_v4(dst + 64 * i, make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]),
                        rfull);
        }
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[(p + 1) & 1]);  // this accumulator is fully read
        DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 3);
        mbar_wait(&recv_full[t & 1], ((t - 1) >> 1) & 1);
        DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 4);
        __syncwarp();
      }
#pragma unroll
      for (int lc = 0; lc < 2; ++lc) {
        const int seq0 = t * KBO + lc * 2;   // this chunk's 2 fp16 k-blocks (gates 0-1, 2-3)
        const int jo = 32 * lc + 4 * u8;     // own unit index of this lane's 4 units
        if (!kHoist) {
#pragma unroll
          for (int it = 0; it < 2; ++it)
            load_fields(lc, it, dho[lc][it], cvv[lc][it], gv0[lc][it], gv1[lc][it]);
        }
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int seq = seq0 + g;
          mbar_wait(&a_empty[seq % kKsAStages], ((seq / kKsAStages) & 1) ^ 1);
        }
        float dcv[8];  // carried dc of this chunk: row it at dcv[4 it .. 4 it + 3]
        tmem_ld8_after_st(tdc + 8 * lc, dcv);
        float bs[16];  // running bias sums of this chunk: gate g at bs[4 g .. 4 g + 3]
        tmem_ld16(tbs + 16 * lc, bs);
#pragma unroll
        for (int it = 0; it < 2; ++it) {
          const int rl = rb + 4 * it + r4;
          const int r = q * 32 + rl;
          float4 dh = zero4();
          if (has_next) {
            const float4 a = lds4(stg_s + (uint32_t)(((4 * it + r4) * kS + jo) * 4));
            const float4 b = lds4(recv_s + (uint32_t)((((t & 1) * kRecv) + (q * kRQ + rl) * HU + jo) * 4));
            const float mn = ((mbits >> (2 + it)) & 1u) ? inv_scale : 0.f;  // S-scaled partials (exact)
            dh = make_float4(mn * (a.x + b.x), mn * (a.y + b.y), mn * (a.z + b.z), mn * (a.w + b.w));
          }
          float4 da[4] = {zero4(), zero4(), zero4(), zero4()};
          float4 dcp = zero4();
          if (inst[it] >= 0) {
            float4 ho;
            if constexpr (DH16) {
              const float2 a = u2h(dho[lc][it].x), b = u2h(dho[lc][it].y);
              ho = make_float4(a.x * inv_scale, a.y * inv_scale, b.x * inv_scale, b.y * inv_scale);
            } else {
              ho = dho[lc][it];
            }
            dh = make_float4(dh.x + ho.x, dh.y + ho.y, dh.z + ho.z, dh.w + ho.w);
            const float2 c01 = u2h(cvv[lc][it].x), c23 = u2h(cvv[lc][it].y);
            const float cin[4] = {c01.x, c01.y, c23.x, c23.y};
            const uint32_t gw[8] = {gv0[lc][it].x, gv0[lc][it].y, gv0[lc][it].z, gv0[lc][it].w,
                                    gv1[lc][it].x, gv1[lc][it].y, gv1[lc][it].z, gv1[lc][it].w};
            const float dhk[4] = {dh.x, dh.y, dh.z, dh.w};
            const float dck[4] = {dcv[4 * it], dcv[4 * it + 1], dcv[4 * it + 2], dcv[4 * it + 3]};
            const float mp = ((mbits >> it) & 1u) ? 1.f : 0.f;
            float dak[4][4], dcpk[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 if_ = u2h(gw[2 * k]), go = u2h(gw[2 * k + 1]);
              const float ig = if_.x, fg = if_.y, gg = go.x, og = go.y;
              const float tc = tanh_fast(fg * cin[k] + ig * gg);  // the forward's tanh(c)
              const float g_ = dhk[k];
              const float d_o = g_ * tc;
              const float dcn = dck[k] + g_ * og * (1.f - tc * tc);
              dak[0][k] = dcn * gg * ig * (1.f - ig);
              dak[1][k] = dcn * cin[k] * fg * (1.f - fg);
              dak[2][k] = dcn * ig * (1.f - gg * gg);
              dak[3][k] = d_o * og * (1.f - og);
              dcpk[k] = dcn * fg * mp;
            }
            dcp = make_float4(dcpk[0], dcpk[1], dcpk[2], dcpk[3]);
            const int64_t oi = (int64_t)inst[it] * G4 + u0 + jo;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              float4 v = make_float4(dak[g][0], dak[g][1], dak[g][2], dak[g][3]);
              if (dgx16) {  // S da as fp16: the operand of the fp16 weight-gradient GEMMs
                sth4(reinterpret_cast<__half*>(dgx) + oi + g * H,
                     make_float4(v.x * da_scale, v.y * da_scale, v.z * da_scale, v.w * da_scale));
              } else {
                if (rnd) v = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
                st4(dgx + oi + g * H, v);
              }
              da[g] = v;
              bs[4 * g] += v.x; bs[4 * g + 1] += v.y; bs[4 * g + 2] += v.z; bs[4 * g + 3] += v.w;
            }
          }
          dcv[4 * it] = dcp.x; dcv[4 * it + 1] = dcp.y; dcv[4 * it + 2] = dcp.z; dcv[4 * it + 3] = dcp.w;
          // chunk 1's fields of this row: issued as soon as chunk 0's fields of the
          // row are consumed (their registers), so they are in flight under the
          // rest of chunk 0
          if (kHoist && lc == 0)
            load_fields(1, it, dho[1][it], cvv[1][it], gv0[1][it], gv1[1][it]);
          // S da as fp16 into the A tiles: gate g -> k-block seq0 + g/2, columns
          // 32 (g & 1) + 4 u8 .. +3 of its 64 (8 B of a 16-B swizzle chunk)
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const int k16 = (g & 1) * 32 + 4 * u8;
            const uint32_t addr = sA_s + (uint32_t)(((seq0 + (g >> 1)) % kKsAStages) * kAStage) +
                                  (uint32_t)(r * 128 + ((((k16 >> 3) ^ (r & 7))) << 4) + (k16 & 7) * 2);
            asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr),
                         "r"(h2u(da[g].x * da_scale, da[g].y * da_scale)),
                         "r"(h2u(da[g].z * da_scale, da[g].w * da_scale))
                         : "memory");
          }
        }
        tmem_st8(tdc + 8 * lc, dcv);
        tmem_st16(tbs + 16 * lc, bs);
        fence_async_smem();
        DGC_TS(lc == 1 && blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 2);
        DGC_TS3(lc == 1 && blockIdx.x == 0 && lane == 0 && t < 256, t, ew);
        DGC_TS(lc == 0 && blockIdx.x == 0 && threadIdx.x == 64 && t < 256, t, 5);
        __syncwarp();
        if (lane == 0) {
#pragma unroll
          for (int g = 0; g < 2; ++g) mbar_arrive(&a_full[(seq0 + g) % kKsAStages]);
        }
      }
      mbits = ((mbits & 3u) << 2) | n_mbits;  // this position's masks become mnext
#pragma unroll
      for (int it = 0; it < 2; ++it) inst[it] = n_inst[it];
    }
    if (bias_partial) {
      // the 4 row lanes of each unit quad (xor 8, 16), then the EW warps in fixed order
#pragma unroll
      for (int lc = 0; lc < 2; ++lc) {
        float bs[16];
        tmem_ld8_after_st(tbs + 16 * lc, bs);
        tmem_ld8(tbs + 16 * lc + 8, bs + 8);
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float4 v = make_float4(bs[4 * g], bs[4 * g + 1], bs[4 * g + 2], bs[4 * g + 3]);
#pragma unroll
          for (int m = 8; m <= 16; m <<= 1) {
            v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
            v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
            v.z += __shfl_xor_sync(0xffffffffu, v.z, m);
            v.w += __shfl_xor_sync(0xffffffffu, v.w, m);
          }
          if (r4 == 0) sts4(stg_s + (uint32_t)(((lc * 4 + g) * 32 + 4 * u8) * 4), v);
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(kEpiT));
      if (ew == 0) {
        for (int lc = 0; lc < 2; ++lc)
          for (int g = 0; g < 4; ++g) {
            float acc = 0.f;
            for (int w = 0; w < EW; ++w) acc += stg_all[w * kStgW + (lc * 4 + g) * 32 + lane];
            bias_partial[tile * G4 + g * H + u0 + 32 * lc + lane] = acc;
          }
      }
    }
  }
  fence_before();
  __syncthreads();
  cluster_sync_all();  // no st.async may still target this CTA's shared memory
  if (warp == 1) tmem_dealloc(tmem_base, kTmemCols);
}

template <int H, int EW, bool DH16>
int launch_lstm_bwd_tc2k_ew(const float* U, const int32_t* slot_row, const uint8_t* slot_mask,
                            int64_t R, int L, const float* save, const float* dh_out, float* dgx,
                            int rnd, float* bias_partial, int rq, float da_scale, int dgx16,
                            cudaStream_t s) {
  const size_t smem = (size_t)ks_a_stages<EW>() * BM * 128 + (size_t)4 * H * 128 +
                      (size_t)2 * 4 * ks_recv_rq<EW>() * (H / 2) * 4 + (size_t)EW * 8 * kKsStgStride * 4 +
                      1024 + 512;
  auto kern = lstm_bwd_tc2k_kernel<H, EW, DH16>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "lstm_bwd_tc2k: set smem");
  const int grid = 2 * (int)cluster_tiles(R);
  // bytes the peer sends into a receive tile per position: 8 rows x H/2 fp32
  // per active peer warp (4 quadrants x ceil(rq / 8) warps)
  const uint32_t recv_bytes = 4u * (uint32_t)((rq + 7) / 8) * 8u * (H / 2) * 4u;
  kern<<<grid, 64 + 32 * EW, smem, s>>>(U, slot_row, slot_mask, R, L, save, dh_out, dgx, rnd,
                                        bias_partial, rq, da_scale, dgx16, recv_bytes);
  DGC_CHECK_LAUNCH("lstm_bwd_tc2k_kernel");
  return DGC_OK;
}

// da_scale: power of two applied to da before its fp16 conversion (the MMA
// operand) and removed exactly from the dh partials; sized by the caller to
// the loss normalisation (mean over n instances: da ~ 1/n).
// dh16: dh_out holds S * dh as fp16 (the fp16 readout / input-gradient GEMMs'
// output), unscaled exactly at use
template <int H>
int launch_lstm_bwd_tc2k(const float* U, const int32_t* slot_row, const uint8_t* slot_mask,
                         int64_t R, int L, const float* save, const float* dh_out, float* dgx,
                         int rnd, float* bias_partial, float da_scale, int dgx16, int dh16,
                         cudaStream_t s) {
  DGC_REQUIRE(R * (int64_t)L < (int64_t)INT32_MAX, "lstm_bwd_tc2k: R * L must fit int32");
  const int rq = cluster_rows_per_quadrant(R);
  const bool ew12 = rq <= 24 && !getenv("DGC_RNN_EW16");
#define DGC_BWD2K(EW, D16)                                                                       \
  launch_lstm_bwd_tc2k_ew<H, EW, D16>(U, slot_row, slot_mask, R, L, save, dh_out, dgx, rnd,     \
                                      bias_partial, rq, da_scale, dgx16, s)
  if (dh16) return ew12 ? DGC_BWD2K(12, true) : DGC_BWD2K(16, true);
  return ew12 ? DGC_BWD2K(12, false) : DGC_BWD2K(16, false);
#undef DGC_BWD2K
}

// BPTT on the 2-SM tensor core (cta_group::2). Each CTA of the pair owns
// 4 x rq rows (rq per TMEM lane quadrant) and ALL H units of them, so the
// position's dh = (S da) U^T needs no exchange of partials: A is the CTA's own
// [128 rows x 4H gates] fp16 da tile (8 k-blocks of 64 gate columns), B = U's
// rows split along N (CTA c holds units 64c .. 64c + 63, all 4H gate columns,
// resident for the launch), and the even CTA issues one M = 256 MMA per k-block
// once both CTAs' epilogue warps have written it; the commits are multicast to
// both CTAs' barriers and each CTA reads its own rows x 128 units from its TMEM.
// Epilogue lane = 4 rows x 8 unit quads (one row, 4 units per 32-unit chunk,
// 4 chunks per position); the TMEM rows pass through a per-warp staging tile to
// reach that mapping. Own gate column k (0..4H-1) of a position: 32-column
// block i = k >> 5 = 4 lc + g (chunk lc, gate g); fp16 k-block k >> 6.
#define TS2M(t, k)                                                     \
  do {                                                                 \
    DGC_TS(blockIdx.x == 0 && threadIdx.x == 64 && (t) < 256, t, k);   \
    DGC_TS2(blockIdx.x == 1 && threadIdx.x == 64 && (t) < 256, t, k);  \
  } while (0)
template <int kEW> __host__ __device__ constexpr int km_a_stages() { return 8; }
constexpr int kKmStgStride = 128 + 4;  // staging row stride (floats, 16-B aligned)
// rows per quadrant of the 2-SM kernel: R over all 148 SMs, at most 16
inline int pair_rows_per_quadrant(int64_t R) {
  const int64_t per = (R + 4 * dgc::kNumSMs - 1) / (4 * dgc::kNumSMs);
  return (int)(per < 1 ? 1 : per > 16 ? 16 : per);
}
inline int64_t pair_cta_tiles(int64_t R) {
  const int64_t rows = 4 * (int64_t)pair_rows_per_quadrant(R);
  const int64_t t = (R + rows - 1) / rows;
  return t + (t & 1);
}
template <int H, int kEW>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * kEW, 1)
    lstm_bwd_tc2m_kernel(const float* __restrict__ U, const int32_t* __restrict__ slot_row,
                         const uint8_t* __restrict__ slot_mask, int64_t R, int L,
                         const float* __restrict__ save, const float* __restrict__ dh_out,
                         float* __restrict__ dgx, int rnd, float* __restrict__ bias_partial,
                         int rq, float da_scale, int dgx16) {
  static_assert(H == 128, "2-SM BPTT is specialised for H = 128");
  constexpr int EW = kEW;
  constexpr int kEpiT = 32 * EW;
  constexpr int RPW = 4;                     // rows per warp (one per lane row group)
  constexpr int G4 = 4 * H;
  constexpr int HN = H / 2;                  // B rows (units) held by each CTA
  constexpr int KB = G4 / 64;                // fp16 k-blocks per position
  constexpr int NC = H / 32;                 // 32-unit chunks per position
  constexpr int kAStage = BM * 128;          // 128 rows x 64 fp16 gate columns
  constexpr int kUBytes = KB * HN * 128;
  constexpr int kS = kKmStgStride;
  constexpr int kStgW = RPW * kS;
  static_assert(kStgW >= 4 * NC * 32, "staging must hold the warp's bias partials");
  constexpr int kAS = km_a_stages<kEW>();
  constexpr uint32_t kTmemCols = 2 * H;      // two N = H accumulators
  constexpr int kSF = tc_save_floats<H>();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sU = sA + kAS * kAStage;
  float* stg_all = reinterpret_cast<float*>(sU + kUBytes);
  uint64_t* a_full = reinterpret_cast<uint64_t*>(stg_all + EW * kStgW);  // used in CTA 0
  uint64_t* a_empty = a_full + kAS;
  uint64_t* acc_full = a_empty + kAS;    // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2], used in CTA 0
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const int64_t tile = blockIdx.x;
  const int64_t row0 = tile * 4 * rq;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kAS; ++s) {
      mbar_init(&a_full[s], 2 * EW);  // one arrival per epilogue warp of both CTAs
      mbar_init(&a_empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2 * EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    // this CTA's half of B: U rows 64 crank + n (n < 64) over all 4H gate
    // columns in k order, fp16, K-major SWIZZLE_128B ([KB][HN rows][128 B]);
    // every thread takes a share before the barriers below
#pragma unroll 4
    for (int c = threadIdx.x; c < HN * (G4 / 8); c += 64 + 32 * EW) {
      const int n = c % HN, k0 = (c / HN) * 8;
      const int i = k0 >> 5, gcol = (i & 3) * H + 32 * (i >> 2) + (k0 & 31);
      const float* src = U + (int64_t)(HN * (int)crank + n) * G4 + gcol;
      const float4 a = ldg4(src), b = ldg4(src + 4);
      const uint32_t dst = smem_u32(sU) + (uint32_t)((k0 >> 6) * HN * 128 + n * 128 +
                                                     ((((k0 & 63) >> 3) ^ (n & 7)) << 4));
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(dst), "r"(h2u(a.x, a.y)),
                   "r"(h2u(a.z, a.w)), "r"(h2u(b.x, b.y)), "r"(h2u(b.z, b.w))
                   : "memory");
    }
    fence_async_smem();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, kTmemCols);
  fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers initialised before any remote arrival
  fence_after();
  const uint32_t tmem_base = *tmem_slot;
  DGC_TS3(blockIdx.x == 0 && threadIdx.x == 0, 0, 30);

  if (warp == 0) {
    // idle after the prologue
  } else if (warp == 1) {
    if (crank == 0) {
      const uint32_t idesc = idesc_f16_m256(H);
      const uint32_t a_base = smem_u32(sA), u_base = smem_u32(sU);
      DGC_TS3(blockIdx.x == 0 && lane == 0, 0, 31);
      for (int t = 0; t < L; ++t) {
        const int a = (L - 1 - t) & 1;
        mbar_wait_cluster(&acc_empty[a], ((t >> 1) & 1) ^ 1);
        fence_after();
        for (int i = 0; i < KB; ++i) {
          const int seq = t * KB + i;
          const int sa = seq % kAS;
          mbar_wait_cluster(&a_full[sa], (seq / kAS) & 1);
          fence_after();
          DGC_TS(i == KB - 1 && blockIdx.x == 0 && lane == 0 && t < 256, t, 7);
          DGC_TS2(i == 0 && blockIdx.x == 0 && lane == 0 && t < 256, t, 7);
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma2_f16(tmem_base + a * H, kdesc(a_base + sa * kAStage + kk * 32),
                       kdesc(u_base + i * HN * 128 + kk * 32), idesc, (i > 0 || kk > 0) ? 1u : 0u);
            mma2_commit_mc(&a_empty[sa], 3);
            if (i == KB - 1) mma2_commit_mc(&acc_full[a], 3);
          }
          __syncwarp();
        }
      }
    }
  } else {
    const int ew = warp - 2;
    const int q = warp & 3;                   // TMEM lane quadrant (warp id % 4)
    const int rb = (ew >> 2) * RPW;           // first quadrant row of this warp
    const int r4 = lane >> 3, u8 = lane & 7;  // row rb + r4, units 32 lc + 4 u8 .. +3
    const int rl = rb + r4;
    const int r = q * 32 + rl;                // A-tile / TMEM row
    const uint32_t stg_s = smem_u32(stg_all + ew * kStgW);
    const uint32_t sA_s = smem_u32(sA);
    const uint32_t tl = tmem_base + ((uint32_t)(q * 32) << 16);
    const uint32_t a_full_l = map_peer(a_full, 0), acc_empty_l = map_peer(acc_empty, 0);
    const bool active = rb < rq;
    const float inv_scale = 1.f / da_scale;
    const int64_t vrow = row0 + q * rq + rl;
    const int sbase = (rl < rq && vrow < R) ? (int)(vrow * L) : -1;
    int inst = sbase >= 0 ? slot_row[sbase + L - 1] : -1;
    int mk = sbase >= 0 ? slot_mask[sbase + L - 1] : 0;
    float mnext = 0.f;
    float4 bsum[NC][4], dcr[NC];
#pragma unroll
    for (int lc = 0; lc < NC; ++lc) {
#pragma unroll
      for (int g = 0; g < 4; ++g) bsum[lc][g] = zero4();
      dcr[lc] = zero4();
    }
    auto load_fields = [&](int lc, float4& dho, uint2& cv, uint4& g0, uint4& g1) {
      const int j = 32 * lc + 4 * u8;
      if (inst >= 0) {
        dho = ldg4(dh_out + (int64_t)inst * H + j);
        const __half* sv = reinterpret_cast<const __half*>(save + (int64_t)inst * kSF) + H;
        cv = __ldg(reinterpret_cast<const uint2*>(sv + j));
        g0 = __ldg(reinterpret_cast<const uint4*>(sv + H + 4 * j));
        g1 = __ldg(reinterpret_cast<const uint4*>(sv + H + 4 * j + 8));
      } else {
        dho = zero4();
        cv = make_uint2(0u, 0u);
        g0 = g1 = make_uint4(0u, 0u, 0u, 0u);
      }
    };
    for (int t = 0; t < L; ++t) {
      const int p = L - 1 - t;
      const bool has_next = p + 1 < L;
      TS2M(t, 0);
      float4 dho[NC];
      uint2 cvv[NC];
      uint4 gv0[NC], gv1[NC];
      // chunks 0-1 now, the rest of the row's lines into L2
#pragma unroll
      for (int lc = 0; lc < 2; ++lc) load_fields(lc, dho[lc], cvv[lc], gv0[lc], gv1[lc]);
      if (inst >= 0) {
        const __half* sv = reinterpret_cast<const __half*>(save + (int64_t)inst * kSF) + H;
#pragma unroll
        for (int lc = 2; lc < NC; ++lc) {
          const int j = 32 * lc + 4 * u8;
          asm volatile("prefetch.global.L2 [%0];" ::"l"(sv + H + 4 * j));
        }
        if (u8 == 0) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(sv + 64));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(dh_out + (int64_t)inst * H + 64));
        }
      }
      const bool nok = sbase >= 0 && p > 0;
      const int n_inst = nok ? slot_row[sbase + p - 1] : -1;
      const int n_mk = nok ? slot_mask[sbase + p - 1] : 0;
      if (has_next) {
        mbar_wait(&acc_full[(p + 1) & 1], ((t - 1) >> 1) & 1);
        fence_after();
        TS2M(t, 1);
        if (active) {
          const uint32_t ta = tl + ((p + 1) & 1) * H;
          const bool mine = lane >= rb && lane < rb + RPW;
#pragma unroll
          for (int h4 = 0; h4 < H / 16; ++h4) {
            float v[16];
            tmem_ld16(ta + 16 * h4, v);
            if (mine) {
              const uint32_t d = stg_s + (uint32_t)(((lane - rb) * kS + 16 * h4) * 4);
#pragma unroll
              for (int u = 0; u < 16; u += 4)
                sts4(d + u * 4, make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]));
            }
          }
        }
        fence_before();
        __syncwarp();
        if (lane == 0) {
          if (crank) mbar_arrive_remote(acc_empty_l + (uint32_t)(((p + 1) & 1) * 8));
          else mbar_arrive(&acc_empty[(p + 1) & 1]);
        }
        TS2M(t, 3);
      }
#pragma unroll
      for (int lc = 0; lc < NC; ++lc) {
        const int seq0 = t * KB + lc * 2;   // this chunk's 2 fp16 k-blocks (gates 0-1, 2-3)
        const int jo = 32 * lc + 4 * u8;
        if (lc >= 2) load_fields(lc, dho[lc], cvv[lc], gv0[lc], gv1[lc]);
#pragma unroll
        for (int g = 0; g < 2; ++g) {
          const int seq = seq0 + g;
          mbar_wait(&a_empty[seq % kAS], ((seq / kAS) & 1) ^ 1);
        }
        float4 dh = zero4();
        if (has_next) {
          const float4 a = lds4(stg_s + (uint32_t)((r4 * kS + jo) * 4));
          const float mn = mnext * inv_scale;  // the accumulator is S-scaled (exact)
          dh = make_float4(mn * a.x, mn * a.y, mn * a.z, mn * a.w);
        }
        float4 da[4] = {zero4(), zero4(), zero4(), zero4()};
        float4 dcp = zero4();
        if (inst >= 0) {
          const float4 ho = dho[lc];
          dh = make_float4(dh.x + ho.x, dh.y + ho.y, dh.z + ho.z, dh.w + ho.w);
          const float2 c01 = u2h(cvv[lc].x), c23 = u2h(cvv[lc].y);
          const float cin[4] = {c01.x, c01.y, c23.x, c23.y};
          const uint32_t gw[8] = {gv0[lc].x, gv0[lc].y, gv0[lc].z, gv0[lc].w,
                                  gv1[lc].x, gv1[lc].y, gv1[lc].z, gv1[lc].w};
          const float dhk[4] = {dh.x, dh.y, dh.z, dh.w};
          const float dck[4] = {dcr[lc].x, dcr[lc].y, dcr[lc].z, dcr[lc].w};
          const float mp = (float)mk;
          float dak[4][4], dcpk[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 if_ = u2h(gw[2 * k]), go = u2h(gw[2 * k + 1]);
            const float ig = if_.x, fg = if_.y, gg = go.x, og = go.y;
            const float tc = tanh_fast(fg * cin[k] + ig * gg);  // the forward's tanh(c)
            const float g_ = dhk[k];
            const float d_o = g_ * tc;
            const float dcn = dck[k] + g_ * og * (1.f - tc * tc);
            dak[0][k] = dcn * gg * ig * (1.f - ig);
            dak[1][k] = dcn * cin[k] * fg * (1.f - fg);
            dak[2][k] = dcn * ig * (1.f - gg * gg);
            dak[3][k] = d_o * og * (1.f - og);
            dcpk[k] = dcn * fg * mp;
          }
          dcp = make_float4(dcpk[0], dcpk[1], dcpk[2], dcpk[3]);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            float4 v = make_float4(dak[g][0], dak[g][1], dak[g][2], dak[g][3]);
            if (!dgx16 && rnd) v = make_float4(rna_tf32(v.x), rna_tf32(v.y), rna_tf32(v.z), rna_tf32(v.w));
            da[g] = v;
          }
        }
        dcr[lc] = dcp;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int k16 = (g & 1) * 32 + 4 * u8;
          const uint32_t addr = sA_s + (uint32_t)(((seq0 + (g >> 1)) % kAS) * kAStage) +
                                (uint32_t)(r * 128 + ((((k16 >> 3) ^ (r & 7))) << 4) + (k16 & 7) * 2);
          asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(addr),
                       "r"(h2u(da[g].x * da_scale, da[g].y * da_scale)),
                       "r"(h2u(da[g].z * da_scale, da[g].w * da_scale))
                       : "memory");
        }
        fence_async_smem();
        __syncwarp();
        // the even CTA's MMA reads both CTAs' k-blocks: the odd CTA arrives on
        // the even CTA's barrier (CTA-scope release after the proxy fence)
        if (lane == 0) {
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            if (crank) mbar_arrive_remote(a_full_l + (uint32_t)(((seq0 + g) % kAS) * 8));
            else mbar_arrive(&a_full[(seq0 + g) % kAS]);
          }
        }
        if (inst >= 0) {
          const int64_t oi = (int64_t)inst * G4 + jo;
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 v = da[g];
            if (dgx16)
              sth4(reinterpret_cast<__half*>(dgx) + oi + g * H,
                   make_float4(v.x * da_scale, v.y * da_scale, v.z * da_scale, v.w * da_scale));
            else
              st4(dgx + oi + g * H, v);
            bsum[lc][g] = make_float4(bsum[lc][g].x + v.x, bsum[lc][g].y + v.y,
                                      bsum[lc][g].z + v.z, bsum[lc][g].w + v.w);
          }
        }
        TS2M(t, lc == NC - 1 ? 2 : 4 + lc);
        DGC_TS3(lc == NC - 1 && blockIdx.x < 2 && lane == 0 && t < 256, t, ew + 16 * (int)blockIdx.x);
              }
      mnext = (float)mk;
      inst = n_inst;
      mk = n_mk;
    }
    if (bias_partial) {
#pragma unroll
      for (int lc = 0; lc < NC; ++lc)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          float4 v = bsum[lc][g];
#pragma unroll
          for (int m = 8; m <= 16; m <<= 1) {
            v.x += __shfl_xor_sync(0xffffffffu, v.x, m);
            v.y += __shfl_xor_sync(0xffffffffu, v.y, m);
            v.z += __shfl_xor_sync(0xffffffffu, v.z, m);
            v.w += __shfl_xor_sync(0xffffffffu, v.w, m);
          }
          if (r4 == 0) sts4(stg_s + (uint32_t)(((lc * 4 + g) * 32 + 4 * u8) * 4), v);
        }
      asm volatile("bar.sync 1, %0;" ::"r"(kEpiT));
      if (ew == 0) {
        for (int lc = 0; lc < NC; ++lc)
          for (int g = 0; g < 4; ++g) {
            float acc = 0.f;
            for (int w = 0; w < EW; ++w) acc += stg_all[w * kStgW + (lc * 4 + g) * 32 + lane];
            bias_partial[tile * G4 + g * H + 32 * lc + lane] = acc;
          }
      }
    }
  }
  fence_before();
  __syncthreads();
  DGC_TS3(blockIdx.x == 0 && threadIdx.x == 0, 1, 30);
  cluster_sync_all();  // the pair's MMAs and remote arrivals are done before TMEM is freed
  if (warp == 1) tmem_dealloc2(tmem_base, kTmemCols);
}

template <int H, int EW>
int launch_lstm_bwd_tc2m_ew(const float* U, const int32_t* slot_row, const uint8_t* slot_mask,
                            int64_t R, int L, const float* save, const float* dh_out, float* dgx,
                            int rnd, float* bias_partial, int rq, float da_scale, int dgx16,
                            cudaStream_t s) {
  const size_t smem = (size_t)km_a_stages<EW>() * BM * 128 + (size_t)(4 * H / 64) * (H / 2) * 128 +
                      (size_t)EW * 4 * kKmStgStride * 4 + 1024 + 512;
  auto kern = lstm_bwd_tc2m_kernel<H, EW>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "lstm_bwd_tc2m: set smem");
  const int grid = (int)pair_cta_tiles(R);
  kern<<<grid, 64 + 32 * EW, smem, s>>>(U, slot_row, slot_mask, R, L, save, dh_out, dgx, rnd,
                                        bias_partial, rq, da_scale, dgx16);
  DGC_CHECK_LAUNCH("lstm_bwd_tc2m_kernel");
  return DGC_OK;
}

template <int H>
int launch_lstm_bwd_tc2m(const float* U, const int32_t* slot_row, const uint8_t* slot_mask,
                         int64_t R, int L, const float* save, const float* dh_out, float* dgx,
                         int rnd, float* bias_partial, float da_scale, int dgx16, cudaStream_t s) {
  DGC_REQUIRE(R * (int64_t)L < (int64_t)INT32_MAX, "lstm_bwd_tc2m: R * L must fit int32");
  const int rq = pair_rows_per_quadrant(R);
  DGC_REQUIRE(rq <= 12, "lstm_bwd_tc2m: at most 12 rows per quadrant");
  return launch_lstm_bwd_tc2m_ew<H, 12>(U, slot_row, slot_mask, R, L, save, dh_out, dgx, rnd,
                                        bias_partial, rq, da_scale, dgx16, s);
}
// The 2-SM BPTT is opt-in (DGC_BPTT_2SM; up to 48 rows per SM in one wave,
// R <= 7104): at C2 its positions take 7.7 us against the K-split kernel's 7.2
// (the exchange it removes is cheaper than the four-chunk epilogue it costs).
static bool bptt_2sm(int64_t R) {
  return getenv("DGC_BPTT_2SM") != nullptr && (R + 4 * dgc::kNumSMs - 1) / (4 * dgc::kNumSMs) <= 12;
}

template <int H>
int launch_lstm_bwd_tc(const float* U, const int32_t* slot_row, const uint8_t* slot_mask,
                       int64_t R, int L, const float* save, const float* dh_out, float* dgx,
                       float* dc_scr, int rnd, float* bias_partial, cudaStream_t s) {
  CUtensorMap m;
  int rc = make_map(&m, U, H, 4 * H, 4 * H, 32, H, false);
  if (rc) return rc;
  const size_t smem = (size_t)kBwdAStages * BM * 128 + (size_t)kBwdBStages * H * 128 +
                      (size_t)kBwdEpiWarps * 32 * 33 * 4 + 1024 + 512;
  auto kern = lstm_bwd_tc_kernel<H>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "lstm_bwd_tc: set smem");
  const int grid = (int)((R + BM - 1) / BM);
  kern<<<grid, kBwdThreads, smem, s>>>(m, slot_row, slot_mask, R, L, save, dh_out, dgx, dc_scr,
                                       rnd, bias_partial);
  DGC_CHECK_LAUNCH("lstm_bwd_tc_kernel");
  return DGC_OK;
}

template <int H>
int launch_lstm_tc(const float* gx, const float* Ut, const int32_t* slot_row,
                   const uint8_t* slot_mask, const int32_t* slot_carry, const float* carry,
                   int64_t R, int L, int64_t ld, float* h_out, float* c_out, float* save,
                   cudaStream_t s) {
  CUtensorMap m;
  const uint32_t box_rows = 4 * H > 256 ? 256 : 4 * H;
  int rc = make_map(&m, Ut, 4 * H, H, H, 32, box_rows, false);
  if (rc) return rc;
  const size_t smem = (size_t)(H / BK) * BM * 128 + (size_t)kStages * box_rows * 128 +
                      (size_t)kEpiWarps * kStgFloats * 4 + 1024 + 256;
  auto kern = lstm_fwd_tc_kernel<H>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "lstm_fwd_tc: set smem");
  const int grid = (int)((R + BM - 1) / BM);
  kern<<<grid, kThreads, smem, s>>>(m, gx, slot_row, slot_mask, slot_carry, carry, R, L, ld,
                                    h_out, c_out, save);
  DGC_CHECK_LAUNCH("lstm_fwd_tc_kernel");
  return DGC_OK;
}

}  // namespace

static bool cluster_rnn_enabled() { return getenv("DGC_NO_CLUSTER_RNN") == nullptr; }

extern "C" int dgc_rnn_fwd_tc(int32_t cell, const float* gx, const float* Ut,
                              const int32_t* slot_row, const uint8_t* slot_mask,
                              const int32_t* slot_carry, const float* carry, int64_t n_rows,
                              int32_t row_len, int32_t H, int64_t ld_out, float* h_out,
                              float* c_out, float* save, void* stream) {
  DGC_REQUIRE(cell == 1, "rnn_fwd_tc: only the LSTM cell has a tensor-core kernel yet");
  DGC_REQUIRE(c_out != nullptr, "rnn_fwd_tc: LSTM needs c_out");
  if (n_rows == 0 || row_len == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const bool cl = cluster_rnn_enabled();
  switch (H) {
    case 32: return launch_lstm_tc<32>(gx, Ut, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, ld_out, h_out, c_out, save, s);
    case 64:
      return cl ? launch_lstm_tc2v<64>(gx, Ut, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, ld_out, h_out, c_out, save, s)
                : launch_lstm_tc<64>(gx, Ut, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, ld_out, h_out, c_out, save, s);
    case 128:
      return cl ? launch_lstm_tc2v<128>(gx, Ut, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, ld_out, h_out, c_out, save, s)
                : launch_lstm_tc<128>(gx, Ut, slot_row, slot_mask, slot_carry, carry, n_rows, row_len, ld_out, h_out, c_out, save, s);
    default: return dgc::fail(DGC_ERR_ARG, "rnn_fwd_tc: H must be 32, 64 or 128");
  }
}

extern "C" int dgc_lstm_fwd_tc_f16x(const void* x16, int64_t n_x, const float* Wx,
                                    const float* U, const float* bias, const int32_t* slot_row,
                                    const uint8_t* slot_mask, const int32_t* slot_carry,
                                    const float* carry, int64_t n_rows, int32_t row_len,
                                    int64_t ld_out, float* h_out, float* c_out, float* save,
                                    void* h_out16, int32_t flags, void* stream) {
  DGC_REQUIRE(cluster_rnn_enabled(), "lstm_fwd_tc_f16x: needs the cluster kernels (DGC_NO_CLUSTER_RNN set)");
  DGC_REQUIRE(!(flags & 1) || h_out16 != nullptr, "lstm_fwd_tc_f16x: h at run ends only needs h_out16");
  DGC_REQUIRE(c_out != nullptr && bias != nullptr, "lstm_fwd_tc_f16x: c_out and bias required");
  if (n_rows == 0 || row_len == 0) return DGC_OK;
  return launch_lstm_tc2x(x16, n_x, Wx, U, bias, slot_row, slot_mask, slot_carry, carry, n_rows,
                          row_len, ld_out, h_out, c_out, save, static_cast<__half*>(h_out16),
                          flags & 1, dgc::as_stream(stream));
}

extern "C" int dgc_rnn_fwd_tc_fused_available(int32_t F, int32_t H) {
  return (F == 128 && H == 128 && cluster_rnn_enabled() && !getenv("DGC_NO_FUSED_XPROJ")) ? 1 : 0;
}

extern "C" int dgc_debug_lstm_timestamps(unsigned long long* out, int n) {
  if (n > 256 * 16) n = 256 * 16;
  cudaError_t e = cudaMemcpyFromSymbol(out, g_lstm_ts, (n < 256 * 8 ? n : 256 * 8) * sizeof(unsigned long long));
  if (e == cudaSuccess && n > 256 * 8)
    e = cudaMemcpyFromSymbol(out + 256 * 8, g_lstm_ts2, (n - 256 * 8) * sizeof(unsigned long long));
  return e == cudaSuccess ? DGC_OK : dgc::cuda_fail(e, "debug timestamps");
}

extern "C" int dgc_debug_lstm_timestamps_warps(unsigned long long* out, int n) {
  if (n > 256 * 32) n = 256 * 32;
  cudaError_t e = cudaMemcpyFromSymbol(out, g_lstm_ts3, n * sizeof(unsigned long long));
  return e == cudaSuccess ? DGC_OK : dgc::cuda_fail(e, "debug timestamps");
}

extern "C" int dgc_rnn_bwd_tc(int32_t cell_flags, const float* U, const int32_t* slot_row,
                              const uint8_t* slot_mask, int64_t n_rows, int32_t row_len, int32_t H,
                              const float* save, const float* dh_out, float* dgx, float* dc_scratch,
                              float* bias_partial, void* stream) {
  const int cell = cell_flags & 0xff, rnd = (cell_flags >> 8) & 1;
  DGC_REQUIRE(cell == 1, "rnn_bwd_tc: only the LSTM cell has a tensor-core kernel yet");
  if (n_rows == 0 || row_len == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  switch (H) {
    case 32: return launch_lstm_bwd_tc<32>(U, slot_row, slot_mask, n_rows, row_len, save, dh_out, dgx, dc_scratch, rnd, bias_partial, s);
    case 64: return launch_lstm_bwd_tc<64>(U, slot_row, slot_mask, n_rows, row_len, save, dh_out, dgx, dc_scratch, rnd, bias_partial, s);
    case 128:
      DGC_REQUIRE(!((cell_flags >> 25) & 1) || (cluster_rnn_enabled() && !bptt_2sm(n_rows)),
                  "rnn_bwd_tc: an fp16 dh_out needs the K-split cluster BPTT");
      return cluster_rnn_enabled()
                 ? (bptt_2sm(n_rows) ? launch_lstm_bwd_tc2m<128>(U, slot_row, slot_mask, n_rows, row_len, save, dh_out, dgx, rnd,
                                                           bias_partial, ldexpf(1.f, (cell_flags >> 16) & 0x7f),
                                                           (cell_flags >> 24) & 1, s)
                               : launch_lstm_bwd_tc2k<128>(U, slot_row, slot_mask, n_rows, row_len, save, dh_out, dgx, rnd,
                                                           bias_partial, ldexpf(1.f, (cell_flags >> 16) & 0x7f),
                                                           (cell_flags >> 24) & 1, (cell_flags >> 25) & 1, s))
                 : launch_lstm_bwd_tc<128>(U, slot_row, slot_mask, n_rows, row_len, save, dh_out, dgx, dc_scratch, rnd, bias_partial, s);
    default: return dgc::fail(DGC_ERR_ARG, "rnn_bwd_tc: H must be 32, 64 or 128");
  }
}

extern "C" int32_t dgc_rnn_tc_save_floats(int32_t H) {
  return (H == 128 && cluster_rnn_enabled()) ? tc_save_floats<128>() : 7 * H;
}

extern "C" int64_t dgc_rnn_tc_tiles(int64_t n_rows, int32_t H) {
  if (H == 128 && cluster_rnn_enabled()) return bptt_2sm(n_rows) ? pair_cta_tiles(n_rows) : cluster_tiles(n_rows);
  return (n_rows + 127) / 128;
}
