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
#include <cuda.h>

#include <cstdlib>

#include "common.cuh"

namespace {

constexpr int BM = 128;  // UMMA M
constexpr int BK = 32;   // fp32 elements per k-block = one 128-byte swizzle row
constexpr int kThreads = 192;
constexpr int kABytes = BM * BK * 4;  // 16 KiB

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint64_t t0 = globaltimer();
  while (true) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (globaltimer() - t0 > 4000000000ull) __trap();  // watchdog
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// UMMA shared-memory descriptor (sm_100 version bit). K-major operands use
// SWIZZLE_128B (layout 2): 8-row x 128-B atoms, SBO = 1024 B between row groups.
// MN-major 32-bit operands must use SWIZZLE_128B_BASE32B (layout 1): 4 k-rows
// x 128 B atoms (32-B swizzle granules), LBO = stride between 32-element MN
// chunks, SBO = 512 B between 4-row k groups (the TMA side writes it with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                          uint32_t layout) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__device__ __forceinline__ uint64_t kdesc(uint32_t saddr) { return sdesc(saddr, 16, 1024, 2); }
__device__ __forceinline__ uint64_t mndesc(uint32_t saddr) { return sdesc(saddr, 4096, 512, 1); }
// Instruction descriptor: D f32, A/B tf32, M=128, N=n.
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

template <bool A_MN, bool B_MN, bool SPLIT3>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     float* __restrict__ C, int64_t ldc, int64_t M, int64_t N, int bn, int stages,
                     int kb_total, int kb_per_split, int m_tiles, int n_tiles, int splits,
                     const float* __restrict__ bias, const float* __restrict__ relu_src,
                     int accumulate, float* __restrict__ partial) {
  // Persistent: CTA c owns tiles c, c+G, ... of the (split, n-tile, m-tile)
  // space (m fastest, so a CTA's consecutive tiles share the B panel). Two TMEM
  // accumulators let the epilogue drain tile i while the MMA runs tile i+1.
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~(uintptr_t)1023);
  const int b_bytes = bn * BK * 4;
  const int ab_bytes = kABytes + b_bytes;
  const int stage_bytes = ab_bytes * (SPLIT3 ? 2 : 1);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  uint64_t* conv = empty + stages;
  uint64_t* tfull = conv + stages;   // [2]
  uint64_t* tempty = tfull + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* stg_base = reinterpret_cast<float*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_tiles_total = m_tiles * n_tiles * splits;
  const uint32_t acc_cols = bn <= 32 ? 32 : bn <= 64 ? 64 : bn <= 128 ? 128 : 256;
  const uint32_t tmem_cols = 2 * acc_cols;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&conv[s], 128);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
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
    const int mt = t % m_tiles;
    const int rest = t / m_tiles;
    const int nt = rest % n_tiles;
    z = rest / n_tiles;
    m0 = (int64_t)mt * BM;
    n0 = (int64_t)nt * bn;
    kb0 = z * kb_per_split;
    nkb = min(kb_total, kb0 + kb_per_split) - kb0;
  };

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;
      for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        int64_t m0, n0;
        int z, kb0, nkb;
        tile_coords(t, m0, n0, z, kb0, nkb);
        for (int kb = 0; kb < nkb; ++kb, ++g) {
          const int s = g % stages;
          const uint32_t ph = (g / stages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + (size_t)s * stage_bytes;
          uint8_t* sb = sa + kABytes;
          mbar_expect_tx(&full[s], (uint32_t)ab_bytes);
          const int k0 = (kb0 + kb) * BK;
          if (!A_MN) {
            tma_load_2d(sa, &tmA, k0, (int)m0, &full[s]);
          } else {
#pragma unroll
            for (int i = 0; i < BM / 32; ++i)
              tma_load_2d(sa + i * 4096, &tmA, (int)m0 + 32 * i, k0, &full[s]);
          }
          if (!B_MN) {
            tma_load_2d(sb, &tmB, k0, (int)n0, &full[s]);
          } else {
            for (int i = 0; i < bn / 32; ++i)
              tma_load_2d(sb + i * 4096, &tmB, (int)n0 + 32 * i, k0, &full[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_tf32(bn, A_MN, B_MN);
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
          const uint32_t sa = smem_u32(smem + (size_t)s * stage_bytes);
          const uint32_t sb = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
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
    const int tq = threadIdx.x - 64;  // 0..127
    const int q = warp & 3;           // TMEM lane quadrant this warp may access
    float* stg = stg_base + (warp - 2) * 32 * 33;
    int g = 0, i = 0;
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
          for (int e = tq; e < ab_bytes / 16; e += 128) {
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
      mbar_wait(&tfull[a], aph);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // TMEM -> registers (thread = row) -> padded smem transpose -> coalesced
      // 128-byte row stores (lane = column), epilogue fused into the store pass.
      for (int c = 0; c < bn; c += 32) {
        float v[32];
        tmem_ld32(tmem_base + (uint32_t)a * acc_cols + ((uint32_t)(q * 32) << 16) + (uint32_t)c, v);
#pragma unroll
        for (int u = 0; u < 32; ++u) stg[lane * 33 + u] = v[u];
        __syncwarp();
        const int64_t n = n0 + c + lane;
        const bool col_ok = (c + lane < bn) && (n < N);
        const float bn_v = (bias && col_ok) ? __ldg(bias + n) : 0.f;
#pragma unroll
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
              C[row * ldc + n] = y;
            }
          }
        }
        __syncwarp();
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tempty[a]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(tmem_cols));
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

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// Row-major [rows, cols] fp32 tensor with row stride ld (elements).
int make_map(CUtensorMap* map, const float* ptr, int64_t rows, int64_t cols, int64_t ld,
             uint32_t box_cols, uint32_t box_rows, bool mn_major) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return dgc::fail(DGC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || ((ld * 4) & 15))
    return dgc::fail(DGC_ERR_ARG, "gemm: operands need 16-byte aligned base and row stride");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return dgc::fail(DGC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return DGC_OK;
}

template <bool A_MN, bool B_MN, bool SPLIT3>
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, float* C, int64_t ldc, int64_t M,
                int64_t N, int bn, int ntiles, int kb_total, int splits, int kb_per,
                const float* bias, const float* relu_src, int accumulate, float* partial,
                cudaStream_t s) {
  const int ab = kABytes + bn * BK * 4;
  const int stage_bytes = ab * (SPLIT3 ? 2 : 1);
  const int budget = 190 * 1024;
  int stages = budget / stage_bytes;
  stages = stages > 4 ? 4 : stages;
  if (const char* env = getenv("DGC_GEMM_MAX_STAGES")) {
    const int cap = atoi(env);
    if (cap >= 1 && cap < stages) stages = cap;
  }
  if (stages < 1) return dgc::fail(DGC_ERR_ARG, "gemm: tile does not fit shared memory");
  const size_t smem = (size_t)stages * stage_bytes + 1024 + 256 + 4 * 32 * 33 * 4;
  auto kern = gemm_tf32_kernel<A_MN, B_MN, SPLIT3>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return dgc::cuda_fail(e, "gemm: set smem");
  const int m_tiles = (int)((M + BM - 1) / BM);
  const int total = m_tiles * ntiles * splits;
  const int grid = total < dgc::kNumSMs ? total : dgc::kNumSMs;
  kern<<<grid, kThreads, smem, s>>>(ma, mb, C, ldc, M, N, bn, stages, kb_total, kb_per, m_tiles,
                                    ntiles, splits, bias, relu_src, accumulate, partial);
  DGC_CHECK_LAUNCH("gemm_tf32_kernel");
  return DGC_OK;
}

}  // namespace

extern "C" int dgc_gemm_splits(int64_t K, int32_t precision, int32_t k_splits) {
  const int kb_total = (int)((K + BK - 1) / BK);
  if (k_splits < 1) k_splits = 1;
  int kb_per = (kb_total + k_splits - 1) / k_splits;
  if (precision == 3 && kb_per > 16) kb_per = 16;
  return kb_per > 0 ? (kb_total + kb_per - 1) / kb_per : 1;
}

extern "C" int dgc_gemm_tf32(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                             int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn,
                             int32_t b_mn, int32_t precision, const float* bias,
                             const float* relu_src, int32_t accumulate, int32_t k_splits,
                             float* partial, void* stream) {
  DGC_REQUIRE(M >= 0 && N >= 0 && K >= 1, "gemm: bad shape");
  DGC_REQUIRE(precision == 1 || precision == 3, "gemm: precision must be 1 (TF32) or 3 (3xTF32)");
  DGC_REQUIRE(k_splits >= 1, "gemm: k_splits >= 1");
  if (M == 0 || N == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int align = b_mn ? 32 : 16;
  const int ntiles = (int)((N + 255) / 256);
  int bn = (int)((N + ntiles - 1) / ntiles);
  bn = (bn + align - 1) / align * align;
  if (bn > 256) bn = 256;
  const int kb_total = (int)((K + BK - 1) / BK);
  int kb_per = (kb_total + k_splits - 1) / k_splits;
  // The tcgen05 fp32 accumulator truncates (measured: a systematic -1.2e-4
  // relative bias after 625 k-blocks of 3xTF32, tools/debug_gemm.py), so the
  // fp32-parity mode caps every TMEM accumulation chain at kMaxChainKb k-blocks
  // and finishes the sum in the round-to-nearest split-K reduction.
  constexpr int kMaxChainKb = 16;
  if (precision == 3 && kb_per > kMaxChainKb) kb_per = kMaxChainKb;
  const int splits = (kb_total + kb_per - 1) / kb_per;
  if (splits > 1) DGC_REQUIRE(partial != nullptr, "gemm: k_splits > 1 needs a partial buffer");
  CUtensorMap ma, mb;
  int rc = a_mn ? make_map(&ma, A, K, M, lda, 32, 32, true)
                 : make_map(&ma, A, M, K, lda, 32, BM, false);
  if (rc) return rc;
  rc = b_mn ? make_map(&mb, B, K, N, ldb, 32, 32, true)
            : make_map(&mb, B, N, K, ldb, 32, (uint32_t)bn, false);
  if (rc) return rc;
  float* part = splits > 1 ? partial : nullptr;
  const bool s3 = precision == 3;
#define DGC_GEMM_CASE(AM, BMN, S3)                                                               \
  if ((bool)a_mn == AM && (bool)b_mn == BMN && s3 == S3)                                          \
    rc = launch_gemm<AM, BMN, S3>(ma, mb, C, ldc, M, N, bn, ntiles, kb_total, splits, kb_per,   \
                                  part ? nullptr : bias, part ? nullptr : relu_src,              \
                                  part ? 0 : accumulate, part, s);
  DGC_GEMM_CASE(false, false, false)
  DGC_GEMM_CASE(false, true, false)
  DGC_GEMM_CASE(true, false, false)
  DGC_GEMM_CASE(true, true, false)
  DGC_GEMM_CASE(false, false, true)
  DGC_GEMM_CASE(false, true, true)
  DGC_GEMM_CASE(true, false, true)
  DGC_GEMM_CASE(true, true, true)
#undef DGC_GEMM_CASE
  if (rc) return rc;
  if (part) {
    splitk_reduce_kernel<<<dgc::grid_for(M * N, 256), 256, 0, s>>>(part, splits, M, N, C, ldc,
                                                                   bias, relu_src, accumulate);
    DGC_CHECK_LAUNCH("splitk_reduce_kernel");
  }
  return DGC_OK;
}
