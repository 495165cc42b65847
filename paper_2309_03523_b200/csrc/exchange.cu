// K6: boundary-row exchange pack/unpack for the NCCL all-to-allv.
//
// The reference bills one message per cut edge (sim.py:464-469,514-543); a
// real halo exchange moves each (source row, destination device) once. The
// send list of a peer is the ascending-global-index list of own rows that the
// peer needs (derived from MessageSet.cut_mask, costmodel.py:160-165); the
// stale filter (K5) compacts it to the keys whose decision is "send".
#include "common.cuh"

namespace {

// Order-preserving compaction in one CTA (send lists are <= ~1e5 entries).
__global__ void __launch_bounds__(1024) compact_sent_kernel(const int32_t* __restrict__ pos,
                                                           int64_t n, const uint8_t* __restrict__ send,
                                                           int32_t* __restrict__ out_idx,
                                                           int32_t* __restrict__ count) {
  __shared__ int warp_sums[32];
  __shared__ int base_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) base_s = 0;
  __syncthreads();
  for (int64_t start = 0; start < n; start += blockDim.x) {
    const int64_t i = start + tid;
    const int flag = (i < n && send[pos[i]]) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, flag);
    const int prefix = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_sums[wid] = __popc(bal);
    __syncthreads();
    if (wid == 0) {
      int v = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      int incl = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += t;
      }
      warp_sums[lane] = incl - v;  // exclusive
      if (lane == 31) warp_sums[31] = incl;  // total in slot 31 after use below
    }
    __syncthreads();
    const int total = warp_sums[31];
    const int excl = (wid == 31) ? (total - __popc(bal)) : warp_sums[wid];
    if (flag) out_idx[base_s + excl + prefix] = (int32_t)i;
    __syncthreads();
    if (tid == 0) base_s += total;
    __syncthreads();
  }
  if (tid == 0) *count = base_s;
}

template <int LPR>
__global__ void gather_rows_kernel(const float4* __restrict__ Y, const int32_t* __restrict__ rows,
                                   const int32_t* __restrict__ idx, int64_t n, int w4,
                                   float4* __restrict__ out) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t i = tid / LPR; i < n; i += stride) {
    int64_t r = idx ? idx[i] : i;
    if (rows) r = rows[r];
    for (int j = lane; j < w4; j += LPR) out[i * w4 + j] = __ldg(Y + r * w4 + j);
  }
}

template <int LPR>
__global__ void scatter_rows_kernel(const float4* __restrict__ src, const int32_t* __restrict__ rows,
                                    const int32_t* __restrict__ idx, int64_t n, int w4,
                                    float4* __restrict__ dst, int add) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t i = tid / LPR; i < n; i += stride) {
    int64_t r = idx ? idx[i] : i;
    if (rows) r = rows[r];
    for (int j = lane; j < w4; j += LPR) {
      float4 v = __ldg(src + i * w4 + j);
      if (add) {
        const float4 o = dst[r * w4 + j];
        v.x += o.x;
        v.y += o.y;
        v.z += o.z;
        v.w += o.w;
      }
      dst[r * w4 + j] = v;
    }
  }
}

}  // namespace

extern "C" int dgc_compact_sent(const int32_t* pos, int64_t n, const uint8_t* send,
                                int32_t* out_idx, int32_t* count, void* stream) {
  cudaStream_t s = dgc::as_stream(stream);
  compact_sent_kernel<<<1, 1024, 0, s>>>(pos, n, send, out_idx, count);
  DGC_CHECK_LAUNCH("compact_sent_kernel");
  return DGC_OK;
}

extern "C" int dgc_gather_rows(const float* Y, const int32_t* rows, const int32_t* idx, int64_t n,
                               int32_t width, float* out, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "gather_rows: width must be a multiple of 4");
  if (n == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4, block = 256;
  const auto* y = reinterpret_cast<const float4*>(Y);
  auto* o = reinterpret_cast<float4*>(out);
  if (w4 >= 32) gather_rows_kernel<32><<<dgc::grid_for(n * 32, block), block, 0, s>>>(y, rows, idx, n, w4, o);
  else if (w4 >= 8) gather_rows_kernel<8><<<dgc::grid_for(n * 8, block), block, 0, s>>>(y, rows, idx, n, w4, o);
  else gather_rows_kernel<1><<<dgc::grid_for(n, block), block, 0, s>>>(y, rows, idx, n, w4, o);
  DGC_CHECK_LAUNCH("gather_rows_kernel");
  return DGC_OK;
}

extern "C" int dgc_scatter_rows(const float* src, const int32_t* rows, const int32_t* idx,
                                int64_t n, int32_t width, float* dst, int32_t add, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "scatter_rows: width must be a multiple of 4");
  if (n == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4, block = 256;
  const auto* sp = reinterpret_cast<const float4*>(src);
  auto* d = reinterpret_cast<float4*>(dst);
  if (w4 >= 32) scatter_rows_kernel<32><<<dgc::grid_for(n * 32, block), block, 0, s>>>(sp, rows, idx, n, w4, d, add);
  else if (w4 >= 8) scatter_rows_kernel<8><<<dgc::grid_for(n * 8, block), block, 0, s>>>(sp, rows, idx, n, w4, d, add);
  else scatter_rows_kernel<1><<<dgc::grid_for(n, block), block, 0, s>>>(sp, rows, idx, n, w4, d, add);
  DGC_CHECK_LAUNCH("scatter_rows_kernel");
  return DGC_OK;
}

// ---------------------------------------------------------------------------
// One-buffer exchange data plane (all peers per launch).
//
// The send lists of all peers are concatenated peer-major into "entries"
// (entry e = (peer p, list position j), ent_key[e] = the boundary key it
// carries, ent_ptr[p] = first entry of peer p; the lists derive from
// MessageSet.cut_mask, costmodel.py:160-165). A send buffer holds one RECORD
// per sent entry, peer-major, so the whole buffer is one NCCL all-to-allv
// with split p = count_p records:
//     record = [ int32 list position j | 3 pad words | width floats ]
// (16-byte header: rows stay float4-aligned). Staleness compacts the lists on
// the device (dgc_exchange_rank): no per-peer host round trip; the receiver
// learns the list positions from the headers.
namespace {

// Single-CTA two-pass compaction over all entries (peer-major): thread t owns
// a contiguous run; ent_slot[e] = global ordinal among sent entries or -1;
// counts[p] = sent entries of peer p.
__global__ void __launch_bounds__(1024) exch_rank_kernel(const int32_t* __restrict__ ent_key,
                                                        int64_t n_ent,
                                                        const int32_t* __restrict__ ent_ptr, int D,
                                                        const uint8_t* __restrict__ send,
                                                        int32_t* __restrict__ ent_slot,
                                                        int32_t* __restrict__ counts) {
  __shared__ int scan[1024];
  __shared__ int cnt_s[8];
  const int t = threadIdx.x, nt = blockDim.x;
  if (t < 8) cnt_s[t] = 0;
  const int64_t per = (n_ent + nt - 1) / nt;
  const int64_t b = min((int64_t)t * per, n_ent), e_end = min(b + per, n_ent);
  int cnt = 0;
  for (int64_t e = b; e < e_end; ++e) cnt += send[ent_key[e]] ? 1 : 0;
  scan[t] = cnt;
  __syncthreads();
  for (int off = 1; off < nt; off <<= 1) {  // Hillis-Steele inclusive scan
    const int v = t >= off ? scan[t - off] : 0;
    __syncthreads();
    scan[t] += v;
    __syncthreads();
  }
  int run = scan[t] - cnt;  // exclusive base of this thread's run
  int p = 0, pc = 0;        // per-peer counts of this run (entries are peer-major)
  for (int64_t e = b; e < e_end; ++e) {
    while (p < D && e >= ent_ptr[p + 1]) {
      if (pc) atomicAdd(&cnt_s[p], pc);
      pc = 0;
      ++p;
    }
    const bool s = send[ent_key[e]] != 0;
    ent_slot[e] = s ? run : -1;
    run += s ? 1 : 0;
    pc += s ? 1 : 0;
  }
  if (pc && p < D) atomicAdd(&cnt_s[p], pc);
  __syncthreads();
  if (t < D) counts[t] = cnt_s[t];
}

template <int LPR>
__global__ void exch_pack_kernel(const float4* __restrict__ Y, int w4,
                                 const int32_t* __restrict__ key_rows,
                                 const int32_t* __restrict__ ent_key,
                                 const int32_t* __restrict__ ent_idx,
                                 const int32_t* __restrict__ ent_slot, int64_t n_ent,
                                 float4* __restrict__ buf) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  const int rw4 = w4 + 1;
  for (int64_t e = tid / LPR; e < n_ent; e += stride) {
    const int64_t s = ent_slot ? __ldg(ent_slot + e) : e;
    if (s < 0) continue;
    const int64_t r = __ldg(key_rows + __ldg(ent_key + e));
    float4* rec = buf + s * rw4;
    if (lane == 0) rec[0] = make_float4(__int_as_float(__ldg(ent_idx + e)), 0.f, 0.f, 0.f);
    for (int j = lane; j < w4; j += LPR) rec[1 + j] = __ldg(Y + r * w4 + j);
  }
}

// peer of record i from the per-peer record counts (D <= 8, in shared memory)
__device__ __forceinline__ int peer_of(const int* off, int D, int64_t i) {
  int p = 0;
  while (p + 1 < D && i >= off[p + 1]) ++p;
  return p;
}

template <int LPR>
__global__ void exch_unpack_kernel(const float4* __restrict__ buf, int w4,
                                   const int32_t* __restrict__ rcounts, int D,
                                   const int32_t* __restrict__ rlist,
                                   const int32_t* __restrict__ rlist_ptr, int64_t n_max,
                                   float4* __restrict__ dst) {
  __shared__ int off[9];
  if (threadIdx.x == 0) {
    int a = 0;
    for (int p = 0; p < D; ++p) { off[p] = a; a += rcounts[p]; }
    off[D] = a;
  }
  __syncthreads();
  const int64_t total = min((int64_t)off[D], n_max);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  const int rw4 = w4 + 1;
  for (int64_t i = tid / LPR; i < total; i += stride) {
    const float4* rec = buf + i * rw4;
    const int p = peer_of(off, D, i);
    const int j = __float_as_int(__ldg(rec).x);
    const int64_t slot = __ldg(rlist + __ldg(rlist_ptr + p) + j);
    for (int k = lane; k < w4; k += LPR) dst[slot * w4 + k] = __ldg(rec + 1 + k);
  }
}

template <int LPR>
__global__ void exch_pack_back_kernel(const float4* __restrict__ fwd, int w4,
                                      const int32_t* __restrict__ rcounts, int D,
                                      const int32_t* __restrict__ rlist,
                                      const int32_t* __restrict__ rlist_ptr, int64_t n_max,
                                      const float4* __restrict__ dY, float4* __restrict__ out) {
  __shared__ int off[9];
  if (threadIdx.x == 0) {
    int a = 0;
    for (int p = 0; p < D; ++p) { off[p] = a; a += rcounts[p]; }
    off[D] = a;
  }
  __syncthreads();
  const int64_t total = min((int64_t)off[D], n_max);
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  const int rw4 = w4 + 1;
  for (int64_t i = tid / LPR; i < total; i += stride) {
    const int p = peer_of(off, D, i);
    const int j = __float_as_int(__ldg(fwd + i * rw4).x);
    const int64_t slot = __ldg(rlist + __ldg(rlist_ptr + p) + j);
    for (int k = lane; k < w4; k += LPR) out[i * w4 + k] = __ldg(dY + slot * w4 + k);
  }
}

// dY[key_rows[k]] += sum over the key's entries (ascending peer) of the
// gradient row returned for that entry (fixed order: bitwise deterministic)
template <int LPR>
__global__ void exch_add_back_kernel(const float4* __restrict__ back, int w4,
                                     const int32_t* __restrict__ key_rows,
                                     const int32_t* __restrict__ kent_ptr,
                                     const int32_t* __restrict__ kent,
                                     const int32_t* __restrict__ ent_slot, int64_t n_keys,
                                     float4* __restrict__ dY) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = (int)(tid % LPR);
  const int64_t stride = ((int64_t)gridDim.x * blockDim.x) / LPR;
  for (int64_t k = tid / LPR; k < n_keys; k += stride) {
    const int b = __ldg(kent_ptr + k), e = __ldg(kent_ptr + k + 1);
    bool any = false;
    for (int q = b; q < e; ++q) {
      const int en = __ldg(kent + q);
      if ((ent_slot ? __ldg(ent_slot + en) : en) >= 0) any = true;
    }
    if (!any) continue;
    const int64_t r = __ldg(key_rows + k);
    for (int j = lane; j < w4; j += LPR) {
      float4 acc = dY[r * w4 + j];
      for (int q = b; q < e; ++q) {
        const int en = __ldg(kent + q);
        const int64_t s = ent_slot ? __ldg(ent_slot + en) : en;
        if (s < 0) continue;
        const float4 g = __ldg(back + s * w4 + j);
        acc.x += g.x;
        acc.y += g.y;
        acc.z += g.z;
        acc.w += g.w;
      }
      dY[r * w4 + j] = acc;
    }
  }
}

inline int lpr_for(int w4) { return w4 >= 32 ? 32 : (w4 >= 8 ? 8 : 1); }

}  // namespace

extern "C" int dgc_exchange_rank(const int32_t* ent_key, int64_t n_ent, const int32_t* ent_ptr,
                                 int32_t D, const uint8_t* send, int32_t* ent_slot,
                                 int32_t* counts, void* stream) {
  DGC_REQUIRE(D >= 1 && D <= 8, "exchange_rank: 1 <= D <= 8");
  cudaStream_t s = dgc::as_stream(stream);
  exch_rank_kernel<<<1, 1024, 0, s>>>(ent_key, n_ent, ent_ptr, D, send, ent_slot, counts);
  DGC_CHECK_LAUNCH("exch_rank_kernel");
  return DGC_OK;
}

#define DGC_EXCH_LAUNCH(KERNEL, n, ...)                                                     \
  do {                                                                                      \
    const int block_ = 256;                                                                 \
    const int lpr_ = lpr_for(w4);                                                           \
    if (lpr_ == 32)                                                                         \
      KERNEL<32><<<dgc::grid_for((n) * 32, block_), block_, 0, s>>>(__VA_ARGS__);          \
    else if (lpr_ == 8)                                                                     \
      KERNEL<8><<<dgc::grid_for((n) * 8, block_), block_, 0, s>>>(__VA_ARGS__);            \
    else                                                                                    \
      KERNEL<1><<<dgc::grid_for((n), block_), block_, 0, s>>>(__VA_ARGS__);                \
    DGC_CHECK_LAUNCH(#KERNEL);                                                              \
  } while (0)

extern "C" int dgc_exchange_pack(const float* Y, int32_t width, const int32_t* key_rows,
                                 const int32_t* ent_key, const int32_t* ent_idx,
                                 const int32_t* ent_slot, int64_t n_ent, float* sendbuf,
                                 void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "exchange_pack: width must be a multiple of 4");
  if (n_ent == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4;
  DGC_EXCH_LAUNCH(exch_pack_kernel, n_ent, reinterpret_cast<const float4*>(Y), w4, key_rows,
                  ent_key, ent_idx, ent_slot, n_ent, reinterpret_cast<float4*>(sendbuf));
  return DGC_OK;
}

extern "C" int dgc_exchange_unpack(const float* recvbuf, int32_t width, const int32_t* rcounts,
                                   int32_t D, const int32_t* rlist, const int32_t* rlist_ptr,
                                   int64_t n_max, float* dst, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "exchange_unpack: width must be a multiple of 4");
  DGC_REQUIRE(D >= 1 && D <= 8, "exchange_unpack: 1 <= D <= 8");
  if (n_max == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4;
  DGC_EXCH_LAUNCH(exch_unpack_kernel, n_max, reinterpret_cast<const float4*>(recvbuf), w4, rcounts,
                  D, rlist, rlist_ptr, n_max, reinterpret_cast<float4*>(dst));
  return DGC_OK;
}

extern "C" int dgc_exchange_pack_back(const float* fwd_recvbuf, int32_t width,
                                      const int32_t* rcounts, int32_t D, const int32_t* rlist,
                                      const int32_t* rlist_ptr, int64_t n_max, const float* dY,
                                      float* backbuf, void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "exchange_pack_back: width must be a multiple of 4");
  DGC_REQUIRE(D >= 1 && D <= 8, "exchange_pack_back: 1 <= D <= 8");
  if (n_max == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4;
  DGC_EXCH_LAUNCH(exch_pack_back_kernel, n_max, reinterpret_cast<const float4*>(fwd_recvbuf), w4,
                  rcounts, D, rlist, rlist_ptr, n_max, reinterpret_cast<const float4*>(dY),
                  reinterpret_cast<float4*>(backbuf));
  return DGC_OK;
}

extern "C" int dgc_exchange_add_back(const float* backbuf, int32_t width, const int32_t* key_rows,
                                     const int32_t* kent_ptr, const int32_t* kent,
                                     const int32_t* ent_slot, int64_t n_keys, float* dY,
                                     void* stream) {
  DGC_REQUIRE(width % 4 == 0 && width > 0, "exchange_add_back: width must be a multiple of 4");
  if (n_keys == 0) return DGC_OK;
  cudaStream_t s = dgc::as_stream(stream);
  const int w4 = width / 4;
  DGC_EXCH_LAUNCH(exch_add_back_kernel, n_keys, reinterpret_cast<const float4*>(backbuf), w4,
                  key_rows, kent_ptr, kent, ent_slot, n_keys, reinterpret_cast<float4*>(dY));
  return DGC_OK;
}
