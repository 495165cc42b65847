/*
 * dgc_b200.h -- C ABI of the B200-native DGC chunk-partitioned DGNN step.
 *
 * Plain pointers and sizes only: device pointers are CUDA global-memory
 * addresses, `stream` is a cudaStream_t passed as void*. Every entry point
 * returns 0 on success and a negative code on failure; dgc_last_error()
 * returns the message (thread-local). Nothing here allocates or frees caller
 * memory except the opaque layout handle.
 *
 * The reference (`dynpart`, pure Python) has no FFI; each entry
 * point below names the reference function whose semantics it implements on
 * the GPU (file:line relative to the reference's pkg/src/dynpart/). The
 * ctypes binding a maintainer adds to the reference is in INTEGRATION.md.
 */
#ifndef DGC_B200_H
#define DGC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DGC_OK 0
#define DGC_ERR_ARG -1
#define DGC_ERR_CUDA -2
#define DGC_ERR_PLAN -3 /* plan/graph mismatch, cf. sim.py:108 PlanGraphMismatch */

int dgc_version(void);
const char* dgc_last_error(void);

/* ------------------------------------------------------------------ */
/* Host: plan -> per-device layout.                  */
/* Consumes the reference plan unchanged: Plan.structure_device        */
/* (sim.py:120), chunk membership (partition.py:49-56), FusionPlan      */
/* groups (fusion.py:78-105), DynamicGraph index views                 */
/* (graphstore.py:209-221).                                           */
/* ------------------------------------------------------------------ */
typedef struct dgc_plan_view {
  int64_t n_instances;
  const int32_t* inst_entity;     /* [n_instances] global (snapshot-major) order */
  const int32_t* inst_t;          /* [n_instances] 1-based timestep */
  int64_t n_spatial_edges;
  const int32_t* spatial_edges;   /* [E,2] spatial_edge_index() order */
  int64_t n_temporal_links;
  const int32_t* temporal_links;  /* [L,2] temporal_link_index() order */
  const int32_t* structure_device;/* [n_instances] Plan.structure_device */
  const int32_t* chunk_of;        /* [n_instances] chunk id */
  int32_t n_devices;
  int64_t n_groups;               /* 0 = no fusion plan (build_plan(fuse=False)) */
  const int32_t* group_device;    /* [n_groups] in FusionPlan order */
  const int64_t* group_ptr;       /* [n_groups+1] */
  const int32_t* group_chunks;    /* chunk ids per group */
  int32_t segment_rows;           /* 0, or: group rows by snapshot, each snapshot block
                                     padded (own_gid -1) to a multiple of segment_rows
                                     (per-snapshot weights, EvolveGCN) */
} dgc_plan_view;

/* Native synthetic generator, the contract of
 * dynpart.graphstore.generate (graphstore.py:525-579) with its own random
 * stream: presence lengths from the LengthDistribution (graphstore.py:367-382)
 * until they sum to total_vertices, uniform starts, clipped-normal per-snapshot
 * edge counts renormalised by largest remainder, uniform or preferential
 * distinct-pair sampling per snapshot. Outputs (caller-allocated): presences
 * [total_vertices][2] = (entity, t) grouped by entity, t ascending; edges
 * [total_edges][3] = (t, u, v), u < v, by snapshot, sorted pairs. Returns
 * DGC_ERR_ARG for an invalid spec or a snapshot that cannot host its quota. */
#define DGC_LEN_CONSTANT 0
#define DGC_LEN_UNIFORM 1
#define DGC_LEN_BIMODAL 2
#define DGC_LEN_GEOMETRIC 3
typedef struct dgc_length_dist {
  int32_t kind;
  int32_t value, low, high, long_low, long_high;
  double long_fraction, mean;
} dgc_length_dist;
typedef struct dgc_synthetic_spec {
  int64_t total_vertices, total_edges;
  int32_t T;
  double edges_per_snapshot_mean, edges_per_snapshot_stddev;
  dgc_length_dist length;
  uint64_t rng_seed;
  int32_t preferential; /* edge_attachment == "preferential" */
} dgc_synthetic_spec;
int dgc_generate_graph(const dgc_synthetic_spec* spec, int32_t* presences, int32_t* edges,
                       int64_t* n_entities, int32_t n_threads);

typedef struct dgc_layout dgc_layout;

/* Field ids of dgc_layout_field(); all fields are int64 arrays. */
enum dgc_layout_field_id {
  DGC_F_OWN_GID = 0, DGC_F_HALO_GID, DGC_F_GROUP_PTR, DGC_F_ROW_PTR, DGC_F_COL,
  DGC_F_DEG, DGC_F_T_ROW_PTR, DGC_F_T_COL, DGC_F_KEY_ROWS, DGC_F_SEND_PTR,
  DGC_F_SEND_POS, DGC_F_RECV_PTR, DGC_F_RECV_SLOT, DGC_F_RUN_PTR, DGC_F_RUN_ROWS,
  DGC_F_RUN_PRED_GID, DGC_F_RUN_CARRY, DGC_F_SLOT_ROW, DGC_F_SLOT_MASK,
  DGC_F_SLOT_CARRY, DGC_F_TKEY_ROWS, DGC_F_TSEND_PTR, DGC_F_TSEND_POS,
  DGC_F_TRECV_PTR, DGC_F_TRECV_CARRY, DGC_F_SCALARS, DGC_F_KEY_NCUT, DGC_F_SEG_PTR,
  DGC_F_COUNT
};
/* DGC_F_SCALARS = [n_own, n_halo, n_rows, row_len, padding, naive_padding,
 *                  n_carry, loaded_rows] (loaded_rows: sim.py:339-360)
 * DGC_F_SEG_PTR = row start of each snapshot block (segment_rows > 0 only)
 * DGC_F_KEY_NCUT = cut spatial messages sourced by each boundary key
 * (MessageSet rows with src = key, costmodel.py:121-123) for the billing. */

int dgc_layout_build(const dgc_plan_view* plan, int32_t device, dgc_layout** out);
int64_t dgc_layout_field(const dgc_layout* lay, int32_t field, const int64_t** data);
void dgc_layout_free(dgc_layout* lay);

/* fusion.py:278-313 pack_sequences keyed by sequence index (FFD,
 * fusion.py:249-275). Outputs are [capacity_rows*row_len]; row_len must be
 * max(lengths). slot_seq/slot_pos = -1 on padding. */
int dgc_pack_sequences(const int32_t* lengths, int64_t n, int32_t row_len,
                       int64_t capacity_rows, int32_t* slot_seq, int32_t* slot_pos,
                       uint8_t* mask, int64_t* n_rows, int64_t* padding);

/* Chunk generation (PGC weighted label propagation), bit-exact port of
 * dynpart.partition.propagate's label computation (partition.py:200-270 with
 * _propagation_edges :138-152, _greedy_coloring :155-168, _class_argmax
 * :171-197). spatial_edges [n_spatial, 2] / temporal_links [n_temporal, 2] are
 * DynamicGraph.spatial_edge_index() / temporal_link_index() (int64, reference
 * order); spatial_weight = edge_traffic(profile, "spatial"); temporal_weights
 * [n_temporal] = _temporal_link_weights(g, profile). labels [n] out (final
 * label per instance; _build_chunk_graph turns them into chunks); rounds_run
 * and n_colors (may be NULL) report the sweeps done and colour classes. */
int dgc_propagate_labels(int64_t n, int64_t n_spatial, const int64_t* spatial_edges,
                         int64_t n_temporal, const int64_t* temporal_links, int64_t spatial_weight,
                         const int64_t* temporal_weights, int64_t size_cap, int32_t max_rounds,
                         int64_t* labels, int32_t* rounds_run, int32_t* n_colors);

/* Native bit-exact plan_spatial_fusion (fusion.py:108-203) for ONE device:
 * chunk stats (degree sums, halos over spatial edges + temporal links, inter-
 * chunk message bytes, partition.py:273-359) are derived from the graph
 * arrays and chunk_of; device_chunks = Assignment.queues[d]. Outputs: group
 * index per device chunk (groups numbered in representative-id order),
 * per-group memory_bytes and saved_bytes, group count. Returns DGC_ERR_PLAN
 * (BudgetExceededError) if one chunk alone exceeds the budget. */
int dgc_plan_spatial_fusion(int64_t n_instances, const int32_t* spatial_edges,
                            int64_t n_spatial_edges, const int32_t* temporal_links,
                            int64_t n_temporal_links, const int32_t* chunk_of, int64_t n_chunks,
                            const int32_t* device_chunks, int64_t n_device_chunks,
                            int64_t spatial_msg_bytes, int64_t temporal_msg_bytes,
                            int64_t memory_budget, int64_t bytes_per_vertex,
                            int64_t bytes_per_edge, int32_t* out_group_of_chunk,
                            int64_t* out_group_memory, int64_t* out_group_saved,
                            int64_t* n_groups_out);

/* ------------------------------------------------------------------ */
/* Device index arrays are int32 (per-device nnz < 2^31).              */
/* ------------------------------------------------------------------ */

/* K1: structure encoder aggregation (GCNConv normalisation), fp32.
 * Replaces the analytic structure cost true_cost('structure')
 * (costmodel.py:259-263, billed per fusion group sim.py:339-360,485-486).
 *   out[i] = act( dinv[i] * sum_{c in row i} dinv[c] * Y[c] + bias )
 * act bit 0: relu; bit 1: round the output to TF32 (TF32 mode). Rows in fusion-group order; ONE launch covers all
 * fusion groups of the device. bias may be NULL. The backward uses the same
 * kernel on the transposed CSR (t_row_ptr, t_col). */
int dgc_spmm_csr(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                 const float* Y, const float* bias, float* out,
                 int64_t n_rows, int32_t width, int32_t act, void* stream);

/* K1 over a row subset: rows != NULL -> the rows rows[0..n_rows); rows ==
 * NULL -> the range [row_begin, row_begin + n_rows). Same per-row arithmetic
 * and reduction order as dgc_spmm_csr (bitwise identical rows). Used to split
 * a device's rows into interior rows (no halo column; run while the boundary
 * exchange is in flight) and boundary rows (after it lands), and the
 * transposed backward into its halo block (sent back first) and own block. */
int dgc_spmm_csr_rows(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                      const float* Y, const float* bias, float* out, const int32_t* rows,
                      int64_t n_rows, int64_t row_begin, int32_t width, int32_t act,
                      void* stream);

/* K1 (as dgc_spmm_csr_rows) that also writes an fp16 copy of `out` to out16
 * (same [rows, width] layout; may be NULL): the gathered x operand of the
 * fp16 tensor-core recurrence (dgc_lstm_fwd_tc_f16x) or of the fp16 GEMMs, as
 * fp16(scale16 * out) (a power of two lifting a gradient into fp16's normal
 * range; 1 for activations); out may then be NULL. work (may be NULL): two
 * int32 zeros in device memory; on large graphs (>= 256 rows per resident
 * warp) the warps then take rows in order from this counter (the rows in
 * flight stay one compact window, so their neighbour rows stay L2-resident)
 * and the kernel leaves it zeroed. One counter pair per stream (launches
 * sharing it must be stream-ordered). */
int dgc_spmm_csr_x(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                   const float* Y, const float* bias, float* out, void* out16,
                   const int32_t* rows, int64_t n_rows, int64_t row_begin, int32_t width,
                   int32_t act, int32_t* work, float scale16, void* stream);

/* K1 over all rows with an fp16 gathered operand Y16 [rows, width] (width 32..256):
 * TF32 mode's resident fp16 features feed the layer-1 aggregation directly (no
 * fp32 copy, no expansion kernel in the input pipeline). fp32 accumulation in CSR
 * order; fp32 out and / or fp16(scale16 * out) in out16; act and work as
 * dgc_spmm_csr_x. */
int dgc_spmm_csr_h(const int32_t* row_ptr, const int32_t* col, const float* dinv,
                   const void* Y16, const float* bias, float* out, void* out16, float scale16,
                   int64_t n_rows, int32_t width, int32_t act, int32_t* work, void* stream);

/* Cap on the CTAs of the following GEMM launches (0: one per SM); returns the
 * previous cap. For two GEMMs issued on concurrent streams that stream the
 * same operand (each takes part of the machine, and the second reader of a
 * tile finds it in L2). Host-side state of the calling process. */
int32_t dgc_gemm_max_ctas(int32_t n);
/* K2: tcgen05 TF32 GEMM (TMA -> SMEM -> TMEM), fp32 storage, fp32 accumulate.
 *   C[M,N] = (accumulate ? C : 0) + op(A) op(B)  (+ bias[N]) (* (relu_src > 0))
 *   a_mn = 0: A is [M,K] (row stride lda); a_mn = 1: A stored as [K,M] (A^T)
 *   b_mn = 1: B is [K,N] (row stride ldb); b_mn = 0: B stored as [N,K] (B^T)
 * precision: 1 = TF32, 3 = 3xTF32 (fp32-accurate; the parity mode).
 * k_splits > 1 splits K over CTAs, writes partials to `partial`
 * [splits, M, N] and reduces them in fixed order (deterministic). With
 * precision 3 the library raises splits so that no TMEM accumulation chain
 * exceeds 16 k-blocks (512 K): the tensor-core fp32 accumulator truncates,
 * which biases long chains. dgc_gemm_splits() returns the split count a call
 * will use, to size `partial` (splits * M * N floats).
 * accumulate: bit 0 = add into C; bit 1 = ReLU on the output; bit 2 = round the
 * output to TF32 (bits 1-2 need an unsplit K; applied after bias / relu_src).
 * Replaces the x@W / h@U products of GruCell.step (fusion.py:410-412). */
int dgc_gemm_splits(int64_t K, int32_t precision, int32_t k_splits);
int dgc_gemm_tf32(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                  int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn, int32_t b_mn,
                  int32_t precision, const float* bias, const float* relu_src,
                  int32_t accumulate, int32_t k_splits, float* partial, float* colsum_partial,
                  void* stream);
/* colsum_partial (may be NULL, needs k_splits == 1): column sums of the final
 * output per (128-row tile, TMEM quadrant): [4*ceil(M/128), N]; reduce with
 * dgc_reduce_rows -> bias gradients without re-reading C. */

/* Segmented K2 for per-snapshot weights (EvolveGCN). Exactly one of:
 *  row-segmented: seg_of_mtile [ceil(M/128)] = snapshot of each 128-row tile
 *    (rows grouped by snapshot and 128-aligned, dgc_plan_view.segment_rows);
 *    B holds b_nseg stacked matrices ([b_nseg*K, N] if b_mn else [b_nseg*N, K]);
 *  K-segmented: kitems [n_kitems, 2] = (first k-block, k-block count >= 1) work
 *    items, item_ptr [n_seg+1] = items of each segment; every item writes
 *    partial[item] [M, N]; C [n_seg*M, N] (row stride ldc) = per-segment sums
 *    in fixed order (segments without items -> 0): per-snapshot dW = X_t^T dY_t. */
int dgc_gemm_tf32_segmented(const float* A, int64_t lda, const float* B, int64_t ldb, float* C,
                            int64_t ldc, int64_t M, int64_t N, int64_t K, int32_t a_mn,
                            int32_t b_mn, int32_t precision, const float* bias,
                            const float* relu_src, const int32_t* seg_of_mtile, int32_t b_nseg,
                            const int32_t* kitems, int32_t n_kitems, const int32_t* item_ptr,
                            int32_t n_seg, float* partial, float* colsum_partial, int32_t act,
                            void* stream);
/* act: bit 0 ReLU, bit 1 TF32-round the output (row-segmented calls; as bits 1-2
 * of dgc_gemm_tf32's accumulate). */

/* Stacked-A GEMM: op(A) = [op(A0) ; op(A1)] along M (rows [0, M0) from A0,
 * [M0, M) from A1; M0 % 128 == 0), every other argument as dgc_gemm_tf32.
 * One launch for the two LSTM weight gradients that share B = dgx:
 * [dWx ; dU] = [x ; h_in]^T dgx, so the 4H-wide dgx is streamed once (the
 * split-K CTAs of both row tiles read each B k-block concurrently, L2 dedups).
 * C is [M, N] (dWx and dU are adjacent in the flat gradient buffer). */
int dgc_gemm_tf32_stacked_a(const float* A0, int64_t lda0, const float* A1, int64_t lda1,
                            int64_t M0, const float* B, int64_t ldb, float* C, int64_t ldc,
                            int64_t M, int64_t N, int64_t K, int32_t a_mn, int32_t b_mn,
                            int32_t precision, int32_t k_splits, float* partial, void* stream);

/* K2 with fp16 operands (kind::f16, the same 10-bit mantissa as TF32; fp32
 * accumulation and C): C = alpha * op(A) op(B) (+ bias) (* (relu_src > 0)),
 * alpha undoing a power-of-two operand scale exactly (the BPTT's fp16 dgx is
 * S * dgx). Majorness, split-K, accumulate and colsum as dgc_gemm_tf32; A and
 * B are fp16 with row strides lda / ldb in elements (multiples of 8); an
 * MN-major B needs N % 64 == 0. Unsplit K only: C16 (may be NULL) receives fp16(c16_scale * C)
 * of the final C (after bias / activation / mask; row stride ldc16) -- the next fp16 operand,
 * c16_scale a power of two for gradients -- and with C == NULL it is the only output; relu16
 * (may be NULL) is an fp16 ReLU-mask source (row stride ldr16) in place of relu_src. The stacked
 * form = dgc_gemm_tf32_stacked_a. */
int dgc_gemm_f16(const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                 int64_t M, int64_t N, int64_t K, int32_t a_mn, int32_t b_mn, float alpha,
                 const float* bias, const float* relu_src, int32_t accumulate, int32_t k_splits,
                 float* partial, float* colsum_partial, void* C16, int64_t ldc16, float c16_scale,
                 const void* relu16, int64_t ldr16, void* stream);
int dgc_gemm_f16_stacked_a(const void* A0, int64_t lda0, const void* A1, int64_t lda1, int64_t M0,
                           const void* B, int64_t ldb, float* C, int64_t ldc, int64_t M, int64_t N,
                           int64_t K, int32_t a_mn, int32_t b_mn, float alpha, int32_t k_splits,
                           float* partial, void* stream);

/* EvolveGCN-O weight evolution (matrix GRU in the reference gate form of
 * GruCell.step, fusion.py:409-413, input = hidden = W_{t-1}):
 *   R = s(S_r W + B_r), Z = s(S_z W + B_z), C = tanh(P_c W + Q_c (R*W) + B_c),
 *   W_t = (1-Z)*C + Z*W_{t-1}.  W, B_* [Fl, Hl]; S_r, S_z, P_c, Q_c [Fl, Fl].
 * fwd and bwd take the gate matrices as they are; fwd writes Wstack [T+1, Fl, Hl]
 * (Wstack[0] = W0) and saves r, z, c, w_prev, r*w_prev laid out [Fl, T, Hl].
 * bwd takes dW_direct [T, Fl, Hl] (d loss / d W_t
 * from the snapshot-t GCN rows); writes dW0 [Fl, Hl], pre-activation grads
 * da_r, da_z, da_c [Fl, T, Hl] (then dS_r = da_r w^T etc. are K2 GEMMs with
 * K = T*Hl) and the bias grads dB_* [Fl, Hl]. flags bit 0: TF32-round saves. */
int dgc_evolve_fwd(int32_t Fl, int32_t Hl, int32_t T, const float* W0, const float* Sr,
                   const float* Sz, const float* Pc, const float* Qc, const float* Br,
                   const float* Bz, const float* Bc, float* Wstack, float* sv_r, float* sv_z,
                   float* sv_c, float* sv_w, float* sv_rw, int32_t flags, void* stream);
int dgc_evolve_bwd(int32_t Fl, int32_t Hl, int32_t T, const float* Sr, const float* Sz,
                   const float* Pc, const float* Qc, const float* sv_r, const float* sv_z,
                   const float* sv_c, const float* sv_w, const float* dW_direct, float* dW0,
                   float* da_r, float* da_z, float* da_c, float* dBr, float* dBz, float* dBc,
                   int32_t flags, void* stream);

/* K3/K4: masked recurrent time encoder over FFD-packed runs.
 * cell: 0 = GRU in the reference form of GruCell.step (fusion.py:409-413),
 *       1 = LSTM (same conventions). Gate order GRU (r,z,c), LSTM (i,f,g,o).
 *       | DGC_RNN_ROUND_TF32 (0x100): store GEMM-operand outputs (h, r*h, dgx)
 *       rounded to TF32 (TF32 mode).
 * gx [n_inst, G*H] = x Wx + b (precomputed by K2), U [H, G*H].
 * slot_row/slot_carry [R*L] int32 (-1 = none), slot_mask [R*L] uint8: the
 * carry mask of gru_forward_masked (fusion.py:457-462). A run start with a
 * remote predecessor loads carry[slot_carry] (h | c for LSTM) instead of 0.
 * h_out/c_out rows have stride ld_out (LSTM: one [n_inst, 2H] h|c buffer). The H = 128
 * cluster kernels write c_out only at the last slot of each run (the carry rows).
 * save [n_inst, dgc_rnn_save_floats] per-instance activations (instance order:
 * GRU [h_in, r*h_in, r, z, c], LSTM [h_in, c_in, i, f, g, o, tanh(c)]).
 * The first H columns of save are the operand of dU = save[:, :H]^T dgx. */
#define DGC_RNN_ROUND_TF32 0x100
int dgc_rnn_save_floats(int32_t cell, int32_t H);
int dgc_rnn_fwd(int32_t cell, const float* gx, const float* U, const int32_t* slot_row,
                const uint8_t* slot_mask, const int32_t* slot_carry, const float* carry,
                int64_t n_rows, int32_t row_len, int32_t H, int64_t ld_out, float* h_out,
                float* c_out, float* save, void* stream);
/* Tensor-core variant of dgc_rnn_fwd (TF32 tcgen05, persistent CTA per 128
 * packed rows, h x U on the tensor cores): LSTM, H in {32, 64, 128}. Takes
 * Ut = U^T [4H, H] (K-major B operand) instead of U; same outputs. */
int dgc_rnn_fwd_tc(int32_t cell, const float* gx, const float* Ut, const int32_t* slot_row,
                   const uint8_t* slot_mask, const int32_t* slot_carry, const float* carry,
                   int64_t n_rows, int32_t row_len, int32_t H, int64_t ld_out, float* h_out,
                   float* c_out, float* save, void* stream);
/* Tensor-core LSTM forward with the input projection fused (F = H = 128, the
 * 2-CTA cluster kernel), all gate-product operands fp16 (kind::f16, the same
 * 10-bit mantissa as TF32; fp32 accumulation): x Wx + h U + b accumulate in
 * TMEM from TMA row gathers of x16 (tile::gather4 by slot_row) and the fp16 h
 * tile against this CTA's halves of Wx and U, converted once per launch into
 * resident shared memory (no weight traffic per position). x16 [n_x, 128]
 * fp16 (the layer input); Wx, U [128, 512] fp32 as the model stores them; bias
 * [512]. h_out is rounded to fp16 precision (exact in TF32), so the next
 * position's fp16 h tile equals it; h_out16 (may be NULL) receives its fp16
 * copy [n, 128] for the next layer's x16. flags bit 0 (needs h_out16): h_out
 * (fp32) is written only at run ends, like c (the fp16 copy is then the
 * layer's output; the run-end rows are the carries). Replaces the gx GEMM +
 * dgc_rnn_fwd_tc pair; save/h/c outputs as dgc_rnn_fwd_tc. */
int dgc_lstm_fwd_tc_f16x(const void* x16, int64_t n_x, const float* Wx, const float* U,
                         const float* bias, const int32_t* slot_row, const uint8_t* slot_mask,
                         const int32_t* slot_carry, const float* carry, int64_t n_rows,
                         int32_t row_len, int64_t ld_out, float* h_out, float* c_out, float* save,
                         void* h_out16, int32_t flags, void* stream);
/* 1 if dgc_lstm_fwd_tc_f16x serves this (F, H) in this process, else 0. */
int dgc_rnn_fwd_tc_fused_available(int32_t F, int32_t H);
/* Tensor-core BPTT (LSTM, H in {32,64,128}): takes U itself [H, 4H] (the
 * K-major B operand of dh = da U^T), dc_scratch [ceil(n_rows/128)*128, H]
 * floats; bias_partial [dgc_rnn_tc_tiles(n_rows, H), 4H] (may be NULL).
 * H = 128 (2-CTA cluster kernel): the recurrent product runs on kind::f16 with
 * U resident in shared memory as fp16 and da as fp16 scaled by 2^e, e = bits
 * 16..22 of cell (0: unscaled); the scale is removed exactly from dh. Size e to
 * the loss normalisation (a mean over n instances: e = round(log2 n)) so that
 * S da sits in fp16's normal range. Bit 24: dgx is written as fp16 S * dgx.
 * Bit 25 (K-split cluster kernel only): dh_out holds S * dh as fp16 (the fp16
 * readout / input-gradient GEMMs' C16 output), unscaled exactly at use. */
int dgc_rnn_bwd_tc(int32_t cell, const float* U, const int32_t* slot_row,
                   const uint8_t* slot_mask, int64_t n_rows, int32_t row_len, int32_t H,
                   const float* save, const float* dh_out, float* dgx, float* dc_scratch,
                   float* bias_partial, void* stream);
/* Row tiles of the tensor-core BPTT for this H = rows of its bias_partial:
 * 128 packed rows per tile (single-CTA kernels), or 4*rq rows per 2-CTA
 * cluster (H = 128: rq = ceil(n_rows / 296) rows per TMEM lane quadrant, so
 * the recurrence spans up to 74 clusters = all 148 SMs). */
/* Save-row width (floats) of the tensor-core LSTM kernels: 3.5 H at H = 128
 * with the cluster kernels (h_in fp32 | c_in, i, f, g, o fp16), else 7 H. */
int32_t dgc_rnn_tc_save_floats(int32_t H);
int64_t dgc_rnn_tc_tiles(int64_t n_rows, int32_t H);
/* BPTT over the same packing (Ut = U^T, [G*H, H], see dgc_transpose): dh_out [n_inst,H] -> dgx [n_inst,G*H]
 * (d pre-activations; dWx = x^T dgx, db = colsum(dgx), dx = dgx Wx^T,
 * dU = save-operand^T dgx by K2). Carries from other devices are constants. */
int dgc_rnn_bwd(int32_t cell, const float* Ut, const int32_t* slot_row, const uint8_t* slot_mask,
                int64_t n_rows, int32_t row_len, int32_t H, const float* save,
                const float* dh_out, float* dgx, float* bias_partial, void* stream);
/* bias_partial (may be NULL): per-CTA column sums of dgx,
 * [dgc_rnn_bwd_partial_rows(n_rows, H), G*H]; reduce with dgc_reduce_rows. */
int64_t dgc_rnn_bwd_partial_rows(int64_t n_rows, int32_t H);

/* K5: stale filter. dgc_stale_distance = the distance half of
 * filter_transmissions / max_cache_gap (stale.py:140-151,205-212):
 * dist[k] = ||Y[key_rows[k]] - cache[k]||_2 in fp32, fixed sequential order;
 * dmax[0] = max over keys with cached[k] (0 if none), via a fixed-order tree. */
int dgc_stale_distance(const float* Y, const int32_t* key_rows, const float* cache,
                       const uint8_t* cached, int64_t n_keys, int32_t width, float* dist,
                       float* dmax, void* stream);
/* dgc_stale_select = the decision half (stale.py:166-176): send[k] =
 * !cached[k] || dist[k] > theta (strict); sent keys refresh the cache with a
 * copy of the current row and become cached. theta < 0 sends everything. */
int dgc_stale_select(const float* Y, const int32_t* key_rows, const float* dist, float theta,
                     float* cache, uint8_t* cached, uint8_t* send, int64_t n_keys,
                     int32_t width, void* stream);

/* dgc_stale_select2: the same decision with theta = coef * dmax[0] read from
 * device memory (dmax = the MAX all-reduce of dgc_stale_distance's D_r;
 * threshold() of stale.py:97-108 is D_r times a factor the host knows at the
 * start of the epoch), compared in fp64; dmax == NULL uses `theta`. When ncut
 * != NULL, *billed += sum of ncut[k] over sent keys (the reference-billed cut
 * messages of sim.py:464-469 for this send mask). No host round trip. */
int dgc_stale_select2(const float* Y, const int32_t* key_rows, const float* dist, double theta,
                      const float* dmax, double coef, float* cache, uint8_t* cached,
                      uint8_t* send, int64_t n_keys, int32_t width, const int64_t* ncut,
                      uint64_t* billed, void* stream);

/* K6': one-buffer exchange data plane (all peers per launch). Entries =
 * the per-peer send lists concatenated peer-major: ent_key[e] = key index,
 * ent_idx[e] = position in its peer's list, ent_ptr[D+1] = peer segments.
 * A send buffer holds one record [int32 list position, 3 pad | width floats]
 * per sent entry, peer-major -> ONE all-to-allv with split p = count_p.
 * dgc_exchange_rank: stale compaction on the device (send[key] != 0):
 *   ent_slot[e] = ordinal among sent entries or -1, counts[p] per peer. */
int dgc_exchange_rank(const int32_t* ent_key, int64_t n_ent, const int32_t* ent_ptr, int32_t D,
                      const uint8_t* send, int32_t* ent_slot, int32_t* counts, void* stream);
/* record ent_slot[e] (ent_slot NULL: e) = (ent_idx[e], Y[key_rows[ent_key[e]]]) */
int dgc_exchange_pack(const float* Y, int32_t width, const int32_t* key_rows,
                      const int32_t* ent_key, const int32_t* ent_idx, const int32_t* ent_slot,
                      int64_t n_ent, float* sendbuf, void* stream);
/* received records (rcounts[p] from peer p, peer-major; at most n_max):
 * dst[rlist[rlist_ptr[p] + j]] = row, j = the record's list position */
int dgc_exchange_unpack(const float* recvbuf, int32_t width, const int32_t* rcounts, int32_t D,
                        const int32_t* rlist, const int32_t* rlist_ptr, int64_t n_max,
                        float* dst, void* stream);
/* reverse direction: backbuf[i] = dY[rlist[rlist_ptr[p] + j_i]] for the i-th
 * record received in the forward (rows only, width floats each) */
int dgc_exchange_pack_back(const float* fwd_recvbuf, int32_t width, const int32_t* rcounts,
                           int32_t D, const int32_t* rlist, const int32_t* rlist_ptr,
                           int64_t n_max, const float* dY, float* backbuf, void* stream);
/* dY[key_rows[k]] += backbuf[ent_slot[e]] over the key's entries e in
 * kent[kent_ptr[k]..kent_ptr[k+1]) (ascending peer; skipped when -1):
 * fixed-order accumulation of the returned halo gradients */
int dgc_exchange_add_back(const float* backbuf, int32_t width, const int32_t* key_rows,
                          const int32_t* kent_ptr, const int32_t* kent, const int32_t* ent_slot,
                          int64_t n_keys, float* dY, void* stream);

/* K6: exchange pack/unpack (boundary rows; bytes billed as sim.py:514-543).
 * dgc_compact_sent: out_pos = [i for i in 0..n) if send[pos[i]]] in order,
 * *count (device int32) = its length. */
int dgc_compact_sent(const int32_t* pos, int64_t n, const uint8_t* send, int32_t* out_idx,
                     int32_t* count, void* stream);
/* out[i,:] = Y[rows[idx[i]],:]  (rows/idx may be NULL = identity) */
int dgc_gather_rows(const float* Y, const int32_t* rows, const int32_t* idx, int64_t n,
                    int32_t width, float* out, void* stream);
/* dst[rows[idx[i]],:] (+)= src[i,:]  (add != 0 accumulates; indices distinct) */
int dgc_scatter_rows(const float* src, const int32_t* rows, const int32_t* idx, int64_t n,
                     int32_t width, float* dst, int32_t add, void* stream);

/* K8: softmax cross-entropy readout. dlogits = (softmax - onehot) * scale
 * (flags bit 0: rounded to TF32); loss_partial[ceil(n/256)] = per-block fp64
 * sums of -log p[label]. labels < 0 mark padding rows (no loss, zero grad). */
int dgc_softmax_xent(const float* logits, const int32_t* labels, int64_t n, int32_t C,
                     float scale, int32_t flags, float* dlogits, double* loss_partial,
                     float* dl_partial, void* stream);
/* dl_partial (may be NULL): per-block column sums of dlogits [ceil(n/256), C]. */
/* As dgc_softmax_xent (no TF32 rounding) with an fp16 copy dlogits16 =
 * fp16(scale16 * dlogits) [n, C] (the fp16 readout GEMMs' operand; scale16 a
 * power of two lifting ~1/n gradients into fp16's normal range); dlogits
 * (fp32) may be NULL. C in {8, 16, 24, 32}. */
int dgc_softmax_xent_f16(const float* logits, const int32_t* labels, int64_t n, int32_t C,
                         float scale, float* dlogits, double* loss_partial, float* dl_partial,
                         void* dlogits16, float scale16, void* stream);
/* Fused fp16 readout (LSTM model, H = 128, C in {16, 32}), one persistent
 * tcgen05 launch over 128-row tiles of h16 [n, H] (fp16, 16-B aligned rows):
 * logits = h16 Wo16 + bo (Wo16 [H, C] fp16, bo fp32), softmax cross-entropy
 * with labels (y < 0: padding), dlogits = scale (softmax - onehot); writes
 * dh16 [n, H] = fp16(scale16 * dlogits Wo^T) (the S-scaled input of
 * dgc_rnn_bwd_tc bit 25), loss_partial [4 ceil(n/128)] (fp64 per tile and TMEM
 * lane quadrant), dl_partial [4 ceil(n/128), C] (dlogits column sums per tile
 * and quadrant: the bo gradient)
 * and dwo_partial [dgc_readout_f16_grid(n), H, C] (per-CTA dWo sums; reduce the
 * rows with dgc_reduce_rows). Replaces logits GEMM + dgc_softmax_xent_f16 +
 * dWo GEMM + dh GEMM (sim.py:323-324's loss, restated in oracle/dgnn.py). */
int dgc_readout_f16(const void* h16, const void* Wo16, const float* bo, const int32_t* labels,
                    int64_t n, int32_t H, int32_t C, float scale, float scale16, void* dh16,
                    double* loss_partial, float* dl_partial, float* dwo_partial, void* stream);
int32_t dgc_readout_f16_grid(int64_t n);
/* dgc_readout_f16 for EvolveGCN-O (readout input H2 = relu(.), fp16 copy h2_16):
 * instead of S dh it writes dz2 [n, H] fp32 = dh * (H2 > 0) (the mask is the
 * input tile itself) and b2_partial [4 ceil(n/128), H] = dz2 column sums per
 * (tile, lane quadrant), the b2 gradient. Replaces the logits GEMM, the
 * softmax, the dWo GEMM and the masked dZ2 GEMM of the EvolveGCN readout. */
int dgc_readout_f16_evolve(const void* h2_16, const void* Wo16, const float* bo,
                           const int32_t* labels, int64_t n, int32_t H, int32_t C, float scale,
                           float scale16, float* dz2, float* b2_partial, double* loss_partial,
                           float* dl_partial, float* dwo_partial, void* stream);
/* out[j] (+)= sum_r partial[r, j] in fixed row order (deterministic). */
int dgc_reduce_rows(const float* partial, int64_t rows, int32_t width, float* out,
                    int32_t accumulate, void* stream);
/* n_jobs (<= 8) row reductions out_j[c] = sum_r partial_j[r, c] in two launches,
 * bitwise equal to separate dgc_reduce_rows calls (host arrays of pointers /
 * sizes; accumulate not supported). */
int dgc_reduce_rows_batched(int32_t n_jobs, const float* const* partials, const int64_t* rows,
                            const int32_t* widths, float* const* outs, void* stream);
/* out[i] = in[i] rounded to the nearest TF32 (weights / inputs of TF32 mode) */
/* TF32 input pipeline: n values (n % 4 == 0) shipped as 3 bytes each (the top
 * three bytes of the fp32 after round-to-nearest-away to TF32, whose low byte is
 * zero) -> fp32; bit-identical to dgc_round_tf32 of the original values.
 * in: 4-byte aligned, out: 16-byte aligned. */
int dgc_unpack_tf32x24(const uint8_t* in, float* out, int64_t n, void* stream);
int dgc_round_tf32(const float* in, float* out, int64_t n, void* stream);
/* out[i] = fp16(in[i]) (round to nearest): the fp16 weight copies of the
 * fp16-operand GEMMs. */
int dgc_to_f16(const float* in, void* out, int64_t n, void* stream);
/* TF32 mode's features are consumed at fp16 precision when they fit its range
 * (the same 10-bit mantissa): out = fp32(fp16_rn(in)); the host ships them as
 * fp16 (2 bytes per value) and dgc_unpack_f16 expands them (n % 8 == 0,
 * 16-byte aligned) bit-identically to dgc_round_f16 on the device. */
int dgc_round_f16(const float* in, float* out, int64_t n, void* stream);
int dgc_unpack_f16(const void* in, float* out, int64_t n, void* stream);
/* Deterministic column sums out[j] (+)= sum_i X[i, j] (bias gradients);
 * scratch >= 296*width floats (<= 2 row blocks per SM). */
int dgc_colsum(const float* X, int64_t n, int32_t width, int64_t ld, float* out,
               int32_t accumulate, float* scratch, void* stream);
/* dZ = dH * (H > 0) elementwise */
int dgc_relu_bwd(const float* dH, const float* H, float* dZ, int64_t n, void* stream);

/* out[c, r] = in[r, c] (fp32, tiled through shared memory) */
int dgc_transpose(const float* in, int64_t rows, int64_t cols, float* out, void* stream);

/* Optimizers over the flat parameter buffer (after the K7 all-reduce). */
int dgc_sgd(float* p, const float* g, float* mom, int64_t n, float lr, float momentum,
            void* stream);
int dgc_adam(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1,
             float beta2, float eps, int32_t step, void* stream);
/* Adam with the (already incremented) step count read from device memory, so
 * an epoch can be captured once in a CUDA graph and replayed. */
int dgc_adam_dev(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1,
                 float beta2, float eps, const int32_t* step_dev, void* stream);
/* dgc_adam_dev that also refreshes the step's parameter mirrors in the same
 * pass: p_r = TF32 round-to-nearest-away of the updated p, p16 = fp16(p_r)
 * (each may be NULL) -- one launch instead of adam + round_tf32 + to_f16. */
int dgc_adam_dev_mirror(float* p, const float* g, float* m, float* v, int64_t n, float lr,
                        float beta1, float beta2, float eps, const int32_t* step_dev, float* p_r,
                        void* p16, void* stream);
/* End of a training step: loss_out[0] = sum of loss_partial[0..n) (fp64, fixed
 * order, one block) and, when step_dev is non-NULL, ++*step_dev (the device
 * step count a CUDA-graph-replayed Adam reads). */
/* bytes of ptr set to zero on the stream (cudaMemsetAsync: a memset node, not a
 * kernel, inside a captured step) */
int dgc_zero_async(void* ptr, int64_t bytes, void* stream);
int dgc_epoch_finish(const double* loss_partial, int64_t n, double* loss_out, int32_t* step_dev,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif
