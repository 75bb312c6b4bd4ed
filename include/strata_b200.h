/* strata_b200.h — C ABI of the B200-native composable-format sparse operator path.
 *
 * Drop-in boundary for the reference `strata` kit's hot path (paths relative to
 * /root/reference/proj).  Every entry point lists the reference interface it replaces.
 * Conventions:
 *   - plain pointers and sizes only; no torch / C++ types;
 *   - device pointers are caller-owned device memory; only handles are freed here;
 *   - every call returns 0 (STRATA_OK) or the reference ErrKind ordinal + 1
 *     (include/strata/common.hpp:36-45), or STRATA_ERR_CUDA; strata_last_error() gives
 *     the message (thread-local), mirroring strata::Error{kind, what()};
 *   - calls are ordered on the caller's stream (`stream` is a cudaStream_t, may be NULL
 *     for the legacy default stream); the only host synchronisations are inside the
 *     *_decompose / *_from_csr planners (to size allocations) and the *_host e2e entry
 *     points.
 * There is no CPU fallback: without a visible sm_100 device every compute call fails with
 * STRATA_ERR_CUDA.
 */
#ifndef STRATA_B200_H
#define STRATA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: ErrKind ordinal + 1 (common.hpp:36-45) ------------------------- */
enum {
  STRATA_OK = 0,
  STRATA_ERR_VALIDATION = 1,
  STRATA_ERR_SCHEDULE = 2,
  STRATA_ERR_LOWERING = 3,
  STRATA_ERR_CAPACITY = 4,
  STRATA_ERR_LOOKUP = 5,
  STRATA_ERR_USAGE = 6,
  STRATA_ERR_EXEC = 7,
  STRATA_ERR_INTERNAL = 8,
  STRATA_ERR_CUDA = 9 /* no reference analogue: CUDA runtime / device failure */
};

/* Message of the last failing call on this thread (never NULL). */
const char* strata_last_error(void);
/* ABI version (major*10000 + minor*100 + patch). */
int strata_abi_version(void);
/* 1 if a device usable by this library (sm_100) is visible, else 0 (sets last error). */
int strata_device_ok(void);

/* ---- synthetic inputs (host) --------------------------------------------------------
 * Replaces: CooMatrix generate_matrix(kind, n, m, density, band, block, avg_degree, seed)
 *           (driver.hpp:84-85, driver.cpp:365-416) followed by build_csr(m) with F32 values
 *           (storage.cpp:89-124).  Same libstdc++ <random> calls in the same order, so the
 *           graph is identical to the reference's; emitted directly as CSR.
 * The returned arrays are owned by the handle (host memory). */
typedef struct strata_csr_host strata_csr_host;
int strata_generate_csr(const char* kind, int64_t n, int64_t m, double density, int64_t band,
                        int64_t block, double avg_degree, uint64_t seed, strata_csr_host** out);
int strata_csr_host_info(const strata_csr_host* h, int64_t* rows, int64_t* cols, int64_t* nnz);
const int32_t* strata_csr_host_indptr(const strata_csr_host* h);
const int32_t* strata_csr_host_indices(const strata_csr_host* h);
const float* strata_csr_host_values(const strata_csr_host* h);
/* powerlaw only: the generator's triplet order as rows (out[rows]); the reference's COO lists
 * row out[0]'s entries first, then out[1]'s, ... (driver.cpp:400-411).  Consumers that walk
 * the triplets, e.g. the RGCN relation split (strata_cli.cpp:70-82), replay it from this. */
int strata_csr_host_row_order(const strata_csr_host* h, int32_t* out);
int strata_csr_host_destroy(strata_csr_host* h);
/* Dense operand as the reference tuner/driver seeds it: mt19937(seed), uniform_int(-3,3),
 * row-major (tune.cpp:108-111, driver.cpp:320-321).  `out` is host float[count]. */
int strata_dense_int(int64_t count, uint64_t seed, float* out);

/* ---- hyb(c, k) decomposition (device) ------------------------------------------------
 * Replaces: HybDecomposition decompose_hyb(const TensorStorage& csr, int c, int k,
 *           const std::string& prefix)          (storage.hpp:131-132, storage.cpp:271-334)
 *           std::vector<FormatRewriteRule> hyb_rules(csr, c, k, name)
 *                                               (transform.hpp:102-103, transform.cpp:525-557)
 * Input CSR (indptr[rows+1], indices[nnz], values[nnz] f32) is DEVICE memory.  The handle
 * owns the device-resident ELL parts.  Parts are numbered exactly like
 * HybDecomposition::parts: partition-major, bucket ascending, empty (p,b) omitted. */
typedef struct strata_hyb strata_hyb;
int strata_hyb_decompose(const int32_t* indptr, const int32_t* indices, const float* values,
                         int64_t rows, int64_t cols, int64_t nnz, int c, int k, void* stream,
                         strata_hyb** out);
/* hyb_auto_k (storage.hpp:173, storage.cpp:561-565). */
int strata_hyb_auto_k(int64_t rows, int64_t nnz);
int strata_hyb_num_parts(const strata_hyb* h, int* nparts);
/* EllBucketPart fields (storage.hpp:84-91) + the ELL storage's nnz / pad_slots. */
int strata_hyb_part_info(const strata_hyb* h, int part, int* partition, int* bucket,
                         int64_t* width, int64_t* nrows, int64_t* nnz, int64_t* pad_slots,
                         int64_t* col_lo, int64_t* col_hi);
/* Bit-exact readback of one part's arrays into HOST buffers, by the reference's layout:
 * I_indptr[2] = {0, nrows}; I_indices[nrows]; J_indices[nrows*width]; values[nrows*width]
 * (build_ell_bucket, storage.cpp:229-269).  Any pointer may be NULL to skip it. */
int strata_hyb_part_read(const strata_hyb* h, int part, int32_t* I_indptr, int32_t* I_indices,
                         int32_t* J_indices, float* values);
/* The two above in one call (the readback SURVEY §8b names): EllBucketPart's partition /
 * bucket / width / nrows and the part's arrays copied to HOST buffers; any output may be NULL. */
int strata_hyb_get_part(const strata_hyb* h, int part, int* partition, int* bucket, int64_t* width,
                        int64_t* nrows, int32_t* I_indptr, int32_t* I_indices, int32_t* J_indices,
                        float* values);
/* Device views of one part (owned by the handle; valid until destroy). */
int strata_hyb_part_device(const strata_hyb* h, int part, const int32_t** I_indices,
                           const int32_t** J_indices, const float** values);
/* HybDecomposition::padding_ratio (storage.cpp:332, :559). */
int strata_hyb_padding_ratio(const strata_hyb* h, double* ratio);
int strata_hyb_dims(const strata_hyb* h, int64_t* rows, int64_t* cols, int* c, int* k);
int strata_hyb_destroy(strata_hyb* h);
/* SpMM schedule of this decomposition: ELL slots, virtual-warp chunks, split runs crossing
 * chunk boundaries, rows with no entry, and how many kernels one strata_spmm_hyb_f32 call
 * launches (used by bench.py to report gpu_launches). */
int strata_hyb_schedule_info(const strata_hyb* h, int64_t* slots, int64_t* chunks,
                             int64_t* crossing_runs, int64_t* empty_rows, int* launches_per_spmm);
/* Row-work balance of the decomposition — tune.cpp:46-76 (hyb_balance): per part, the max over
 * its ELL rows of the real (non-padding) slots divided by their mean; the worst part (>= 1).
 * Computed on the device; synchronises `stream`. */
int strata_hyb_row_work_balance(const strata_hyb* h, double* balance, void* stream);

/* ---- hyb SpMM (device) ---------------------------------------------------------------
 * Replaces: Pipeline::run_dense() / interpret(stage3, bindings) for
 *           build_matrix_pipeline(KernelOp::SpMM, m, d, F32, "hyb:c=..,k=..")
 *           (driver.cpp:163-217, interp.cpp:564-622; nest = SURVEY Appendix B).
 * X[cols][d] f32 row-major, Y[rows][d] f32 row-major (overwritten: the reference
 * zero-initialises outputs, interp.cpp:584-587).  Deterministic: identical bits on every
 * run.  Exact (bitwise equal to the reference) whenever every partial sum is exactly
 * representable in f32, e.g. the reference's integer operands; otherwise within
 * |x-y| <= 1e-5*max(|x|,|y|,1) of the F64 pipeline (driver.cpp:124-144). */
int strata_spmm_hyb_f32(const strata_hyb* h, const float* X, float* Y, int64_t d, void* stream);
/* End-to-end form: X and Y are HOST buffers (pinned for full PCIe speed); copies in and out
 * are inside the call, which returns after Y is on the host. */
int strata_spmm_hyb_f32_host(const strata_hyb* h, const float* X_host, float* Y_host, int64_t d,
                             void* stream);
/* Batched end-to-end form: nbatch independent feature matrices X_host[b] -> Y_host[b] (host,
 * pinned) through one plan.  Copy-in of matrix b+1 and copy-out of matrix b-1 overlap the SpMM
 * of matrix b (separate copy streams, two device staging slots); returns when every Y_host[b]
 * is written.  Results are identical to nbatch calls of strata_spmm_hyb_f32_host. */
int strata_spmm_hyb_f32_host_batch(const strata_hyb* h, const float* const* X_host,
                                   float* const* Y_host, int64_t nbatch, int64_t d, void* stream);

/* ---- GNN layer step: Z = A · X · W (GraphSAGE/GCN layer)
 * Sparse aggregation on the hyb SpMM, dense transform on the tensor cores (strata_gemm_f32).
 * Associated so the SpMM gathers the narrower rows: d_out < d_in computes T = X·W then Z = A·T,
 * otherwise Y = A·X then Z = Y·W.  X[cols][d_in], W[d_in][d_out], Z[rows][d_out] f32 row-major
 * (device); `work` holds strata_gnn_layer_work_floats() floats (T or Y).  Exact on integer
 * operands whose partial sums fit f32; otherwise within 1e-5 * max(|x|, |y|, 1) of the f64
 * product. */
int64_t strata_gnn_layer_work_floats(const strata_hyb* h, int64_t d_in, int64_t d_out);
int strata_gnn_layer_f32(const strata_hyb* h, const float* X, const float* W, float* Z,
                         float* work, int64_t d_in, int64_t d_out, void* stream);

/* Dense transform Z[M][N] = Y[M][K] · W[K][N] (f32, row-major, device): tcgen05.mma kind::tf32
 * with the 3xTF32 split (a = a_hi + a_lo, products a_lo·w_hi + a_hi·w_lo + a_hi·w_hi accumulated
 * in f32 in TMEM), persistent 128-row tiles, W's tile resident in shared memory.  Tensor-core
 * path for K % 32 == 0 and N % 16 == 0; other shapes run an f64-accumulating CUDA-core kernel. */
int strata_gemm_f32(const float* Y, const float* W, float* Z, int64_t M, int64_t K, int64_t N,
                    void* stream);

/* Multi-destination form — the fused SpMM + all-gather of a row-sharded multi-GPU run: every
 * output row of h (local row i) is stored to Y_dsts[0 .. ndst-1][i][0 .. d-1] (ndst <= 8).  The
 * pointers may be peers' Y replicas mapped over NVLink (strata_ipc_open_handle), pre-offset by
 * the caller to this shard's first global row, so the all-gather's traffic leaves the SMs as the
 * rows are produced instead of in a separate collective.  Stream-ordered; the caller fences the
 * ranks (e.g. a one-element NCCL all-reduce on the same stream) before reading peers' rows. */
int strata_spmm_hyb_f32_multi(const strata_hyb* h, const float* X, float* const* Y_dsts, int ndst,
                              int64_t d, void* stream);

/* CUDA IPC plumbing for the peer mapping above (one process per GPU): a 64-byte handle of the
 * device allocation holding dev_ptr plus dev_ptr's offset in it; the other process opens the
 * handle (allocation base, peer-accessible) and adds the offset. */
#define STRATA_IPC_HANDLE_BYTES 64
int strata_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset);
int strata_ipc_open_handle(const void* handle, void** dev_ptr);
int strata_ipc_close(void* dev_ptr);

/* ---- CSR SpMM (device, row-split baseline form of the same op) ---------------------
 * Replaces: build_matrix_pipeline(SpMM, ..., "csr") + interpret. */
int strata_spmm_csr_f32(const int32_t* indptr, const int32_t* indices, const float* A,
                        const float* X, float* Y, int64_t rows, int64_t cols, int64_t d,
                        void* stream);

/* ---- SDDMM (device) -----------------------------------------------------------------
 * Replaces: build_matrix_pipeline(KernelOp::SDDMM, m, d, F32, "csr") + interpret
 *           (kernels.cpp:110-136: B[ij] = sum_k A[ij]*X[i,k]*Y[k,j]).
 * X[rows][d]; Y[d][cols] (the reference's {"K","Jd"} layout, kernels.cpp:122);
 * B[nnz] positional in CSR order (overwritten). */
int strata_sddmm_csr_f32(const int32_t* indptr, const int32_t* indices, const float* A,
                         const float* X, const float* Y, float* B, int64_t rows, int64_t cols,
                         int64_t nnz, int64_t d, void* stream);

/* ---- BSR (device) ---------------------------------------------------------------------
 * Replaces: TensorStorage csr_to_bsr(csr, b, prefix) (storage.hpp:117, storage.cpp:138-188)
 *           and bsr_rule (transform.cpp:466-483).  Dims are padded up to multiples of b
 *           (driver.cpp:69-78).  Values converted to bf16 for the tensor-core SpMM and kept
 *           in f32 for bit-exact readback. */
typedef struct strata_bsr strata_bsr;
int strata_bsr_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                        int64_t rows, int64_t cols, int64_t nnz, int64_t b, void* stream,
                        strata_bsr** out);
/* mb = padded_rows/b, nb = padded_cols/b. */
int strata_bsr_info(const strata_bsr* h, int64_t* mb, int64_t* nb, int64_t* b, int64_t* nblocks,
                    int64_t* pad_slots);
/* HOST readback: JO_indptr[mb+1], JO_indices[nblocks], values[nblocks*b*b] (f32). */
int strata_bsr_read(const strata_bsr* h, int32_t* jo_indptr, int32_t* jo_indices, float* values);
int strata_bsr_destroy(strata_bsr* h);
/* BSR SpMM on tcgen05 tensor cores: Y[mb*b][d] (f32, overwritten) = A_bsr(bf16) * X
 * (X[nb*b][d] bf16 row-major).  Requires b == 32 and d in {64, 128, 256, 512}. */
int strata_bsr_spmm_bf16(const strata_bsr* h, const void* X_bf16, float* Y, int64_t d,
                         void* stream);
/* Multi-head form (batched SpMM of sparse attention): `heads` problems share the
 * block structure of h; values_bf16 [heads][nblocks][b][b] (row-major blocks, the reference's
 * A_bsr layout) or NULL (heads == 1: h's own values), X [heads][nb*b][d] bf16,
 * Y [heads][mb*b][d] f32.  Grid = block rows x heads. */
int strata_bsr_spmm_bf16_batched(const strata_bsr* h, const void* values_bf16, const void* X_bf16,
                                 float* Y, int64_t heads, int64_t d, void* stream);
/* Block-sparse SDDMM on tcgen05 (the score half of sparse attention): for every
 * stored block q of h and head hd, S[hd][q][ii][ji] = A_bsr[q][ii][ji] *
 * sum_f Q[hd][br*b + ii][f] * K[hd][JO[q]*b + ji][f].  Q [heads][mb*b][d], K [heads][nb*b][d]
 * bf16; S [heads][nblocks][b][b] f32 in the BSR block layout.  b == 32, d in {64, 128}. */
int strata_bsr_sddmm_bf16(const strata_bsr* h, const void* Q_bf16, const void* K_bf16, float* S,
                          int64_t heads, int64_t d, void* stream);

/* ---- COO ingest (device) -------------------------------------------------------------
 * Replaces: build_csr(coo, prefix) (storage.hpp:111, storage.cpp:89-124) for COO triplets
 * already in HBM: row[nnz], col[nnz] (int32), val[nnz] (f32) -> indptr[rows+1], indices[nnz],
 * values[nnz] sorted by (row, col).  STRATA_ERR_VALIDATION "coordinate out of range" or
 * "duplicate coordinate (r, c)" (the first duplicate in sorted order) exactly like the
 * reference.  Radix sort of 64-bit keys; one host sync (the validation verdict). */
int strata_csr_from_coo(const int32_t* row, const int32_t* col, const float* val, int64_t nnz,
                        int64_t rows, int64_t cols, int32_t* indptr, int32_t* indices,
                        float* values, void* stream);

/* ---- DBSR (device) -------------------------------------------------------------------
 * Replaces: csr_to_dbsr(csr, b, prefix) (storage.hpp, storage.cpp:336-370): the BSR of the
 * matrix plus its stored block rows.  Readback: IO_indices[nstored] (stored block rows),
 * JO_indptr[nstored+1], JO_indices[nblocks], values[nblocks*b*b] (f32; the BSR's block order).
 * SpMM: tcgen05 BSR kernel over the stored rows only (row map), unstored rows zero. */
typedef struct strata_dbsr strata_dbsr;
int strata_dbsr_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                         int64_t rows, int64_t cols, int64_t nnz, int64_t b, void* stream,
                         strata_dbsr** out);
int strata_dbsr_info(const strata_dbsr* h, int64_t* mb, int64_t* nb, int64_t* b, int64_t* nstored,
                     int64_t* nblocks, int64_t* pad_slots);
int strata_dbsr_read(const strata_dbsr* h, int32_t* io_indices, int32_t* jo_indptr,
                     int32_t* jo_indices, float* values);
int strata_dbsr_destroy(strata_dbsr* h);
/* Y[mb*b][d] (f32, overwritten) = A_dbsr(bf16) * X (X[nb*b][d] bf16).  b == 32, d in
 * {64, 128, 256, 512}. */
int strata_dbsr_spmm_bf16(const strata_dbsr* h, const void* X_bf16, float* Y, int64_t d,
                          void* stream);

/* ---- SR-BCRS (device) ------------------------------------------------------------------
 * Replaces: csr_to_srbcrs(csr, t, g, prefix) (storage.cpp:372-440): tile rows of t rows, their
 * distinct columns in groups of g (last group padded with the last column), values slot-major
 * [groups*g][t].  Readback: G_indptr[mb+1], JT_indices[groups*g], values[groups*g*t] (f32),
 * bit-exact.  SpMM (t == 8, g == 32): tcgen05, the 32 X rows of a group gathered by TMA
 * tile::gather4 into the A operand, the group's values as the B operand. */
typedef struct strata_srbcrs strata_srbcrs;
int strata_srbcrs_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                           int64_t rows, int64_t cols, int64_t nnz, int64_t t, int64_t g,
                           void* stream, strata_srbcrs** out);
int strata_srbcrs_info(const strata_srbcrs* h, int64_t* mb, int64_t* t, int64_t* g,
                       int64_t* groups, int64_t* pad_slots);
int strata_srbcrs_read(const strata_srbcrs* h, int32_t* g_indptr, int32_t* jt_indices, float* values);
int strata_srbcrs_destroy(strata_srbcrs* h);
/* Y[mb*t][d] (f32, overwritten) = A_srbcrs(bf16) * X (X[cols][d] bf16). */
int strata_srbcrs_spmm_bf16(const strata_srbcrs* h, const void* X_bf16, float* Y, int64_t d,
                            void* stream);

/* ---- ELL (device) ---------------------------------------------------------------------
 * Replaces: csr_to_ell(csr, w, prefix) (storage.hpp:124, storage.cpp:190-227).
 * Output device arrays J_indices[rows*w], values[rows*w] (caller-allocated).  Fails with
 * STRATA_ERR_CAPACITY (message names the row, like the reference) when a row exceeds w. */
int strata_ell_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                        int64_t rows, int64_t cols, int64_t w, int32_t* J_indices,
                        float* ell_values, void* stream);

/* ---- RGMS / RGCN (device) -----------------------------------------------------------
 * Replaces: build_rgms_pipeline(relations, d_in, d_out, F32, "hyb"/"csr") + interpret
 *           (driver.cpp:241-314, kernels.cpp:138-167):
 *           Y[i,l] = sum_r sum_j A[r,i,j] * sum_k X[j,k] * W[r,k,l].
 * The relation-major edge list is the RelSparse layout (kernels.cpp:19-62) flattened:
 * rel_ptr[R+1] (edges of relation r are [rel_ptr[r], rel_ptr[r+1])), dst[nnz] (row i),
 * src[nnz] (col j), A[nnz] f32.  X[n][d_in] bf16, W[R][d_in][d_out] bf16, Y[m][d_out] f32
 * (overwritten).  Per-relation gather -> tcgen05 GEMM (W_r in smem) -> scatter.
 * Requires (d_in, d_out) in {16,32,64} x {16,32,64,128}.  One-shot form of
 * strata_rgms_plan + strata_rgms_run_bf16 + strata_rgms_destroy (synchronises `stream`). */
int strata_rgms_bf16(const int32_t* rel_ptr, const int32_t* dst, const int32_t* src,
                     const float* A, int64_t R, int64_t m, int64_t n, int64_t nnz,
                     const void* X_bf16, const void* W_bf16, float* Y, int64_t d_in,
                     int64_t d_out, void* stream);

/* Plan / run split of the same operator — the build_rgms_pipeline (decomposition, once) /
 * interpret (per run) split of driver.cpp:241-314.  The plan copies what it needs (src, A,
 * rel_ptr) and adds each edge's position in the destination-sorted order (stable: a row's
 * edges stay in relation order) and the row pointer dptr[m+1].  A run is two kernels:
 * per-relation 128-edge tcgen05 tiles write message rows T[pos e] = A_e * (X[src e] W_r),
 * then Y[i] = sum of T rows [dptr i, dptr i+1) — deterministic, no atomics.  The T workspace
 * is taken from the stream-ordered pool per run (a plan may serve several streams). */
typedef struct strata_rgms strata_rgms;
int strata_rgms_plan(const int32_t* rel_ptr, const int32_t* dst, const int32_t* src,
                     const float* A, int64_t R, int64_t m, int64_t n, int64_t nnz,
                     strata_rgms** out, void* stream);
int strata_rgms_run_bf16(const strata_rgms* h, const void* X_bf16, const void* W_bf16, float* Y,
                         int64_t d_in, int64_t d_out, void* stream);
/* tiles_bound: upper bound on 128-edge tiles; t_bytes_per_dout: T bytes per output column. */
int strata_rgms_info(const strata_rgms* h, int64_t* tiles_bound, int64_t* t_bytes_per_dout);
int strata_rgms_destroy(strata_rgms* h);

/* RGMS over per-relation hyb parts — SURVEY §8b's strata_rgms_hyb_bf16; replaces the "hyb"
 * format of build_rgms_pipeline (driver.cpp:290-300: every relation's slice decomposed with
 * hyb_rules, k = hyb_auto_k of the slice, rules lifted to the relation axis) + interpret.
 * hybs[r] is relation r's hyb handle, any c and k, all of the same dims.  The device reads the
 * parts in place, drops the pads (a slot repeating its ELL row's previous column,
 * storage.cpp:528), rebuilds the relation-major edge list in CSR order and plans as
 * strata_rgms_plan; X / W / Y and d_in / d_out as strata_rgms_bf16.  The one-shot form
 * synchronises `stream`; the plan form may be run many times. */
int strata_rgms_plan_hyb(const strata_hyb* const* hybs, int64_t R, strata_rgms** out, void* stream);
int strata_rgms_hyb_bf16(const strata_hyb* const* hybs, int64_t R, const void* X_bf16,
                         const void* W_bf16, float* Y, int64_t d_in, int64_t d_out, void* stream);

/* ---- fused attention layer step (GAT-style) --------------------------
 * SDDMM -> row softmax -> SpMM in one pass over each row's edges (online softmax):
 *   s_ij = A_ij <Q_i, K_j>,  a_ij = softmax_j(s_ij) over the stored j of row i,
 *   Z_i = sum_j a_ij V_j     (Z_i = 0 for an empty row).
 * Q[m][d], K[n][d], V[n][d], Z[m][d] f32 row-major, d in {32, 64, 128}.  The plan (built once
 * per sparsity pattern, one host sync) splits rows longer than 256 edges into chunks merged by
 * a log-sum-exp pass.  Composes the reference's SDDMM (kernels.cpp:110-136) and SpMM
 * (kernels.cpp:85-108) nests with a softmax between them; neither scores nor weights are
 * written to HBM. */
typedef struct strata_attn_plan strata_attn_plan;
int strata_attn_plan_create(const int32_t* indptr, int64_t m, int64_t nnz, strata_attn_plan** out,
                            void* stream);
int strata_attn_plan_destroy(strata_attn_plan* p);
int strata_attn_csr_f32(const strata_attn_plan* p, const int32_t* indptr, const int32_t* indices,
                        const float* A, const float* Q, const float* K, const float* V, float* Z,
                        int64_t d, void* stream);

/* ---- Matrix Market ingest (device) ---------------------------------------------------
 * Replaces: read_matrix_market(std::istream&) and read_matrix_market_file(path)
 * (mmio.hpp:22-23, mmio.cpp:17-62).  text[bytes] holds the file's bytes in host memory; the
 * banner, comment and size lines are read on the host, the nnz entry lines are segmented and
 * parsed on the device (one thread per line; libstdc++ istream grammar for int64 / double,
 * decimals correctly rounded to double like strtod; "pattern" gives 1.0; "symmetric" pushes
 * the mirrored (j, i) of an off-diagonal entry right after it, mmio.cpp:50-51).  The handle
 * owns device triplets in the reference's order: row/col int32 (0-based), value f64 (the
 * reference's Triplet.value) and its f32 rounding (what build_csr stores for F32,
 * storage.cpp:57-61), ready for strata_csr_from_coo.  Errors are STRATA_ERR_USAGE with the
 * reference's messages for the first failing line in file order: "empty matrix market
 * stream", "unsupported matrix market header: <line>", "unsupported matrix market field: <f>",
 * "bad matrix market size line", "bad matrix market entry: <line>", "matrix market entry out of
 * range: <line>", "truncated matrix market entries", "cannot open <path>".  Two host syncs
 * (newline count, verdict). */
typedef struct strata_mtx strata_mtx;
int strata_mtx_parse(const char* text, int64_t bytes, strata_mtx** out, void* stream);
int strata_mtx_read_file(const char* path, strata_mtx** out, void* stream);
int strata_mtx_info(const strata_mtx* h, int64_t* rows, int64_t* cols, int64_t* ntriplets);
/* Device arrays owned by the handle (valid until strata_mtx_destroy). */
int strata_mtx_device(const strata_mtx* h, const int32_t** row, const int32_t** col,
                      const double** val64, const float** val32);
/* Host readback of the triplets (the reference CooMatrix.triplets), any pointer may be null. */
int strata_mtx_read(const strata_mtx* h, int64_t* row, int64_t* col, double* val);
int strata_mtx_destroy(strata_mtx* h);

/* ---- row-partitioned multi-GPU SpMM / SDDMM ---------------------------
 * Replaces: nothing in the reference (single process, single core); this is the sharded form
 * of strata_spmm_hyb_f32 / strata_sddmm_csr_f32 that §8b names
 * (strata_spmm_hyb_f32_sharded(..., const ncclComm_t*, int ndev)).  One process per GPU.
 * The plan cuts rows into `world` contiguous nnz-balanced ranges (strata_partition_rows' rule),
 * this rank's range into `chunks` sub-ranges (same rule), and decomposes each chunk to
 * hyb(c, k) on the calling device.  indices / values must stay valid while the plan lives
 * (the SDDMM reads them).  A plan's calls must be ordered (one stream at a time).
 *   SpMM: X[cols][d] replicated, Y[rows][d] a full replica on every rank.  `comm` points to
 *     this rank's ncclComm_t (rank/size checked against the plan; NULL = no reassembly: only
 *     this rank's rows of Y are written, as at world 1):
 *     chunk q of every rank is broadcast from its owner (grouped ncclBroadcast = uneven
 *     all-gather, in place) on the plan's stream, overlapping chunk q+1's SpMM.  The _p2p form
 *     instead stores every finished row into all ranks' replicas (Y_dsts[rank q] = rank q's Y,
 *     e.g. CUDA IPC mappings) from the SpMM kernel itself.
 *   SDDMM: X[rows][d], Yd[d][cols] replicated, B[nnz]: this rank's contiguous nnz range is
 *     computed; gather=1 all-gathers the ranges (grouped broadcasts), gather=0 leaves B sharded.
 * NCCL is loaded at run time (the process's libnccl.so.2, else the system one). */
#define STRATA_NCCL_ID_BYTES 128
typedef struct strata_shard_plan strata_shard_plan;
int strata_nccl_unique_id(void* id_out);
/* comm_out receives an ncclComm_t. */
int strata_nccl_comm_init(const void* id, int nranks, int rank, void* comm_out);
int strata_nccl_comm_destroy(void* comm);
int strata_shard_plan_create(const int32_t* indptr, const int32_t* indices, const float* values,
                             int64_t rows, int64_t cols, int rank, int world, int chunks, int c,
                             int k, strata_shard_plan** out, void* stream);
/* Rows [row0, row1) of chunk `chunk` of rank `rank` (chunk = -1: the rank's whole range). */
int strata_shard_plan_rows(const strata_shard_plan* p, int rank, int chunk, int64_t* row0,
                           int64_t* row1);
int strata_shard_plan_destroy(strata_shard_plan* p);
int strata_spmm_hyb_f32_sharded(const strata_shard_plan* p, const float* X, float* Y, int64_t d,
                                const void* comm, int ndev, void* stream);
int strata_spmm_hyb_f32_sharded_p2p(const strata_shard_plan* p, const float* X,
                                    float* const* Y_dsts, int ndev, int64_t d, void* stream);
int strata_sddmm_csr_f32_sharded(const strata_shard_plan* p, const float* X, const float* Yd,
                                 float* B, int64_t d, int gather, const void* comm, int ndev,
                                 void* stream);

/* ---- multi-GPU helpers (host logic, no device work) -----------------------------------
 * Row-partition into `parts` contiguous row ranges balanced by nnz: cut p is the first row
 * r with indptr[r] >= nnz*p/parts (binary search on the HOST indptr).  bounds[parts+1]. */
int strata_partition_rows(const int32_t* indptr_host, int64_t rows, int parts, int64_t* bounds);

#ifdef __cplusplus
}
#endif
#endif /* STRATA_B200_H */
