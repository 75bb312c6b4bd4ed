/* strata_oracle.h — plain-C CPU restatement of the reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load liboracle.so; the product path never does.
 *
 * Parity pinned: tests/test_oracle_golden.py checks every function below against the
 * reference's own known-answer tests (proj/tests/test_storage.cpp:30-154,
 * proj/tests/test_kernels.cpp:33-103) and against the unmodified reference library built
 * in oracle/_ref (decompose_hyb / csr_to_bsr / csr_to_ell arrays bitwise; interpret()
 * outputs bitwise on integer AND real-valued f32 data).
 *
 * Numerics of the *_refnum functions follow interp.cpp:88-94 and :346-353 exactly: operands
 * are widened to double, products are formed in double, and each "+=" is
 * acc = (float)((double)acc + product).  Accumulation order per output element is the
 * reference's (ascending column within a row; relation-major for RGMS), which is why the
 * CSR-ordered loops below reproduce the hyb/BSR interpreter runs bit for bit.
 */
#ifndef STRATA_ORACLE_H
#define STRATA_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* hyb plan (storage.cpp:271-334): segments and real entries per (partition p, bucket b),
 * bin index = p*(k+1)+b.  Returns 0, or 6 (Usage) when c < 1 or k < 0. */
int or_hyb_count(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                 int c, int k, int64_t* seg_count, int64_t* nnz_count);

/* hyb fill (storage.cpp:271-334 + build_ell_bucket :229-269).  For every non-empty bin,
 * I_idx[bin] has seg_count[bin] entries and J_idx[bin] / V[bin] seg_count*2^b entries. */
int or_hyb_fill(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                const float* vals, int c, int k, int32_t** I_idx, int32_t** J_idx, float** V);

/* csr_to_bsr (storage.cpp:138-188): two calls; first with out arrays NULL returns nblocks. */
int64_t or_csr_to_bsr(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                      const float* vals, int64_t b, int32_t* jo_indptr, int32_t* jo_indices,
                      float* bvals);

/* csr_to_ell (storage.cpp:190-227).  Returns 0, 4 (Capacity: row over w, *bad_row set) or
 * 6 (Usage: w < 1 or w > cols). */
int or_csr_to_ell(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                  const float* vals, int64_t w, int32_t* j_indices, float* evals,
                  int64_t* bad_row);

/* hyb_auto_k (storage.cpp:561-565). */
int or_hyb_auto_k(int64_t rows, int64_t nnz);

/* SpMM, CSR order, reference numerics.  Y[m][d] is overwritten. */
void or_spmm_csr_refnum(int64_t m, int64_t d, const int32_t* indptr, const int32_t* indices,
                        const float* A, const float* X, float* Y, int threads);

/* SpMM over hyb parts in rule order (Appendix B nest), reference numerics. */
void or_spmm_hyb_refnum(int64_t m, int64_t d, int nparts, const int64_t* part_rows,
                        const int64_t* part_width, int32_t* const* I, int32_t* const* J,
                        float* const* V, const float* X, float* Y);

/* SpMM in double (the reference's F64 pipeline numerics). */
void or_spmm_csr_f64(int64_t m, int64_t d, const int32_t* indptr, const int32_t* indices,
                     const double* A, const double* X, double* Y, int threads);

/* SDDMM fused nest (kernels.cpp:110-136): Y is [d][n]; B[nnz] positional. */
void or_sddmm_csr_refnum(int64_t m, int64_t n, int64_t d, const int32_t* indptr,
                         const int32_t* indices, const float* A, const float* X,
                         const float* Y, float* B, int threads);
void or_sddmm_csr_f64(int64_t m, int64_t n, int64_t d, const int32_t* indptr,
                      const int32_t* indices, const double* A, const double* X,
                      const double* Y, double* B, int threads);

/* BSR SpMM nest (transform.cpp:466-483 lowered), reference numerics.  mb block rows. */
void or_bsr_spmm_refnum(int64_t mb, int64_t b, int64_t d, const int32_t* jo_indptr,
                        const int32_t* jo_indices, const float* bvals, const float* X,
                        float* Y, int threads);

/* RGMS nest over RelSparse arrays (kernels.cpp:138-167): Y[m][dout] overwritten. */
void or_rgms_refnum(int64_t R, int64_t m, int64_t din, int64_t dout, const int32_t* i_indptr,
                    const int32_t* i_indices, const int32_t* j_indptr, const int32_t* j_indices,
                    const float* A, const float* X, const float* W, float* Y);

#ifdef __cplusplus
}
#endif
#endif
