/* strata_oracle.c — plain-C restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * Header: oracle/strata_oracle.h (states who may call this and how it is pinned).
 * Every function cites the reference lines it restates (paths relative to
 * /root/reference/proj).
 */
#include "strata_oracle.h"

#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <stdatomic.h>

/* Minimal dynamic parallel-for over [0, n) (libgomp is not in this image). */
typedef void (*row_fn)(int64_t i, void* ctx);
typedef struct { row_fn fn; void* ctx; int64_t n, grain; atomic_llong next; } par_job;

static void* par_worker(void* arg) {
  par_job* j = (par_job*)arg;
  for (;;) {
    int64_t s = atomic_fetch_add(&j->next, j->grain);
    if (s >= j->n) break;
    int64_t e = s + j->grain < j->n ? s + j->grain : j->n;
    for (int64_t i = s; i < e; ++i) j->fn(i, j->ctx);
  }
  return NULL;
}

static void par_for(int64_t n, int threads, int64_t grain, row_fn fn, void* ctx) {
  par_job j;
  j.fn = fn; j.ctx = ctx; j.n = n; j.grain = grain < 1 ? 1 : grain;
  atomic_init(&j.next, 0);
  if (threads <= 1 || n <= grain) { par_worker(&j); return; }
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, par_worker, &j);
  par_worker(&j);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* common.hpp:58-66 */
static int ceil_log2_i64(int64_t x) {
  int i = 0;
  int64_t v = 1;
  while (v < x) {
    v <<= 1;
    ++i;
  }
  return i;
}

static int64_t ceil_div_i64(int64_t a, int64_t b) { return (a + b - 1) / b; }

/* Reference accumulate (interp.cpp:88-94): float store of (double acc + double product). */
static inline float acc_ref(float acc, double prod) { return (float)((double)acc + prod); }

/* Columns of row i inside [lo, hi): the row is sorted, so this is a contiguous run. */
static void row_range(const int32_t* indptr, const int32_t* indices, int64_t i, int64_t lo,
                      int64_t hi, int64_t* q0, int64_t* q1) {
  int64_t a = indptr[i], b = indptr[i + 1];
  int64_t s = a, e = a;
  /* storage.cpp:291-297 filters the row in CSR order; sorted => one run */
  while (s < b && indices[s] < lo) ++s;
  e = s;
  while (e < b && indices[e] < hi) ++e;
  *q0 = s;
  *q1 = e;
}

int or_hyb_count(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                 int c, int k, int64_t* seg_count, int64_t* nnz_count) {
  if (c < 1 || k < 0) return 6; /* storage.cpp:273 Usage */
  int64_t nb = (int64_t)c * (k + 1);
  memset(seg_count, 0, sizeof(int64_t) * nb);
  if (nnz_count) memset(nnz_count, 0, sizeof(int64_t) * nb);
  int64_t part_w = ceil_div_i64(cols, c); /* storage.cpp:280 */
  int64_t cap = (int64_t)1 << k;
  for (int p = 0; p < c; ++p) {
    int64_t lo = p * part_w, hi = (p + 1) * part_w < cols ? (p + 1) * part_w : cols;
    for (int64_t i = 0; i < rows; ++i) {
      int64_t q0, q1;
      row_range(indptr, indices, i, lo, hi, &q0, &q1);
      int64_t l = q1 - q0;
      if (l == 0) continue;                      /* :299 */
      if (l > cap) {                             /* :301-309 */
        seg_count[p * (k + 1) + k] += ceil_div_i64(l, cap);
        if (nnz_count) nnz_count[p * (k + 1) + k] += l;
      } else {                                   /* :310-314 */
        int b = l <= 1 ? 0 : ceil_log2_i64(l);
        seg_count[p * (k + 1) + b] += 1;
        if (nnz_count) nnz_count[p * (k + 1) + b] += l;
      }
    }
  }
  return 0;
}

/* Write one segment (build_ell_bucket, storage.cpp:250-262): real slots then pad with the
 * segment's last real column and value 0. */
static void put_segment(int32_t* J, float* V, int64_t r, int64_t w, const int32_t* cols,
                        const float* vals, int64_t len) {
  int32_t pad = 0;
  for (int64_t s = 0; s < len; ++s) {
    J[r * w + s] = cols[s];
    V[r * w + s] = vals[s];
    pad = cols[s];
  }
  for (int64_t s = len; s < w; ++s) {
    J[r * w + s] = pad;
    V[r * w + s] = 0.0f;
  }
}

int or_hyb_fill(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                const float* vals, int c, int k, int32_t** I_idx, int32_t** J_idx, float** V) {
  if (c < 1 || k < 0) return 6;
  int64_t nb = (int64_t)c * (k + 1);
  int64_t* fill = (int64_t*)calloc((size_t)nb, sizeof(int64_t));
  int64_t part_w = ceil_div_i64(cols, c);
  int64_t cap = (int64_t)1 << k;
  for (int p = 0; p < c; ++p) {
    int64_t lo = p * part_w, hi = (p + 1) * part_w < cols ? (p + 1) * part_w : cols;
    for (int64_t i = 0; i < rows; ++i) {
      int64_t q0, q1;
      row_range(indptr, indices, i, lo, hi, &q0, &q1);
      int64_t l = q1 - q0;
      if (l == 0) continue;
      if (l > cap) {
        int64_t bin = p * (k + 1) + k;
        for (int64_t off = 0; off < l; off += cap) {
          int64_t end = off + cap < l ? off + cap : l;
          int64_t r = fill[bin]++;
          I_idx[bin][r] = (int32_t)i;
          put_segment(J_idx[bin], V[bin], r, cap, indices + q0 + off, vals + q0 + off, end - off);
        }
      } else {
        int b = l <= 1 ? 0 : ceil_log2_i64(l);
        int64_t bin = p * (k + 1) + b;
        int64_t r = fill[bin]++;
        I_idx[bin][r] = (int32_t)i;
        put_segment(J_idx[bin], V[bin], r, (int64_t)1 << b, indices + q0, vals + q0, l);
      }
    }
  }
  free(fill);
  return 0;
}

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

int64_t or_csr_to_bsr(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                      const float* vals, int64_t b, int32_t* jo_indptr, int32_t* jo_indices,
                      float* bvals) {
  (void)cols;
  int64_t mb = ceil_div_i64(rows, b);
  /* storage.cpp:144-157: sorted unique block columns per block row */
  int64_t total = 0;
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(indptr[rows] + 1));
  for (int64_t br = 0; br < mb; ++br) {
    int64_t r0 = br * b, r1 = (br + 1) * b < rows ? (br + 1) * b : rows;
    int64_t n = 0;
    for (int64_t i = r0; i < r1; ++i)
      for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) tmp[n++] = (int32_t)(indices[q] / b);
    qsort(tmp, (size_t)n, sizeof(int32_t), cmp_i32);
    int64_t u = 0;
    for (int64_t q = 0; q < n; ++q)
      if (q == 0 || tmp[q] != tmp[q - 1]) tmp[u++] = tmp[q];
    if (jo_indices)
      for (int64_t q = 0; q < u; ++q) jo_indices[total + q] = tmp[q];
    total += u;
    if (jo_indptr) {
      if (br == 0) jo_indptr[0] = 0;
      jo_indptr[br + 1] = (int32_t)total;
    }
  }
  free(tmp);
  if (!jo_indptr || !jo_indices || !bvals) return total;
  if (mb == 0) jo_indptr[0] = 0;
  memset(bvals, 0, sizeof(float) * (size_t)(total * b * b));
  /* storage.cpp:175-183: scatter via lower_bound within the block row */
  for (int64_t i = 0; i < rows; ++i) {
    int64_t br = i / b;
    for (int64_t q = indptr[i]; q < indptr[i + 1]; ++q) {
      int32_t bc = (int32_t)(indices[q] / b);
      int64_t lo = jo_indptr[br], hi = jo_indptr[br + 1];
      while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (jo_indices[mid] < bc) lo = mid + 1; else hi = mid;
      }
      bvals[lo * b * b + (i % b) * b + (indices[q] % b)] = vals[q];
    }
  }
  return total;
}

int or_csr_to_ell(int64_t rows, int64_t cols, const int32_t* indptr, const int32_t* indices,
                  const float* vals, int64_t w, int32_t* j_indices, float* evals,
                  int64_t* bad_row) {
  if (w < 1 || w > cols) return 6; /* storage.cpp:191-193 */
  for (int64_t i = 0; i < rows; ++i)
    if (indptr[i + 1] - indptr[i] > w) { /* :194-199 */
      if (bad_row) *bad_row = i;
      return 4;
    }
  for (int64_t i = 0; i < rows; ++i) /* :213-223: empty rows pad with column 0 */
    put_segment(j_indices, evals, i, w, indices + indptr[i], vals + indptr[i],
                indptr[i + 1] - indptr[i]);
  return 0;
}

int or_hyb_auto_k(int64_t rows, int64_t nnz) {
  if (rows == 0 || nnz == 0) return 0; /* storage.cpp:561-565 */
  int64_t avg = ceil_div_i64(nnz, rows);
  return ceil_log2_i64(avg < 1 ? 1 : avg);
}

typedef struct {
  int64_t m, n, d, b;
  const int32_t *indptr, *indices;
  const float *A, *X, *Y;
  float* out;
  const double *Ad, *Xd, *Yd;
  double* outd;
} row_ctx;

static void spmm_csr_row(int64_t i, void* p) {
  const row_ctx* c = (const row_ctx*)p;
  float* y = c->out + i * c->d;
  for (int64_t kk = 0; kk < c->d; ++kk) y[kk] = 0.0f; /* interp.cpp:584-587 zero-init */
  for (int64_t q = c->indptr[i]; q < c->indptr[i + 1]; ++q) {
    double a = (double)c->A[q];
    const float* x = c->X + (int64_t)c->indices[q] * c->d;
    for (int64_t kk = 0; kk < c->d; ++kk) y[kk] = acc_ref(y[kk], a * (double)x[kk]);
  }
}

void or_spmm_csr_refnum(int64_t m, int64_t d, const int32_t* indptr, const int32_t* indices,
                        const float* A, const float* X, float* Y, int threads) {
  row_ctx c = {m, 0, d, 0, indptr, indices, A, X, NULL, Y, NULL, NULL, NULL, NULL};
  par_for(m, threads, 64, spmm_csr_row, &c);
}

void or_spmm_hyb_refnum(int64_t m, int64_t d, int nparts, const int64_t* part_rows,
                        const int64_t* part_width, int32_t* const* I, int32_t* const* J,
                        float* const* V, const float* X, float* Y) {
  memset(Y, 0, sizeof(float) * (size_t)(m * d));
  for (int p = 0; p < nparts; ++p) { /* transform.cpp:384-386 rule order */
    int64_t w = part_width[p];
    for (int64_t r = 0; r < part_rows[p]; ++r) {
      float* y = Y + (int64_t)I[p][r] * d;
      for (int64_t s = 0; s < w; ++s) {
        double a = (double)V[p][r * w + s]; /* pad slots multiply by 0.0, not skipped */
        const float* x = X + (int64_t)J[p][r * w + s] * d;
        for (int64_t kk = 0; kk < d; ++kk) y[kk] = acc_ref(y[kk], a * (double)x[kk]);
      }
    }
  }
}

static void spmm_f64_row(int64_t i, void* p) {
  const row_ctx* c = (const row_ctx*)p;
  double* y = c->outd + i * c->d;
  for (int64_t kk = 0; kk < c->d; ++kk) y[kk] = 0.0;
  for (int64_t q = c->indptr[i]; q < c->indptr[i + 1]; ++q) {
    const double* x = c->Xd + (int64_t)c->indices[q] * c->d;
    for (int64_t kk = 0; kk < c->d; ++kk) y[kk] += c->Ad[q] * x[kk];
  }
}

void or_spmm_csr_f64(int64_t m, int64_t d, const int32_t* indptr, const int32_t* indices,
                     const double* A, const double* X, double* Y, int threads) {
  row_ctx c = {m, 0, d, 0, indptr, indices, NULL, NULL, NULL, NULL, A, X, NULL, Y};
  par_for(m, threads, 64, spmm_f64_row, &c);
}

/* kernels.cpp:125-135: B[ij] += (A[ij]*X[i,k])*Y[k,j], fused ij, k inner; Y is [d][n] */
static void sddmm_row(int64_t i, void* p) {
  const row_ctx* c = (const row_ctx*)p;
  for (int64_t q = c->indptr[i]; q < c->indptr[i + 1]; ++q) {
    float b = 0.0f;
    int64_t j = c->indices[q];
    for (int64_t kk = 0; kk < c->d; ++kk)
      b = acc_ref(b, ((double)c->A[q] * (double)c->X[i * c->d + kk]) * (double)c->Y[kk * c->n + j]);
    c->out[q] = b;
  }
}

void or_sddmm_csr_refnum(int64_t m, int64_t n, int64_t d, const int32_t* indptr,
                         const int32_t* indices, const float* A, const float* X,
                         const float* Y, float* B, int threads) {
  row_ctx c = {m, n, d, 0, indptr, indices, A, X, Y, B, NULL, NULL, NULL, NULL};
  par_for(m, threads, 64, sddmm_row, &c);
}

static void sddmm_f64_row(int64_t i, void* p) {
  const row_ctx* c = (const row_ctx*)p;
  for (int64_t q = c->indptr[i]; q < c->indptr[i + 1]; ++q) {
    double b = 0.0;
    int64_t j = c->indices[q];
    for (int64_t kk = 0; kk < c->d; ++kk) b += (c->Ad[q] * c->Xd[i * c->d + kk]) * c->Yd[kk * c->n + j];
    c->outd[q] = b;
  }
}

void or_sddmm_csr_f64(int64_t m, int64_t n, int64_t d, const int32_t* indptr,
                      const int32_t* indices, const double* A, const double* X,
                      const double* Y, double* B, int threads) {
  row_ctx c = {m, n, d, 0, indptr, indices, NULL, NULL, NULL, NULL, A, X, Y, B};
  par_for(m, threads, 64, sddmm_f64_row, &c);
}

/* lowered BSR nest: io, jo, ii, ji, k (Appendix B); indptr/indices are JO_indptr/JO_indices */
static void bsr_row(int64_t io, void* p) {
  const row_ctx* c = (const row_ctx*)p;
  int64_t b = c->b, d = c->d;
  for (int64_t ii = 0; ii < b; ++ii)
    for (int64_t kk = 0; kk < d; ++kk) c->out[(io * b + ii) * d + kk] = 0.0f;
  for (int64_t q = c->indptr[io]; q < c->indptr[io + 1]; ++q)
    for (int64_t ii = 0; ii < b; ++ii)
      for (int64_t ji = 0; ji < b; ++ji) {
        double a = (double)c->A[q * b * b + ii * b + ji];
        const float* x = c->X + ((int64_t)c->indices[q] * b + ji) * d;
        float* y = c->out + (io * b + ii) * d;
        for (int64_t kk = 0; kk < d; ++kk) y[kk] = acc_ref(y[kk], a * (double)x[kk]);
      }
}

void or_bsr_spmm_refnum(int64_t mb, int64_t b, int64_t d, const int32_t* jo_indptr,
                        const int32_t* jo_indices, const float* bvals, const float* X,
                        float* Y, int threads) {
  row_ctx c = {mb, 0, d, b, jo_indptr, jo_indices, bvals, X, NULL, Y, NULL, NULL, NULL, NULL};
  par_for(mb, threads, 1, bsr_row, &c);
}

void or_rgms_refnum(int64_t R, int64_t m, int64_t din, int64_t dout, const int32_t* i_indptr,
                    const int32_t* i_indices, const int32_t* j_indptr, const int32_t* j_indices,
                    const float* A, const float* X, const float* W, float* Y) {
  memset(Y, 0, sizeof(float) * (size_t)(m * dout));
  /* kernels.cpp:154-165: r, i, j, k, l; value (A*X)*W */
  for (int64_t r = 0; r < R; ++r)
    for (int64_t q = i_indptr[r]; q < i_indptr[r + 1]; ++q) {
      float* y = Y + (int64_t)i_indices[q] * dout;
      for (int64_t e = j_indptr[q]; e < j_indptr[q + 1]; ++e) {
        const float* x = X + (int64_t)j_indices[e] * din;
        for (int64_t kk = 0; kk < din; ++kk) {
          double ax = (double)A[e] * (double)x[kk];
          const float* w = W + (r * din + kk) * dout;
          for (int64_t l = 0; l < dout; ++l) y[l] = acc_ref(y[l], ax * (double)w[l]);
        }
      }
    }
}
