// capi.cu — the extern "C" boundary (include/strata_b200.h).
//
// Error behaviour mirrors the reference: strata::Error{ErrKind, msg} (common.hpp:36-53)
// becomes "return ErrKind ordinal + 1" plus a thread-local message; CUDA failures are
// STRATA_ERR_CUDA.  No entry point has a CPU fallback.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>

#include <cudaTypedefs.h>


#include "capi_internal.h"

using namespace strata_b200;

struct strata_csr_host : CsrHost {};

namespace {

thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return STRATA_OK;
  } catch (const ApiError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return STRATA_ERR_INTERNAL;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return STRATA_ERR_INTERNAL;
  }
}

void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw ApiError(code, msg);
}

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// The kernels are compiled for sm_100a only; fail loudly anywhere else.
void require_device() {
  int dev = 0;
  STRATA_CUDA_CHECK(cudaGetDevice(&dev));
  int major = 0, minor = 0;
  STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
  if (major != 10 || minor != 0)
    throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a; device is sm_" +
                                        std::to_string(major * 10 + minor));
}

const strata_hyb_impl& hyb_of(const strata_hyb* h) {
  require(h != nullptr, STRATA_ERR_USAGE, "null hyb handle");
  return *h;
}

}  // namespace

namespace strata_b200 {
void set_last_error(const std::string& msg) { g_last_error = msg; }

CUtensorMap make_tensor_map_bf16_2d(const void* base, long long rows, long long cols,
                                    int box_cols, int box_rows, CUtensorMapSwizzle swizzle) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    STRATA_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      throw ApiError(STRATA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap map;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(cols) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim,
                            gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ApiError(STRATA_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return map;
}

// Stream-ordered workspaces (cudaMallocAsync) come from the device's default pool; keep freed
// blocks cached there instead of returning them to the driver at every synchronisation, so
// per-call temporaries cost a pool hit, not a re-map.
void* workspace_alloc(size_t bytes, cudaStream_t s) {
  static bool configured[64] = {};
  int dev = 0;
  STRATA_CUDA_CHECK(cudaGetDevice(&dev));
  if (dev < 64 && !configured[dev]) {
    cudaMemPool_t pool;
    STRATA_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = UINT64_MAX;
    STRATA_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    configured[dev] = true;
  }
  void* p = nullptr;
  STRATA_CUDA_CHECK(cudaMallocAsync(&p, std::max<size_t>(bytes, 1), s));
  return p;
}

long long l2_bytes() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrL2CacheSize, dev);
  return n > 0 ? n : (126ll << 20);
}

int num_sms() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}
}  // namespace strata_b200

extern "C" {

const char* strata_last_error(void) { return g_last_error.c_str(); }

int strata_abi_version(void) { return 100; }

int strata_device_ok(void) {
  return guard([] { require_device(); }) == STRATA_OK ? 1 : 0;
}

// ---- synthetic inputs ----------------------------------------------------------------
int strata_generate_csr(const char* kind, int64_t n, int64_t m, double density, int64_t band,
                        int64_t block, double avg_degree, uint64_t seed, strata_csr_host** out) {
  return guard([&] {
    require(kind && out, STRATA_ERR_USAGE, "null argument");
    require(n >= 0 && m >= 0, STRATA_ERR_USAGE, "matrix dims must be >= 0");
    auto* h = new strata_csr_host();
    try {
      generate_csr(kind, n, m, density, band, block, avg_degree, seed, *h);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int strata_csr_host_info(const strata_csr_host* h, int64_t* rows, int64_t* cols, int64_t* nnz) {
  return guard([&] {
    require(h, STRATA_ERR_USAGE, "null handle");
    if (rows) *rows = h->rows;
    if (cols) *cols = h->cols;
    if (nnz) *nnz = h->nnz;
  });
}
const int32_t* strata_csr_host_indptr(const strata_csr_host* h) { return h ? h->indptr.data() : nullptr; }
const int32_t* strata_csr_host_indices(const strata_csr_host* h) { return h ? h->indices.data() : nullptr; }
const float* strata_csr_host_values(const strata_csr_host* h) { return h ? h->values.data() : nullptr; }
int strata_csr_host_row_order(const strata_csr_host* h, int32_t* out) {
  return guard([&] {
    require(h && out, STRATA_ERR_USAGE, "null argument");
    require(static_cast<int64_t>(h->row_order.size()) == h->rows, STRATA_ERR_USAGE,
            "row order is only recorded for the powerlaw generator");
    std::copy(h->row_order.begin(), h->row_order.end(), out);
  });
}
int strata_csr_host_destroy(strata_csr_host* h) {
  delete h;
  return STRATA_OK;
}

int strata_dense_int(int64_t count, uint64_t seed, float* out) {
  return guard([&] {
    require(count >= 0 && (count == 0 || out), STRATA_ERR_USAGE, "bad dense_int arguments");
    dense_int(count, seed, out);
  });
}

// ---- hyb -------------------------------------------------------------------------------
int strata_hyb_auto_k(int64_t rows, int64_t nnz) {
  if (rows == 0 || nnz == 0) return 0;  // storage.cpp:561-565
  int64_t avg = (nnz + rows - 1) / rows;
  int k = 0;
  for (int64_t v = 1; v < std::max<int64_t>(1, avg); v <<= 1) ++k;
  return k;
}

int strata_hyb_decompose(const int32_t* indptr, const int32_t* indices, const float* values,
                         int64_t rows, int64_t cols, int64_t nnz, int c, int k, void* stream,
                         strata_hyb** out) {
  return guard([&] {
    require(out != nullptr, STRATA_ERR_USAGE, "null output handle");
    if (c < 1 || k < 0) throw ApiError(STRATA_ERR_USAGE, "hyb requires c >= 1 and k >= 0");
    require(k <= 30, STRATA_ERR_USAGE, "hyb requires k <= 30");
    require(rows >= 0 && cols >= 0 && nnz >= 0, STRATA_ERR_USAGE, "negative dims");
    require(nnz <= INT32_MAX && rows < INT32_MAX && cols <= INT32_MAX, STRATA_ERR_CAPACITY,
            "CSR exceeds int32 index range");
    require(rows == 0 || indptr, STRATA_ERR_USAGE, "null indptr");
    require(nnz == 0 || (indices && values), STRATA_ERR_USAGE, "null CSR arrays");
    require_device();
    auto* h = new strata_hyb();
    try {
      STRATA_CUDA_CHECK(cudaGetDevice(&h->device));
      h->rows = rows;
      h->cols = cols;
      h->nnz = nnz;
      h->c = c;
      h->k = k;
      hyb_decompose_device(*h, indptr, indices, values, as_stream(stream));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int strata_hyb_num_parts(const strata_hyb* h, int* nparts) {
  return guard([&] { *nparts = static_cast<int>(hyb_of(h).parts.size()); });
}

int strata_hyb_part_info(const strata_hyb* h, int part, int* partition, int* bucket,
                         int64_t* width, int64_t* nrows, int64_t* nnz, int64_t* pad_slots,
                         int64_t* col_lo, int64_t* col_hi) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(part >= 0 && part < static_cast<int>(H.parts.size()), STRATA_ERR_LOOKUP,
            "hyb part index out of range");
    const HybPart& P = H.parts[part];
    if (partition) *partition = P.partition;
    if (bucket) *bucket = P.bucket;
    if (width) *width = P.width;
    if (nrows) *nrows = P.nrows;
    if (nnz) *nnz = P.nnz;
    if (pad_slots) *pad_slots = P.pad_slots;
    if (col_lo) *col_lo = P.col_lo;
    if (col_hi) *col_hi = P.col_hi;
  });
}

int strata_hyb_part_read(const strata_hyb* h, int part, int32_t* I_indptr, int32_t* I_indices,
                         int32_t* J_indices, float* values) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(part >= 0 && part < static_cast<int>(H.parts.size()), STRATA_ERR_LOOKUP,
            "hyb part index out of range");
    const HybPart& P = H.parts[part];
    if (I_indptr) {
      I_indptr[0] = 0;
      I_indptr[1] = static_cast<int32_t>(P.nrows);
    }
    if (I_indices)
      STRATA_CUDA_CHECK(cudaMemcpy(I_indices, H.I.p + P.row_off, sizeof(int32_t) * P.nrows,
                                   cudaMemcpyDeviceToHost));
    if (J_indices)
      STRATA_CUDA_CHECK(cudaMemcpy(J_indices, H.J.p + P.slot_off,
                                   sizeof(int32_t) * P.nrows * P.width, cudaMemcpyDeviceToHost));
    if (values)
      STRATA_CUDA_CHECK(cudaMemcpy(values, H.V.p + P.slot_off, sizeof(float) * P.nrows * P.width,
                                   cudaMemcpyDeviceToHost));
  });
}

int strata_hyb_get_part(const strata_hyb* h, int part, int* partition, int* bucket, int64_t* width,
                        int64_t* nrows, int32_t* I_indptr, int32_t* I_indices, int32_t* J_indices,
                        float* values) {
  const int rc = strata_hyb_part_info(h, part, partition, bucket, width, nrows, nullptr, nullptr,
                                      nullptr, nullptr);
  return rc != STRATA_OK ? rc : strata_hyb_part_read(h, part, I_indptr, I_indices, J_indices, values);
}

int strata_hyb_part_device(const strata_hyb* h, int part, const int32_t** I_indices,
                           const int32_t** J_indices, const float** values) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(part >= 0 && part < static_cast<int>(H.parts.size()), STRATA_ERR_LOOKUP,
            "hyb part index out of range");
    const HybPart& P = H.parts[part];
    if (I_indices) *I_indices = H.I.p + P.row_off;
    if (J_indices) *J_indices = H.J.p + P.slot_off;
    if (values) *values = H.V.p + P.slot_off;
  });
}

int strata_hyb_padding_ratio(const strata_hyb* h, double* ratio) {
  return guard([&] { *ratio = hyb_of(h).padding_ratio; });
}

int strata_hyb_dims(const strata_hyb* h, int64_t* rows, int64_t* cols, int* c, int* k) {
  return guard([&] {
    const auto& H = hyb_of(h);
    if (rows) *rows = H.rows;
    if (cols) *cols = H.cols;
    if (c) *c = H.c;
    if (k) *k = H.k;
  });
}

int strata_hyb_schedule_info(const strata_hyb* h, int64_t* slots, int64_t* chunks,
                             int64_t* crossing_runs, int64_t* empty_rows, int* launches_per_spmm) {
  return guard([&] {
    const auto& H = hyb_of(h);
    int64_t sl = 0, ch = 0, ru = 0;
    int partitions = 0, prev = -1;
    for (const auto& P : H.parts) {
      sl += P.nrows * P.width;
      ch += P.nchunks;
      ru += P.nruns;
      if (P.partition != prev) ++partitions;
      prev = P.partition;
    }
    int launches = partitions;  // one spmm_hyb_kernel per column partition
    for (const auto& R : H.fix_ranges)  // fix-up level 1 / level 2 per partition
      launches += (R.tile_end > R.tile_begin ? 1 : 0) + (R.run_end > R.run_begin ? 1 : 0);
    if (H.c == 1 && H.n_empty > 0) launches += 1;  // zero_rows_kernel (c > 1 uses a memset)
    if (slots) *slots = sl;
    if (chunks) *chunks = ch;
    if (crossing_runs) *crossing_runs = ru;
    if (empty_rows) *empty_rows = H.n_empty;
    if (launches_per_spmm) *launches_per_spmm = launches;
  });
}

int strata_hyb_row_work_balance(const strata_hyb* h, double* balance, void* stream) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(balance != nullptr, STRATA_ERR_USAGE, "null output");
    require_device();
    *balance = hyb_row_work_balance(H, as_stream(stream));
  });
}

int strata_hyb_destroy(strata_hyb* h) {
  delete h;
  return STRATA_OK;
}

// ---- SpMM / SDDMM ----------------------------------------------------------------------
int strata_spmm_hyb_f32(const strata_hyb* h, const float* X, float* Y, int64_t d, void* stream) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(d >= 1, STRATA_ERR_USAGE, "spmm: d must be >= 1");
    require((H.cols == 0 || X) && (H.rows == 0 || Y), STRATA_ERR_USAGE, "null operand");
    require_device();
    spmm_hyb_launch(H, X, &Y, 1, d, as_stream(stream));
  });
}

int strata_spmm_hyb_f32_host(const strata_hyb* h, const float* X_host, float* Y_host, int64_t d,
                             void* stream) {
  return strata_spmm_hyb_f32_host_batch(h, &X_host, &Y_host, 1, d, stream);
}

// Batched end-to-end form.  Three streams and two staging slots: the copy-in of matrix b+1
// (H2D engine) and the copy-out of matrix b-1 (D2H engine) overlap the SpMM of matrix b, so on
// a full-duplex link a batch costs max(H2D, D2H) per matrix instead of H2D + SpMM + D2H.
int strata_spmm_hyb_f32_host_batch(const strata_hyb* h, const float* const* X_host,
                                   float* const* Y_host, int64_t nbatch, int64_t d, void* stream) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(d >= 1, STRATA_ERR_USAGE, "spmm: d must be >= 1");
    require(nbatch >= 0 && (nbatch == 0 || (X_host && Y_host)), STRATA_ERR_USAGE,
            "spmm_host_batch: bad batch arguments");
    DeviceGuard dg(H.device);  // host buffers in, host buffers out: run on the handle's device
    require_device();
    if (nbatch == 0) return;
    cudaStream_t s = as_stream(stream);
    std::lock_guard<std::mutex> lock(H.stage_mu);  // the staging slots belong to the handle
    const size_t xn = static_cast<size_t>(H.cols) * d, yn = static_cast<size_t>(H.rows) * d;
    const int nslots = nbatch > 1 ? 2 : 1;
    for (int k = 0; k < nslots; ++k) {
      if (H.stage_x[k].n < xn) H.stage_x[k].alloc(xn);
      if (H.stage_y[k].n < yn) H.stage_y[k].alloc(yn);
    }
    H.e2e.ensure();
    cudaStream_t cin = H.e2e.cin, cout = H.e2e.cout;
    cudaEvent_t* ev = H.e2e.ev;
    cudaEvent_t entry = ev[0], *x_ready = ev + 1, *x_free = ev + 3, *y_ready = ev + 5,
                *y_free = ev + 7;
    STRATA_CUDA_CHECK(cudaEventRecord(entry, s));  // everything follows prior work on `s`
    STRATA_CUDA_CHECK(cudaStreamWaitEvent(cin, entry, 0));
    STRATA_CUDA_CHECK(cudaStreamWaitEvent(cout, entry, 0));
    for (int64_t b = 0; b < nbatch; ++b) {
      const int k = static_cast<int>(b % nslots);
      float* sx = H.stage_x[k].p;
      float* sy = H.stage_y[k].p;
      if (b >= nslots) STRATA_CUDA_CHECK(cudaStreamWaitEvent(cin, x_free[k], 0));
      if (xn) STRATA_CUDA_CHECK(cudaMemcpyAsync(sx, X_host[b], xn * 4, cudaMemcpyHostToDevice, cin));
      STRATA_CUDA_CHECK(cudaEventRecord(x_ready[k], cin));
      STRATA_CUDA_CHECK(cudaStreamWaitEvent(s, x_ready[k], 0));
      if (b >= nslots) STRATA_CUDA_CHECK(cudaStreamWaitEvent(s, y_free[k], 0));
      spmm_hyb_launch(H, sx, &sy, 1, d, s);
      STRATA_CUDA_CHECK(cudaEventRecord(x_free[k], s));
      STRATA_CUDA_CHECK(cudaEventRecord(y_ready[k], s));
      STRATA_CUDA_CHECK(cudaStreamWaitEvent(cout, y_ready[k], 0));
      if (yn) STRATA_CUDA_CHECK(cudaMemcpyAsync(Y_host[b], sy, yn * 4, cudaMemcpyDeviceToHost, cout));
      STRATA_CUDA_CHECK(cudaEventRecord(y_free[k], cout));
    }
    STRATA_CUDA_CHECK(cudaStreamSynchronize(cout));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  });
}

// GNN layer step (the GraphSAGE/GCN end-to-end pattern PAPER.md:457-460):
// Z = A · X · W with the sparse aggregation on the hyb SpMM and the dense transform on the
// tensor cores (gemm_tf32.cu: tcgen05 kind::tf32 with the 3xTF32 split, fp32-accurate).  The
// product is associated so the SpMM gathers the narrower feature matrix: d_out < d_in ->
// T = X·W first, then Z = A·T; otherwise Y = A·X, Z = Y·W.
int64_t strata_gnn_layer_work_floats(const strata_hyb* h, int64_t d_in, int64_t d_out) {
  if (!h || d_in < 1 || d_out < 1) return -1;
  return d_out < d_in ? h->cols * d_out : h->rows * d_in;
}

int strata_gnn_layer_f32(const strata_hyb* h, const float* X, const float* W, float* Z,
                         float* work, int64_t d_in, int64_t d_out, void* stream) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(d_in >= 1 && d_out >= 1, STRATA_ERR_USAGE, "gnn_layer: d_in and d_out must be >= 1");
    require(d_in <= INT32_MAX && d_out <= INT32_MAX, STRATA_ERR_USAGE, "gnn_layer: d_in and d_out must fit int32");
    require((H.cols == 0 || X) && (H.rows == 0 || Z) && W && work, STRATA_ERR_USAGE,
            "gnn_layer: null operand");
    require_device();
    cudaStream_t s = as_stream(stream);
    if (d_out < d_in) {  // transform, then aggregate the narrower rows
      gemm_f32_launch(X, W, work, H.cols, static_cast<int>(d_in), static_cast<int>(d_out), s);
      spmm_hyb_launch(H, work, &Z, 1, d_out, s);
    } else {             // aggregate, then transform
      spmm_hyb_launch(H, X, &work, 1, d_in, s);
      gemm_f32_launch(work, W, Z, H.rows, static_cast<int>(d_in), static_cast<int>(d_out), s);
    }
  });
}

// Dense transform on its own (the GEMM half of the GNN layer step): tcgen05 3xTF32.
int strata_gemm_f32(const float* Y, const float* W, float* Z, int64_t M, int64_t K, int64_t N,
                    void* stream) {
  return guard([&] {
    require(M >= 0 && K >= 1 && N >= 1, STRATA_ERR_USAGE, "gemm: M >= 0, K >= 1, N >= 1 required");
    require(K <= INT32_MAX && N <= INT32_MAX, STRATA_ERR_USAGE, "gemm: K and N must fit int32");
    require(M == 0 || (Y && W && Z), STRATA_ERR_USAGE, "gemm: null operand");
    require_device();
    gemm_f32_launch(Y, W, Z, M, static_cast<int>(K), static_cast<int>(N), as_stream(stream));
  });
}

int strata_spmm_hyb_f32_multi(const strata_hyb* h, const float* X, float* const* Y_dsts, int ndst,
                              int64_t d, void* stream) {
  return guard([&] {
    const auto& H = hyb_of(h);
    require(d >= 1, STRATA_ERR_USAGE, "spmm: d must be >= 1");
    require(Y_dsts != nullptr && ndst >= 1 && ndst <= STRATA_MAX_Y_DESTS, STRATA_ERR_USAGE,
            "spmm_multi: 1 to " + std::to_string(STRATA_MAX_Y_DESTS) + " output buffers");
    for (int i = 0; i < ndst; ++i) require(Y_dsts[i] != nullptr, STRATA_ERR_USAGE, "spmm_multi: null output");
    require_device();
    spmm_hyb_launch(H, X, Y_dsts, ndst, d, as_stream(stream));
  });
}

int strata_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset) {
  return guard([&] {
    require(dev_ptr && handle_out && offset, STRATA_ERR_USAGE, "ipc: null pointer");
    static_assert(sizeof(cudaIpcMemHandle_t) == STRATA_IPC_HANDLE_BYTES, "IPC handle size");
    // The handle names the whole allocation; pooled allocators hand out interior pointers, so
    // the pointer's offset from the allocation base travels with it.
    using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
    static GetRange get_range = nullptr;
    if (!get_range) {
      void* fn = nullptr;
      cudaDriverEntryPointQueryResult q;
      STRATA_CUDA_CHECK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
      require(fn && q == cudaDriverEntryPointSuccess, STRATA_ERR_CUDA, "cuMemGetAddressRange unavailable");
      get_range = reinterpret_cast<GetRange>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    require(get_range(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) == CUDA_SUCCESS,
            STRATA_ERR_CUDA, "ipc: not a device allocation");
    cudaIpcMemHandle_t hd;
    STRATA_CUDA_CHECK(cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base)));
    std::memcpy(handle_out, &hd, sizeof(hd));
    *offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(dev_ptr) - base);
  });
}

int strata_ipc_open_handle(const void* handle, void** dev_ptr) {
  return guard([&] {
    require(handle && dev_ptr, STRATA_ERR_USAGE, "ipc: null pointer");
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle, sizeof(hd));
    STRATA_CUDA_CHECK(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess));
  });
}

int strata_ipc_close(void* dev_ptr) {
  return guard([&] {
    require(dev_ptr != nullptr, STRATA_ERR_USAGE, "ipc: null pointer");
    STRATA_CUDA_CHECK(cudaIpcCloseMemHandle(dev_ptr));
  });
}

int strata_spmm_csr_f32(const int32_t* indptr, const int32_t* indices, const float* A,
                        const float* X, float* Y, int64_t rows, int64_t cols, int64_t d,
                        void* stream) {
  return guard([&] {
    (void)cols;
    require(d >= 1, STRATA_ERR_USAGE, "spmm: d must be >= 1");
    require_device();
    spmm_csr_launch(indptr, indices, A, X, Y, rows, d, as_stream(stream));
  });
}

int strata_sddmm_csr_f32(const int32_t* indptr, const int32_t* indices, const float* A,
                         const float* X, const float* Y, float* B, int64_t rows, int64_t cols,
                         int64_t nnz, int64_t d, void* stream) {
  return guard([&] {
    require(d >= 1, STRATA_ERR_USAGE, "sddmm: d must be >= 1");
    require(nnz <= INT32_MAX, STRATA_ERR_CAPACITY, "nnz exceeds int32 index range");
    require_device();
    sddmm_csr_launch(indptr, indices, A, X, Y, B, rows, cols, nnz, d, as_stream(stream));
  });
}

int strata_csr_from_coo(const int32_t* row, const int32_t* col, const float* val, int64_t nnz,
                        int64_t rows, int64_t cols, int32_t* indptr, int32_t* indices,
                        float* values, void* stream) {
  return guard([&] {
    require(nnz == 0 || (row && col && val && indices && values), STRATA_ERR_USAGE, "null array");
    require(indptr != nullptr, STRATA_ERR_USAGE, "null indptr");
    require_device();
    csr_from_coo_device(row, col, val, nnz, rows, cols, indptr, indices, values, as_stream(stream));
  });
}

int strata_ell_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                        int64_t rows, int64_t cols, int64_t w, int32_t* J_indices,
                        float* ell_values, void* stream) {
  return guard([&] {
    require(rows >= 0 && cols >= 0, STRATA_ERR_USAGE, "negative dims");
    if (w >= 1 && w <= cols && rows > 0) require_device();
    ell_from_csr_launch(indptr, indices, values, rows, cols, w, J_indices, ell_values,
                        as_stream(stream));
  });
}

// ---- multi-GPU host helper ---------------------------------------------------------------
int strata_partition_rows(const int32_t* indptr_host, int64_t rows, int parts, int64_t* bounds) {
  return guard([&] {
    require(parts >= 1 && bounds && (rows == 0 || indptr_host), STRATA_ERR_USAGE,
            "bad partition arguments");
    const int64_t nnz = rows > 0 ? indptr_host[rows] : 0;
    bounds[0] = 0;
    for (int p = 1; p < parts; ++p) {
      const int64_t target = (nnz * p) / parts;  // first row r with indptr[r] >= target
      const int32_t* it = std::lower_bound(indptr_host, indptr_host + rows + 1, target,
                                           [](int32_t a, int64_t v) { return a < v; });
      bounds[p] = std::max<int64_t>(bounds[p - 1], std::min<int64_t>(rows, it - indptr_host));
    }
    bounds[parts] = rows;
  });
}

}  // extern "C"
