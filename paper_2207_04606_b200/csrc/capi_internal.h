// capi_internal.h — host-side internals shared by the C-ABI translation units.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/strata_b200.h"

namespace strata_b200 {

// Mirrors strata::Error{ErrKind, msg} (common.hpp:47-53); `code` is the ErrKind ordinal + 1.
struct ApiError : std::runtime_error {
  ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
  int code;
};

#define STRATA_CUDA_CHECK(expr)                                                          \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess)                                                               \
      throw ::strata_b200::ApiError(STRATA_ERR_CUDA, std::string(#expr) + ": " +         \
                                                         cudaGetErrorString(e_));        \
  } while (0)

// Once-per-device guard for cudaFuncSetAttribute (function attributes are per device, so a
// process driving several GPUs must set them on each):  static PerDeviceOnce once;
// once([&] { cudaFuncSetAttribute(...); });
struct PerDeviceOnce {
  std::atomic<uint64_t> done{0};
  template <class F>
  void operator()(F&& f) {
    int dev = 0;
    STRATA_CUDA_CHECK(cudaGetDevice(&dev));
    const uint64_t bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return;
    f();
    done.fetch_or(bit, std::memory_order_acq_rel);
  }
};

// Restores the caller's current device on scope exit (handles may live on another device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct CsrHost {
  int64_t rows = 0, cols = 0, nnz = 0;
  std::vector<int32_t> indptr, indices;
  std::vector<float> values;
  // powerlaw only: rows in the generator's triplet order (driver.cpp:400-411 emits row
  // rows[i] for i = 0..n-1), needed to replay consumers that walk the COO triplets.
  std::vector<int32_t> row_order;
};

void generate_csr(const std::string& kind, int64_t n, int64_t m, double density, int64_t band,
                  int64_t block, double avg_degree, uint64_t seed, CsrHost& out);
void dense_int(int64_t count, uint64_t seed, float* out);

// RAII device buffer.  alloc() = cudaMalloc (freed with cudaFree); alloc_async(n, s) takes
// the memory from the device's stream-ordered pool (workspace_alloc: freed blocks stay cached,
// so rebuilding a plan of the same size costs no driver mapping).  A temporary returns it with
// cudaFreeAsync on `s`; a handle-owned (persistent) buffer on the legacy stream, i.e. after all
// work queued on blocking streams — handles are destroyed by the caller after its work on them,
// as with the reference's value semantics.
void* workspace_alloc(size_t bytes, cudaStream_t s);
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  bool pooled = false;
  cudaStream_t free_stream = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(size_t count, cudaStream_t s) { alloc_async(count, s); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), pooled(o.pooled), free_stream(o.free_stream) {
    o.p = nullptr;
    o.n = 0;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    reset();
    p = o.p; n = o.n; pooled = o.pooled; free_stream = o.free_stream;
    o.p = nullptr; o.n = 0;
    return *this;
  }
  void alloc(size_t count) {
    reset();
    n = count;
    pooled = false;
    if (count) STRATA_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T)));
  }
  void alloc_async(size_t count, cudaStream_t s, bool persistent = false) {
    reset();
    n = count;
    pooled = true;
    free_stream = persistent ? nullptr : s;
    if (count) p = static_cast<T*>(workspace_alloc(count * sizeof(T), s));
  }
  void reset() {
    if (p) {
      if (pooled) cudaFreeAsync(p, free_stream); else cudaFree(p);
    }
    p = nullptr;
    n = 0;
  }
  ~DevBuf() { reset(); }
};

// Fix-up plan entries (see spmm_hyb.cu).  A crossing run's contributions are, in chunk
// order, the tail carry of its first chunk and the head carries of the following chunks.
constexpr int kFixTile = 32;  // contributions summed by one level-1 CTA
struct FixTile {
  long long carry0;  // carry row (chunk index incl. carry_off) of contribution 0
  long long out;     // >= 0: Y row (run fits one tile); < 0: -(level-2 slot + 1)
  int count;         // contributions in this tile
  int first_slot;    // carry slot of contribution 0 (1 = tail carry of the run's first chunk)
};
struct FixRun {
  long long l2_first;  // first level-2 slot of this run
  long long row;       // Y row
  int ntiles, pad_;
};
struct FixRange {
  int partition;
  long long tile_begin, tile_end, run_begin, run_end;
};

// One non-empty (partition, bucket) ELL part — EllBucketPart (storage.hpp:84-91).
struct HybPart {
  int partition = 0, bucket = 0;
  int64_t width = 1, nrows = 0, nnz = 0, pad_slots = 0, col_lo = 0, col_hi = 0;
  int64_t row_off = 0;   // into the concatenated I_indices
  int64_t slot_off = 0;  // into the concatenated J_indices / values
  // SpMM schedule: rows per chunk (power of two) and the crossing-run list for the split part
  int rpc_log2 = 0;
  int64_t nchunks = 0;
  bool may_split = false;
  int64_t nruns = 0;     // split runs that cross chunk boundaries
  int64_t carry_off = 0; // in chunks, into the carry buffer
};

// Device-resident hyb decomposition.  Layout in HBM: all parts concatenated
// in part order — one I array (int32), one J array (int32) and one value array (f32) — so the
// whole decomposition is three allocations and one SpMM launch covers every part.
struct strata_hyb_impl {
  int device = 0;
  int64_t rows = 0, cols = 0, nnz = 0;
  int c = 1, k = 0;
  double padding_ratio = 0.0;
  std::vector<HybPart> parts;
  DevBuf<int32_t> I, J;
  DevBuf<float> V;
  DevBuf<int32_t> empty_rows;  // rows with no stored entry (zeroed by SpMM when c == 1)
  int64_t n_empty = 0;
  int64_t total_chunks_carry = 0;      // chunks of split parts (carry buffer rows)
  // Fix-up plan for split runs crossing chunk boundaries (two-level fixed-shape tree):
  // level 1 sums <= kFixTile consecutive carries per tile, level 2 sums a run's tiles.
  DevBuf<FixTile> fix_tiles;
  DevBuf<FixRun> fix_runs;
  std::vector<FixRange> fix_ranges;    // per column partition, in partition order
  int64_t l2_slots = 0;
  // Per-call scratch (split-row carries [total_chunks_carry][2][d] f64, level-2 partials
  // [l2_slots][d] f64, the c > 1 f64 accumulator [rows][d]) is taken from the stream-ordered
  // pool for each SpMM, so one handle may serve several streams / threads at once.
  mutable std::mutex stage_mu;                   // guards the e2e staging buffers below
  mutable DevBuf<float> stage_x[2], stage_y[2];  // e2e staging (double-buffered)
  // The e2e path's copy streams and hand-off events, made on first use and kept with the
  // handle (creating them per call cost more than a C1-sized copy).
  struct E2eSync {
    cudaStream_t cin = nullptr, cout = nullptr;
    cudaEvent_t ev[9] = {};  // entry, x_ready[2], x_free[2], y_ready[2], y_free[2]
    void ensure() {
      if (!cin) STRATA_CUDA_CHECK(cudaStreamCreateWithFlags(&cin, cudaStreamNonBlocking));
      if (!cout) STRATA_CUDA_CHECK(cudaStreamCreateWithFlags(&cout, cudaStreamNonBlocking));
      for (auto& e : ev)
        if (!e) STRATA_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ~E2eSync() {
      for (auto& e : ev) if (e) cudaEventDestroy(e);
      if (cin) cudaStreamDestroy(cin);
      if (cout) cudaStreamDestroy(cout);
    }
  };
  mutable E2eSync e2e;  // guarded by stage_mu
};

// Kernel launchers (defined in .cu files).
void hyb_decompose_device(strata_hyb_impl& h, const int32_t* indptr, const int32_t* indices,
                          const float* values, cudaStream_t s);
// max / mean real (non-padding) slots per ELL row, worst over the parts (tune.cpp hyb_balance).
double hyb_row_work_balance(const strata_hyb_impl& h, cudaStream_t s);
// Every finished Y row is stored to each of Ydst[0 .. ndst-1] (ndst <= STRATA_MAX_Y_DESTS).
#define STRATA_MAX_Y_DESTS 8
void spmm_hyb_launch(const strata_hyb_impl& h, const float* X, float* const* Ydst, int ndst,
                     int64_t d, cudaStream_t s);
void spmm_csr_launch(const int32_t* indptr, const int32_t* indices, const float* A,
                     const float* X, float* Y, int64_t rows, int64_t d, cudaStream_t s);
// Z[M][N] = Y[M][K] · W[K][N] (f32, row-major) on tcgen05 kind::tf32 with the 3xTF32 split
// (gemm_tf32.cu); shapes outside its tiling go to an f64-accumulating CUDA-core kernel.
void gemm_f32_launch(const float* Y, const float* W, float* Z, long long M, int K, int N,
                     cudaStream_t s);
int gemm_tf32_tile_n(int K, int N);
void sddmm_csr_launch(const int32_t* indptr, const int32_t* indices, const float* A,
                      const float* X, const float* Y, float* B, int64_t rows, int64_t cols,
                      int64_t nnz, int64_t d, cudaStream_t s);

void csr_from_coo_device(const int32_t* r, const int32_t* c, const float* v, int64_t nnz,
                         int64_t rows, int64_t cols, int32_t* indptr, int32_t* indices,
                         float* values, cudaStream_t s);
void ell_from_csr_launch(const int32_t* indptr, const int32_t* indices, const float* values,
                         int64_t rows, int64_t cols, int64_t w, int32_t* J, float* V,
                         cudaStream_t s);

int num_sms();
long long l2_bytes();  // the current device's L2 capacity
// 2D bf16 TMA descriptor over a row-major [rows][cols] array with a {box_cols, box_rows} box
// (cuTensorMapEncodeTiled through the runtime's driver entry point).
CUtensorMap make_tensor_map_bf16_2d(const void* base, long long rows, long long cols,
                                    int box_cols, int box_rows, CUtensorMapSwizzle swizzle);
// Thread-local message returned by strata_last_error() (shared by every translation unit).
void set_last_error(const std::string& msg);

}  // namespace strata_b200

struct strata_hyb : strata_b200::strata_hyb_impl {};

// Device BSR (bsr.cu; the SDDMM of bsr_sddmm.cu reads it too).
struct strata_bsr {
  int device = 0;
  int64_t rows = 0, cols = 0, nnz = 0, b = 0, mb = 0, nb = 0, nblocks = 0, pad_slots = 0;
  strata_b200::DevBuf<int32_t> indptr, indices;
  strata_b200::DevBuf<float> values;           // f32, bit-exact readback
  strata_b200::DevBuf<__nv_bfloat16> vals_bf;  // tensor-core operand
};
