// strata_b200.hpp — C++ façade over the C ABI (include/strata_b200.h) that mirrors the
// reference's operator API for the hot path, so existing callers (and tests written like the
// reference's proj/tests/*.cpp) switch by changing the namespace.
//
//   reference (proj/include/strata)                 here (device-backed)
//   ---------------------------------------------   ------------------------------------------
//   Error{ErrKind, msg}          common.hpp:36-53   Error{ErrKind, msg} (+ ErrKind::Cuda)
//   CooMatrix / Triplet          storage.hpp:45-54  same
//   TensorStorage (aux map)      storage.hpp:68-90  same names: "J_indptr", "JO_indices", ...
//   build_csr                    storage.hpp:111    host, same validation (duplicates, range)
//   csr_to_bsr / csr_to_ell      storage.hpp:117/124  device kernels, host result
//   decompose_hyb / EllBucketPart / HybDecomposition  storage.hpp:84-132  device kernels
//   hyb_auto_k / padding_ratio   storage.hpp:166-173
//   generate_matrix              driver.hpp:84-85   same libstdc++ <random> sequence
//   FormatRequest::parse         driver.hpp:25-35
//   build_matrix_pipeline / build_rgms_pipeline / Pipeline::run_dense  driver.hpp:44-71
//
// Host containers are value types exactly like the reference's; the Device* classes keep the
// data resident in HBM for the fast path (no per-call copies).  Header-only; link
// libstrata_b200.so and cudart.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "strata_b200.h"

namespace strata_b200 {

// ---- errors (common.hpp:36-53) ----------------------------------------------------------
enum class ErrKind { Validation, Schedule, Lowering, Capacity, Lookup, Usage, Exec, Internal, Cuda };

class Error : public std::runtime_error {
 public:
  Error(ErrKind k, const std::string& msg) : std::runtime_error(msg), kind(k) {}
  ErrKind kind;
};

[[noreturn]] inline void fail(ErrKind k, const std::string& msg) { throw Error(k, msg); }

inline void check(int rc) {
  if (rc != STRATA_OK) throw Error(static_cast<ErrKind>(rc - 1), strata_last_error());
}

inline void cuda_check(cudaError_t e) {
  if (e != cudaSuccess) fail(ErrKind::Cuda, cudaGetErrorString(e));
}

// ---- value types (storage.hpp) ------------------------------------------------------------
using IntArray = std::vector<int32_t>;

struct Triplet {
  int64_t row = 0, col = 0;
  double value = 0.0;
};

struct CooMatrix {
  int64_t rows = 0, cols = 0;
  std::vector<Triplet> triplets;
};

struct DenseMatrix {
  int64_t rows = 0, cols = 0;
  std::vector<double> v;
  DenseMatrix() = default;
  DenseMatrix(int64_t r, int64_t c) : rows(r), cols(c), v(r * c, 0.0) {}
  double& at(int64_t i, int64_t j) { return v[i * cols + j]; }
  double at(int64_t i, int64_t j) const { return v[i * cols + j]; }
};

enum class FormatKind { Csr, Bsr, Ell, EllBucket };

struct TensorStorage {
  FormatKind kind = FormatKind::Csr;
  std::map<std::string, IntArray> aux;
  std::vector<float> values;
  int64_t rows = 0, cols = 0, nnz = 0, pad_slots = 0, block = 1, width = 0;
  const IntArray& arr(const std::string& name) const {
    auto it = aux.find(name);
    if (it == aux.end()) fail(ErrKind::Lookup, "storage has no aux array: " + name);
    return it->second;
  }
};

struct EllBucketPart {
  int partition = 0, bucket = 0;
  int64_t width = 1, col_lo = 0, col_hi = 0;
  TensorStorage ell;
};

struct HybDecomposition {
  int64_t rows = 0, cols = 0;
  int c = 1, k = 0;
  std::vector<EllBucketPart> parts;
  double padding_ratio = 0.0;
};

inline int ceil_log2(int64_t x) {
  int i = 0;
  for (int64_t v = 1; v < x; v <<= 1) ++i;
  return i;
}

// ---- device plumbing --------------------------------------------------------------------
template <class T>
class DeviceArray {
 public:
  DeviceArray() = default;
  explicit DeviceArray(size_t n) : n_(n) {
    if (n) cuda_check(cudaMalloc(&p_, n * sizeof(T)));
  }
  explicit DeviceArray(const std::vector<T>& h) : DeviceArray(h.size()) {
    if (n_) cuda_check(cudaMemcpy(p_, h.data(), n_ * sizeof(T), cudaMemcpyHostToDevice));
  }
  DeviceArray(DeviceArray&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DeviceArray& operator=(DeviceArray&& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    return *this;
  }
  DeviceArray(const DeviceArray&) = delete;
  ~DeviceArray() { if (p_) cudaFree(p_); }
  T* data() const { return p_; }
  size_t size() const { return n_; }
  std::vector<T> host() const {
    std::vector<T> h(n_);
    if (n_) cuda_check(cudaMemcpy(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// bf16 conversion for the tensor-core operands (round to nearest even).
inline uint16_t to_bf16(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFF + ((u >> 16) & 1);
  return static_cast<uint16_t>(u >> 16);
}

// ---- builders ---------------------------------------------------------------------------
// build_csr (storage.cpp:89-124): sort by (row, col), reject duplicates / out of range.
inline TensorStorage build_csr(const CooMatrix& m, const std::string& prefix = "") {
  std::vector<Triplet> t = m.triplets;
  for (const auto& e : t)
    if (e.row < 0 || e.row >= m.rows || e.col < 0 || e.col >= m.cols)
      fail(ErrKind::Validation, "coordinate out of range");
  std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  for (size_t i = 1; i < t.size(); ++i)
    if (t[i].row == t[i - 1].row && t[i].col == t[i - 1].col)
      fail(ErrKind::Validation, "duplicate coordinate (" + std::to_string(t[i].row) + ", " +
                                    std::to_string(t[i].col) + ")");
  TensorStorage s;
  s.kind = FormatKind::Csr;
  s.rows = m.rows;
  s.cols = m.cols;
  s.nnz = static_cast<int64_t>(t.size());
  IntArray indptr(m.rows + 1, 0), indices(t.size());
  s.values.resize(t.size());
  for (size_t i = 0; i < t.size(); ++i) {
    indptr[t[i].row + 1]++;
    indices[i] = static_cast<int32_t>(t[i].col);
    s.values[i] = static_cast<float>(t[i].value);
  }
  for (int64_t r = 0; r < m.rows; ++r) indptr[r + 1] += indptr[r];
  s.aux[prefix + "J_indptr"] = std::move(indptr);
  s.aux[prefix + "J_indices"] = std::move(indices);
  return s;
}

// A CSR storage resident in HBM (the input every device builder and op takes).
class DeviceCsr {
 public:
  explicit DeviceCsr(const TensorStorage& csr, const std::string& prefix = "")
      : rows(csr.rows), cols(csr.cols), nnz(csr.nnz),
        indptr(csr.arr(prefix + "J_indptr")), indices(csr.arr(prefix + "J_indices")),
        values(csr.values) {}
  int64_t rows, cols, nnz;
  DeviceArray<int32_t> indptr, indices;
  DeviceArray<float> values;
};

inline int hyb_auto_k(const TensorStorage& csr) { return strata_hyb_auto_k(csr.rows, csr.nnz); }

// Device-resident hyb(c, k) (the fast path: decompose once, run SpMM many times).
class DeviceHyb {
 public:
  DeviceHyb(const DeviceCsr& csr, int c, int k, cudaStream_t s = nullptr) {
    strata_hyb* h = nullptr;
    check(strata_hyb_decompose(csr.indptr.data(), csr.indices.data(), csr.values.data(), csr.rows,
                               csr.cols, csr.nnz, c, k, s, &h));
    h_.reset(h);
  }
  const strata_hyb* get() const { return h_.get(); }
  // Y[rows][d] = A X  (device pointers, f32)
  void spmm(const float* X, float* Y, int64_t d, cudaStream_t s = nullptr) const {
    check(strata_spmm_hyb_f32(h_.get(), X, Y, d, s));
  }
  // GNN layer step Z[rows][d_out] = A X W (X[cols][d_in], W[d_in][d_out]; device, f32).
  // `work` holds gnn_layer_work_floats(d_in, d_out) floats.
  int64_t gnn_layer_work_floats(int64_t d_in, int64_t d_out) const {
    return strata_gnn_layer_work_floats(h_.get(), d_in, d_out);
  }
  void gnn_layer(const float* X, const float* W, float* Z, float* work, int64_t d_in,
                 int64_t d_out, cudaStream_t s = nullptr) const {
    check(strata_gnn_layer_f32(h_.get(), X, W, Z, work, d_in, d_out, s));
  }
  HybDecomposition host(const std::string& prefix = "") const {
    HybDecomposition out;
    int n = 0;
    check(strata_hyb_dims(h_.get(), &out.rows, &out.cols, &out.c, &out.k));
    check(strata_hyb_padding_ratio(h_.get(), &out.padding_ratio));
    check(strata_hyb_num_parts(h_.get(), &n));
    for (int i = 0; i < n; ++i) {
      EllBucketPart p;
      int64_t nrows = 0, nnz = 0, pad = 0;
      check(strata_hyb_part_info(h_.get(), i, &p.partition, &p.bucket, &p.width, &nrows, &nnz,
                                 &pad, &p.col_lo, &p.col_hi));
      const std::string pre =
          prefix + "hyb_p" + std::to_string(p.partition) + "_b" + std::to_string(p.bucket) + "_";
      IntArray iptr(2), ii(nrows), jj(nrows * p.width);
      p.ell.values.resize(nrows * p.width);
      check(strata_hyb_part_read(h_.get(), i, iptr.data(), ii.data(), jj.data(), p.ell.values.data()));
      p.ell.kind = FormatKind::EllBucket;
      p.ell.rows = out.rows;
      p.ell.cols = out.cols;
      p.ell.nnz = nnz;
      p.ell.pad_slots = pad;
      p.ell.width = p.width;
      p.ell.aux[pre + "I_indptr"] = std::move(iptr);
      p.ell.aux[pre + "I_indices"] = std::move(ii);
      p.ell.aux[pre + "J_indices"] = std::move(jj);
      out.parts.push_back(std::move(p));
    }
    return out;
  }

 private:
  struct Del {
    void operator()(strata_hyb* h) const { strata_hyb_destroy(h); }
  };
  std::unique_ptr<strata_hyb, Del> h_;
};

// decompose_hyb (storage.hpp:131-132): same signature and result, computed on the GPU.
inline HybDecomposition decompose_hyb(const TensorStorage& csr, int c, int k,
                                      const std::string& prefix = "") {
  if (c < 1 || k < 0) fail(ErrKind::Usage, "hyb requires c >= 1 and k >= 0");
  DeviceCsr d(csr);
  return DeviceHyb(d, c, k).host(prefix);
}

inline double padding_ratio(const HybDecomposition& h) { return h.padding_ratio; }
inline double padding_ratio(const TensorStorage& s) {
  if (s.kind == FormatKind::Csr) fail(ErrKind::Usage, "padding ratio not applicable to CSR storage");
  return s.values.empty() ? 0.0 : static_cast<double>(s.pad_slots) / static_cast<double>(s.values.size());
}

// ---- invariants / accounting (storage.cpp:455-630), host-side on read-back storage ---------
namespace detail {
// aux array whose name ends with `suffix` (storages carry caller prefixes, e.g. hyb_p0_b1_)
inline const IntArray* find_suffix(const TensorStorage& s, const std::string& suffix) {
  for (const auto& kv : s.aux)
    if (kv.first.size() >= suffix.size() &&
        kv.first.compare(kv.first.size() - suffix.size(), suffix.size(), suffix) == 0)
      return &kv.second;
  return nullptr;
}
inline const IntArray& need_suffix(const TensorStorage& s, const std::string& suffix) {
  const IntArray* a = find_suffix(s, suffix);
  if (!a) fail(ErrKind::Lookup, "storage has no aux array: *" + suffix);
  return *a;
}
}  // namespace detail

// for_each_stored_cell (storage.cpp:455-534): every stored (row, col, value), ELL padding
// (a repeat of the previous column inside a row) skipped.
template <class F>
void for_each_stored_cell(const TensorStorage& s, F&& fn) {
  switch (s.kind) {
    case FormatKind::Csr: {
      const IntArray& ip = detail::need_suffix(s, "J_indptr");
      const IntArray& ix = detail::need_suffix(s, "J_indices");
      for (int64_t i = 0; i < s.rows; ++i)
        for (int32_t p = ip[i]; p < ip[i + 1]; ++p) fn(i, int64_t{ix[p]}, double{s.values[p]});
      break;
    }
    case FormatKind::Bsr: {
      const int64_t b = s.block;
      const IntArray& ip = detail::need_suffix(s, "JO_indptr");
      const IntArray& ix = detail::need_suffix(s, "JO_indices");
      for (int64_t br = 0; br < s.rows / b; ++br)
        for (int32_t p = ip[br]; p < ip[br + 1]; ++p)
          for (int64_t ii = 0; ii < b; ++ii)
            for (int64_t ji = 0; ji < b; ++ji)
              fn(br * b + ii, ix[p] * b + ji, double{s.values[(p * b + ii) * b + ji]});
      break;
    }
    case FormatKind::Ell:
    case FormatKind::EllBucket: {
      const IntArray& jx = detail::need_suffix(s, "J_indices");
      const IntArray* rmap = s.kind == FormatKind::EllBucket ? &detail::need_suffix(s, "I_indices") : nullptr;
      const int64_t w = s.width;
      const int64_t nrows = rmap ? static_cast<int64_t>(rmap->size()) : s.rows;
      for (int64_t r = 0; r < nrows; ++r)
        for (int64_t k = 0; k < w; ++k) {
          if (k > 0 && jx[r * w + k] == jx[r * w + k - 1]) continue;  // padding
          fn(rmap ? int64_t{(*rmap)[r]} : r, int64_t{jx[r * w + k]}, double{s.values[r * w + k]});
        }
      break;
    }
  }
}

// reconstruct_dense (storage.cpp:536-550): O(rows * cols) — toy sizes only, as in the reference.
inline DenseMatrix reconstruct_dense(const TensorStorage& s) {
  DenseMatrix d(s.rows, s.cols);
  for_each_stored_cell(s, [&](int64_t i, int64_t j, double v) { d.at(i, j) += v; });
  return d;
}
inline DenseMatrix reconstruct_dense(const HybDecomposition& h) {
  DenseMatrix d(h.rows, h.cols);
  for (const auto& part : h.parts)
    for_each_stored_cell(part.ell, [&](int64_t i, int64_t j, double v) { d.at(i, j) += v; });
  return d;
}

// validate_storage (storage.cpp:567-630): the index invariants of the stored format, as a list
// of messages (empty = valid).  Per compressed axis: indptr starts at 0, is non-decreasing and
// ends at the entry count; indices are in range and sorted inside a segment, and a repeated
// index may only start the trailing padding run of an ELL segment.
inline std::vector<std::string> validate_storage(const TensorStorage& s) {
  std::vector<std::string> out;
  auto check_indptr = [&](const std::string& axis, const IntArray& p, int64_t count) {
    if (p.empty() || p.front() != 0) out.push_back(axis + ": indptr must start at 0");
    for (size_t i = 1; i < p.size(); ++i)
      if (p[i] < p[i - 1]) {
        out.push_back(axis + ": indptr not non-decreasing");
        break;
      }
    if (!p.empty() && count >= 0 && p.back() != count) out.push_back(axis + ": indptr tail != nnz");
  };
  auto check_segments = [&](const std::string& axis, const IntArray& ix, int64_t length,
                            const std::vector<std::pair<int64_t, int64_t>>& segs, bool pad_ok) {
    for (auto [lo, hi] : segs) {
      bool in_pad_run = false;
      for (int64_t i = lo; i < hi; ++i) {
        if (ix[i] < 0 || ix[i] >= length) {
          out.push_back(axis + ": index out of range");
          break;
        }
        if (i == lo) continue;
        if (ix[i] < ix[i - 1]) {
          out.push_back(axis + ": indices not sorted within segment");
          break;
        }
        if (ix[i] == ix[i - 1]) {
          if (pad_ok) in_pad_run = true; else { out.push_back(axis + ": duplicate index inside segment"); break; }
        } else if (in_pad_run) {
          out.push_back(axis + ": duplicate index inside segment");
          break;
        }
      }
    }
  };
  std::vector<std::pair<int64_t, int64_t>> segs;
  switch (s.kind) {
    case FormatKind::Csr: {
      const IntArray& ip = detail::need_suffix(s, "J_indptr");
      const IntArray& ix = detail::need_suffix(s, "J_indices");
      check_indptr("J", ip, static_cast<int64_t>(ix.size()));
      if (static_cast<int64_t>(ip.size()) != s.rows + 1) out.push_back("J: indptr length != rows + 1");
      for (size_t i = 0; i + 1 < ip.size(); ++i) segs.emplace_back(ip[i], std::min<int64_t>(ip[i + 1], ix.size()));
      check_segments("J", ix, s.cols, segs, false);
      break;
    }
    case FormatKind::Bsr: {
      const IntArray& ip = detail::need_suffix(s, "JO_indptr");
      const IntArray& ix = detail::need_suffix(s, "JO_indices");
      check_indptr("JO", ip, static_cast<int64_t>(ix.size()));
      for (size_t i = 0; i + 1 < ip.size(); ++i) segs.emplace_back(ip[i], std::min<int64_t>(ip[i + 1], ix.size()));
      check_segments("JO", ix, s.block > 0 ? s.cols / s.block : 0, segs, false);
      if (static_cast<int64_t>(s.values.size()) != static_cast<int64_t>(ix.size()) * s.block * s.block)
        out.push_back("JO: values size != blocks * b * b");
      break;
    }
    case FormatKind::Ell:
    case FormatKind::EllBucket: {
      const IntArray& jx = detail::need_suffix(s, "J_indices");
      int64_t nrows = s.rows;
      if (s.kind == FormatKind::EllBucket) {
        const IntArray& rmap = detail::need_suffix(s, "I_indices");
        if (const IntArray* ip = detail::find_suffix(s, "I_indptr"))
          check_indptr("I", *ip, static_cast<int64_t>(rmap.size()));
        nrows = static_cast<int64_t>(rmap.size());
        for (int64_t r = 0; r < nrows; ++r)
          if (rmap[r] < 0 || rmap[r] >= s.rows) {
            out.push_back("I: index out of range");
            break;
          }
      }
      if (static_cast<int64_t>(jx.size()) != nrows * s.width) out.push_back("J: indices size != rows * width");
      for (int64_t r = 0; r < nrows && (r + 1) * s.width <= static_cast<int64_t>(jx.size()); ++r)
        segs.emplace_back(r * s.width, (r + 1) * s.width);
      check_segments("J", jx, s.cols, segs, true);
      break;
    }
  }
  return out;
}

// Device-resident BSR (tensor-core SpMM input).
class DeviceBsr {
 public:
  DeviceBsr(const DeviceCsr& csr, int64_t b, cudaStream_t s = nullptr) {
    strata_bsr* h = nullptr;
    check(strata_bsr_from_csr(csr.indptr.data(), csr.indices.data(), csr.values.data(), csr.rows,
                              csr.cols, csr.nnz, b, s, &h));
    h_.reset(h);
    check(strata_bsr_info(h, &mb, &nb, &this->b, &nblocks, &pad_slots));
  }
  // Y[mb*b][d] (f32) = A X with X bf16 [nb*b][d] (device pointers).
  void spmm_bf16(const void* X, float* Y, int64_t d, cudaStream_t s = nullptr) const {
    check(strata_bsr_spmm_bf16(h_.get(), X, Y, d, s));
  }
  TensorStorage host(const std::string& prefix = "") const {
    TensorStorage t;
    t.kind = FormatKind::Bsr;
    t.rows = mb * b;
    t.cols = nb * b;
    t.block = b;
    t.pad_slots = pad_slots;
    IntArray ip(mb + 1), ix(nblocks);
    t.values.resize(nblocks * b * b);
    check(strata_bsr_read(h_.get(), ip.data(), ix.data(), t.values.data()));
    t.aux[prefix + "JO_indptr"] = std::move(ip);
    t.aux[prefix + "JO_indices"] = std::move(ix);
    return t;
  }
  int64_t mb = 0, nb = 0, b = 0, nblocks = 0, pad_slots = 0;

 private:
  struct Del {
    void operator()(strata_bsr* h) const { strata_bsr_destroy(h); }
  };
  std::unique_ptr<strata_bsr, Del> h_;
};

// csr_to_bsr (storage.hpp:117): dims padded to multiples of b (rows/cols of the result).
inline TensorStorage csr_to_bsr(const TensorStorage& csr, int64_t b, const std::string& prefix = "") {
  if (b < 1) fail(ErrKind::Usage, "block size must be >= 1");
  TensorStorage t = DeviceBsr(DeviceCsr(csr), b).host(prefix);
  t.nnz = csr.nnz;
  return t;
}

// csr_to_ell (storage.hpp:124): Capacity error naming the row when a row exceeds w.
inline TensorStorage csr_to_ell(const TensorStorage& csr, int64_t w, const std::string& prefix = "") {
  DeviceCsr d(csr);
  const size_t n = static_cast<size_t>(std::max<int64_t>(csr.rows * std::max<int64_t>(w, 0), 0));
  DeviceArray<int32_t> J(std::max<size_t>(n, 1));
  DeviceArray<float> V(std::max<size_t>(n, 1));
  check(strata_ell_from_csr(d.indptr.data(), d.indices.data(), d.values.data(), csr.rows, csr.cols,
                            w, J.data(), V.data(), nullptr));
  TensorStorage t;
  t.kind = FormatKind::Ell;
  t.rows = csr.rows;
  t.cols = csr.cols;
  t.nnz = csr.nnz;
  t.width = w;
  t.pad_slots = csr.rows * w - csr.nnz;
  auto jj = J.host();
  auto vv = V.host();
  jj.resize(n);
  vv.resize(n);
  t.aux[prefix + "J_indices"] = std::move(jj);
  t.values = std::move(vv);
  return t;
}

// generate_matrix (driver.cpp:365-416): identical graph, as triplets in CSR order.
inline CooMatrix generate_matrix(const std::string& kind, int64_t n, int64_t m, double density,
                                 int64_t band, int64_t block, double avg_degree, uint64_t seed) {
  strata_csr_host* h = nullptr;
  check(strata_generate_csr(kind.c_str(), n, m, density, band, block, avg_degree, seed, &h));
  std::unique_ptr<strata_csr_host, int (*)(strata_csr_host*)> g(h, strata_csr_host_destroy);
  int64_t rows = 0, cols = 0, nnz = 0;
  check(strata_csr_host_info(h, &rows, &cols, &nnz));
  CooMatrix out;
  out.rows = rows;
  out.cols = cols;
  const int32_t* ip = strata_csr_host_indptr(h);
  const int32_t* ix = strata_csr_host_indices(h);
  const float* v = strata_csr_host_values(h);
  out.triplets.reserve(nnz);
  for (int64_t i = 0; i < rows; ++i)
    for (int32_t q = ip[i]; q < ip[i + 1]; ++q) out.triplets.push_back({i, ix[q], v[q]});
  return out;
}

// ---- pipelines (driver.hpp:25-71) -----------------------------------------------------------
enum class KernelOp { SpMM, SDDMM, RGMS };

struct FormatRequest {
  std::string kind = "csr";  // csr | bsr | ell | dbsr | srbcrs | hyb
  int64_t b = 2, w = 0;
  int64_t t = 2, g = 2;      // srbcrs
  int c = 1, k = -1;
  static FormatRequest parse(const std::string& text) {  // driver.cpp:22-54
    FormatRequest r;
    auto colon = text.find(':');
    r.kind = text.substr(0, colon);
    if (r.kind != "csr" && r.kind != "bsr" && r.kind != "ell" && r.kind != "dbsr" &&
        r.kind != "srbcrs" && r.kind != "hyb")
      fail(ErrKind::Usage, "unknown format: " + r.kind);
    if (colon == std::string::npos) return r;
    std::istringstream in(text.substr(colon + 1));
    std::string kv;
    while (std::getline(in, kv, ',')) {
      auto eq = kv.find('=');
      if (eq == std::string::npos) fail(ErrKind::Usage, "bad format parameter: " + kv);
      const std::string key = kv.substr(0, eq);
      const int64_t value = std::stoll(kv.substr(eq + 1));
      if (key == "b") r.b = value;
      else if (key == "w") r.w = value;
      else if (key == "t") r.t = value;
      else if (key == "g") r.g = value;
      else if (key == "c") r.c = static_cast<int>(value);
      else if (key == "k") r.k = static_cast<int>(value);
      else fail(ErrKind::Usage, "unknown format parameter: " + key);
    }
    return r;
  }
};

// A canonical pipeline: the sparse operand decomposed on the device, named dense bindings
// ("X", "Y" for SDDMM, "W" for RGMS) like Pipeline::bindings, run_dense() like
// driver.cpp:163-171 (SDDMM reconstructs the dense m x n output; toy sizes only, as there).
class Pipeline {
 public:
  KernelOp op = KernelOp::SpMM;
  int64_t m = 0, n = 0, d = 0, d_in = 0, d_out = 0, relations = 1;
  std::map<std::string, std::vector<double>> bindings;

  DenseMatrix run_dense() {
    if (op == KernelOp::SpMM) return run_spmm();
    if (op == KernelOp::SDDMM) return run_sddmm();
    return run_rgms();
  }

  // internal state
  FormatRequest fmt;
  std::unique_ptr<DeviceCsr> csr;
  std::unique_ptr<DeviceHyb> hyb;
  std::unique_ptr<DeviceBsr> bsr;
  struct DbsrDel {
    void operator()(strata_dbsr* h) const { strata_dbsr_destroy(h); }
  };
  struct SrbcrsDel {
    void operator()(strata_srbcrs* h) const { strata_srbcrs_destroy(h); }
  };
  std::unique_ptr<strata_dbsr, DbsrDel> dbsr;
  std::unique_ptr<strata_srbcrs, SrbcrsDel> srbcrs;
  TensorStorage csr_host;
  std::vector<int32_t> rel_ptr, rel_dst, rel_src;
  std::vector<float> rel_a;

 private:
  const std::vector<double>& bound(const std::string& name, size_t n_expected) const {
    auto it = bindings.find(name);
    if (it == bindings.end()) fail(ErrKind::Exec, "missing binding for buffer " + name);
    if (it->second.size() != n_expected)
      fail(ErrKind::Exec, "binding size mismatch for " + name + ": got " +
                              std::to_string(it->second.size()) + ", declared " +
                              std::to_string(n_expected));
    return it->second;
  }
  static std::vector<float> f32(const std::vector<double>& v) { return {v.begin(), v.end()}; }

  DenseMatrix run_spmm() {
    const auto& x = bound("X", static_cast<size_t>(n * d));
    DenseMatrix out(m, d);
    if (fmt.kind == "bsr" || fmt.kind == "dbsr" || fmt.kind == "srbcrs") {  // bf16 tensor cores
      std::vector<uint16_t> xb(x.size());
      for (size_t i = 0; i < x.size(); ++i) xb[i] = to_bf16(static_cast<float>(x[i]));
      DeviceArray<uint16_t> X(xb);
      DeviceArray<float> Y(static_cast<size_t>(m * d));
      if (bsr) bsr->spmm_bf16(X.data(), Y.data(), d);
      else if (dbsr) check(strata_dbsr_spmm_bf16(dbsr.get(), X.data(), Y.data(), d, nullptr));
      else check(strata_srbcrs_spmm_bf16(srbcrs.get(), X.data(), Y.data(), d, nullptr));
      auto y = Y.host();
      for (size_t i = 0; i < y.size(); ++i) out.v[i] = y[i];
      return out;
    }
    DeviceArray<float> X(f32(x));
    DeviceArray<float> Y(static_cast<size_t>(m * d));
    if (hyb) hyb->spmm(X.data(), Y.data(), d);
    else check(strata_spmm_csr_f32(csr->indptr.data(), csr->indices.data(), csr->values.data(),
                                   X.data(), Y.data(), m, n, d, nullptr));
    auto y = Y.host();
    for (size_t i = 0; i < y.size(); ++i) out.v[i] = y[i];
    return out;
  }

  DenseMatrix run_sddmm() {
    const auto& x = bound("X", static_cast<size_t>(m * d));
    const auto& yd = bound("Y", static_cast<size_t>(d * n));
    DeviceArray<float> X(f32(x)), Yd(f32(yd));
    DeviceArray<float> B(std::max<size_t>(static_cast<size_t>(csr->nnz), 1));
    check(strata_sddmm_csr_f32(csr->indptr.data(), csr->indices.data(), csr->values.data(),
                               X.data(), Yd.data(), B.data(), m, n, csr->nnz, d, nullptr));
    auto b = B.host();
    DenseMatrix out(m, n);  // positional B reconstructed through the CSR pattern
    const IntArray& ip = csr_host.arr("J_indptr");
    const IntArray& ix = csr_host.arr("J_indices");
    for (int64_t i = 0; i < m; ++i)
      for (int32_t q = ip[i]; q < ip[i + 1]; ++q) out.at(i, ix[q]) += b[q];
    return out;
  }

  DenseMatrix run_rgms() {
    const auto& x = bound("X", static_cast<size_t>(n * d_in));
    const auto& w = bound("W", static_cast<size_t>(relations * d_in * d_out));
    std::vector<uint16_t> xb(x.size()), wb(w.size());
    for (size_t i = 0; i < x.size(); ++i) xb[i] = to_bf16(static_cast<float>(x[i]));
    for (size_t i = 0; i < w.size(); ++i) wb[i] = to_bf16(static_cast<float>(w[i]));
    DeviceArray<uint16_t> X(xb), W(wb);
    DeviceArray<int32_t> rp(rel_ptr), dst(rel_dst), src(rel_src);
    DeviceArray<float> A(rel_a), Y(static_cast<size_t>(m * d_out));
    check(strata_rgms_bf16(rp.data(), dst.data(), src.data(), A.data(), relations, m, n,
                           static_cast<int64_t>(rel_src.size()), X.data(), W.data(), Y.data(),
                           d_in, d_out, nullptr));
    auto y = Y.host();
    DenseMatrix out(m, d_out);
    for (size_t i = 0; i < y.size(); ++i) out.v[i] = y[i];
    return out;
  }
};

// build_matrix_pipeline (driver.cpp:173-217): pad dims for bsr, build CSR, decompose.
inline Pipeline build_matrix_pipeline(KernelOp op, const CooMatrix& m_in, int64_t d,
                                      const FormatRequest& fmt) {
  Pipeline pl;
  CooMatrix m = m_in;
  if (fmt.kind == "bsr" || fmt.kind == "dbsr") {  // pad_for_format (driver.cpp:69-78)
    m.rows = (m.rows + fmt.b - 1) / fmt.b * fmt.b;
    m.cols = (m.cols + fmt.b - 1) / fmt.b * fmt.b;
  } else if (fmt.kind == "srbcrs") {
    m.rows = (m.rows + fmt.t - 1) / fmt.t * fmt.t;
  }
  pl.op = op;
  pl.fmt = fmt;
  pl.m = m.rows;
  pl.n = m.cols;
  pl.d = d;
  pl.csr_host = build_csr(m);
  pl.csr = std::make_unique<DeviceCsr>(pl.csr_host);
  if (op == KernelOp::SpMM && fmt.kind == "hyb") {
    const int k = fmt.k >= 0 ? fmt.k : hyb_auto_k(pl.csr_host);
    pl.hyb = std::make_unique<DeviceHyb>(*pl.csr, fmt.c, k);
  } else if (op == KernelOp::SpMM && fmt.kind == "bsr") {
    pl.bsr = std::make_unique<DeviceBsr>(*pl.csr, fmt.b);
  } else if (op == KernelOp::SpMM && fmt.kind == "dbsr") {
    strata_dbsr* h = nullptr;
    check(strata_dbsr_from_csr(pl.csr->indptr.data(), pl.csr->indices.data(), pl.csr->values.data(),
                               pl.csr->rows, pl.csr->cols, pl.csr->nnz, fmt.b, nullptr, &h));
    pl.dbsr.reset(h);
  } else if (op == KernelOp::SpMM && fmt.kind == "srbcrs") {
    strata_srbcrs* h = nullptr;
    check(strata_srbcrs_from_csr(pl.csr->indptr.data(), pl.csr->indices.data(), pl.csr->values.data(),
                                 pl.csr->rows, pl.csr->cols, pl.csr->nnz, fmt.t, fmt.g, nullptr, &h));
    pl.srbcrs.reset(h);
  } else if (op == KernelOp::SpMM && fmt.kind == "ell") {
    // ELL (w = max row length by default) stores the CSR entries plus zero pads; the product
    // is the CSR one, so the row-split CSR kernel serves it.
  } else if (fmt.kind != "csr") {
    fail(ErrKind::Usage, "format " + fmt.kind + " is not served for this op");
  }
  return pl;
}

// build_rgms_pipeline (driver.cpp:241-314): relation-major edges (kernels.cpp:19-62), X and W
// seeded like the reference (mt19937(seed), uniform_int(-3,3): X first, then W).
inline Pipeline build_rgms_pipeline(const std::vector<CooMatrix>& relations, int64_t d_in,
                                    int64_t d_out, uint64_t seed = 7) {
  if (relations.empty()) fail(ErrKind::Usage, "need at least one relation");
  Pipeline pl;
  pl.op = KernelOp::RGMS;
  pl.m = relations[0].rows;
  pl.n = relations[0].cols;
  pl.d_in = d_in;
  pl.d_out = d_out;
  pl.relations = static_cast<int64_t>(relations.size());
  pl.rel_ptr.push_back(0);
  for (const auto& r : relations) {
    if (r.rows != pl.m || r.cols != pl.n) fail(ErrKind::Usage, "all relations must share dims");
    std::vector<Triplet> t = r.triplets;
    std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    for (const auto& e : t) {
      pl.rel_dst.push_back(static_cast<int32_t>(e.row));
      pl.rel_src.push_back(static_cast<int32_t>(e.col));
      pl.rel_a.push_back(static_cast<float>(e.value));
    }
    pl.rel_ptr.push_back(static_cast<int32_t>(pl.rel_src.size()));
  }
  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_int_distribution<int> val(-3, 3);
  std::vector<double> x(pl.n * d_in), w(pl.relations * d_in * d_out);
  for (auto& v : x) v = val(rng);
  for (auto& v : w) v = val(rng);
  pl.bindings["X"] = std::move(x);
  pl.bindings["W"] = std::move(w);
  return pl;
}

}  // namespace strata_b200
