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
//   FormatRequest::parse / str   driver.hpp:25-35
//   DType / TensorData / Bindings common.hpp:22, storage.hpp:33-43, interp.hpp:25-28
//   KernelSpec / PipelineOptions / Pipeline  kernels.hpp:24-31, driver.hpp:37-60
//   build_matrix_pipeline(op, m, d, dtype, fmt, opts)       driver.hpp:63-64
//   build_rgms_pipeline(rels, d_in, d_out, dtype, fmt, opts, w_override, x_override, seed)
//                                                           driver.hpp:67-71
//   Pipeline::run_dense / verify_pipeline                   driver.hpp:59, :78-81
//   interpret(Program, Bindings, ExecOptions) -> ExecReport interp.hpp:57 (dispatches the
//                                                           pipeline's device plan)
//   SearchSpace / enumerate / run_trials / report_json      tune.hpp (device-timed trials)
//   read_matrix_market(_file) / write_matrix_market(_file)  mmio.hpp:22-26 (device parse)
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
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <optional>
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

enum class FormatKind { Csr, Bsr, Ell, Dbsr, SrBcrs, EllBucket };  // storage.hpp:66

inline const char* format_kind_name(FormatKind k) {  // storage.cpp:16-26
  switch (k) {
    case FormatKind::Csr: return "csr";
    case FormatKind::Bsr: return "bsr";
    case FormatKind::Ell: return "ell";
    case FormatKind::Dbsr: return "dbsr";
    case FormatKind::SrBcrs: return "srbcrs";
    case FormatKind::EllBucket: return "ell_bucket";
  }
  return "?";
}

struct TensorStorage {
  FormatKind kind = FormatKind::Csr;
  std::map<std::string, IntArray> aux;
  std::vector<float> values;
  int64_t rows = 0, cols = 0, nnz = 0, pad_slots = 0, block = 1, width = 0;
  int64_t group = 1;  // SR-BCRS: tiles per group (g); block = tile height (t)
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

// csr_to_coo (storage.cpp:126-136): the CSR's entries as triplets in row-major order.
inline CooMatrix csr_to_coo(const TensorStorage& s) {
  if (s.kind != FormatKind::Csr) fail(ErrKind::Usage, "csr_to_coo needs CSR storage");
  const IntArray* ip = nullptr;
  const IntArray* ix = nullptr;
  for (const auto& kv : s.aux) {  // the CSR's arrays under any prefix
    const std::string& k = kv.first;
    if (k.size() >= 8 && k.compare(k.size() - 8, 8, "J_indptr") == 0) ip = &kv.second;
    if (k.size() >= 9 && k.compare(k.size() - 9, 9, "J_indices") == 0) ix = &kv.second;
  }
  if (!ip || !ix) fail(ErrKind::Lookup, "storage has no aux array: J_indptr / J_indices");
  CooMatrix m;
  m.rows = s.rows;
  m.cols = s.cols;
  for (int64_t i = 0; i < s.rows; ++i)
    for (int32_t p = (*ip)[i]; p < (*ip)[i + 1]; ++p)
      m.triplets.push_back({i, int64_t{(*ix)[p]}, double{s.values[p]}});
  return m;
}

// dense_from_coo (storage.cpp:449-453): duplicates add up.
inline DenseMatrix dense_from_coo(const CooMatrix& m) {
  DenseMatrix d(m.rows, m.cols);
  for (const auto& t : m.triplets) d.at(t.row, t.col) += t.value;
  return d;
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
    case FormatKind::Dbsr: {  // stored block rows only (IO_indices)
      const int64_t b = s.block;
      const IntArray& rmap = detail::need_suffix(s, "IO_indices");
      const IntArray& jp = detail::need_suffix(s, "JO_indptr");
      const IntArray& jx = detail::need_suffix(s, "JO_indices");
      for (size_t r = 0; r < rmap.size(); ++r)
        for (int32_t p = jp[r]; p < jp[r + 1]; ++p)
          for (int64_t ii = 0; ii < b; ++ii)
            for (int64_t ji = 0; ji < b; ++ji)
              fn(rmap[r] * b + ii, jx[p] * b + ji, double{s.values[(p * b + ii) * b + ji]});
      break;
    }
    case FormatKind::SrBcrs: {  // tile rows of t rows, groups of g column tiles, tail padded
      const int64_t t = s.block, g = s.group;
      const IntArray& gp = detail::need_suffix(s, "G_indptr");
      const IntArray& jx = detail::need_suffix(s, "JT_indices");
      for (int64_t r = 0; r < s.rows / t; ++r)
        for (int32_t q = gp[r]; q < gp[r + 1]; ++q)
          for (int64_t sl = 0; sl < g; ++sl) {
            const int64_t tile = q * g + sl;
            if (tile > int64_t{gp[r]} * g && jx[tile] == jx[tile - 1]) continue;  // padding tile
            for (int64_t e = 0; e < t; ++e) fn(r * t + e, int64_t{jx[tile]}, double{s.values[tile * t + e]});
          }
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
    case FormatKind::Dbsr: {
      const int64_t b = s.block > 0 ? s.block : 1;
      const IntArray& rmap = detail::need_suffix(s, "IO_indices");
      if (const IntArray* ip = detail::find_suffix(s, "IO_indptr"))
        check_indptr("IO", *ip, static_cast<int64_t>(rmap.size()));
      check_segments("IO", rmap, s.rows / b, {{0, static_cast<int64_t>(rmap.size())}}, false);
      const IntArray& ip = detail::need_suffix(s, "JO_indptr");
      const IntArray& ix = detail::need_suffix(s, "JO_indices");
      check_indptr("JO", ip, static_cast<int64_t>(ix.size()));
      if (ip.size() != rmap.size() + 1) out.push_back("JO: indptr length != stored rows + 1");
      for (size_t i = 0; i + 1 < ip.size(); ++i) segs.emplace_back(ip[i], std::min<int64_t>(ip[i + 1], ix.size()));
      check_segments("JO", ix, s.cols / b, segs, false);
      if (static_cast<int64_t>(s.values.size()) != static_cast<int64_t>(ix.size()) * b * b)
        out.push_back("JO: values size != blocks * b * b");
      break;
    }
    case FormatKind::SrBcrs: {
      const int64_t t = s.block > 0 ? s.block : 1, g = s.group > 0 ? s.group : 1;
      const IntArray& gp = detail::need_suffix(s, "G_indptr");
      const IntArray& jx = detail::need_suffix(s, "JT_indices");
      check_indptr("G", gp, static_cast<int64_t>(jx.size()) / g);
      if (static_cast<int64_t>(gp.size()) != s.rows / t + 1) out.push_back("G: indptr length != tile rows + 1");
      for (size_t i = 0; i + 1 < gp.size(); ++i)
        segs.emplace_back(int64_t{gp[i]} * g, std::min<int64_t>(int64_t{gp[i + 1]} * g, jx.size()));
      check_segments("JT", jx, s.cols, segs, true);
      if (static_cast<int64_t>(s.values.size()) != static_cast<int64_t>(jx.size()) * t)
        out.push_back("JT: values size != tiles * t");
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

// csr_to_dbsr (storage.cpp:336-370): the BSR plus its stored block rows, on the device.
inline TensorStorage csr_to_dbsr(const TensorStorage& csr, int64_t b, const std::string& prefix = "") {
  if (b < 1) fail(ErrKind::Usage, "block size must be >= 1");
  DeviceCsr d(csr);
  strata_dbsr* h = nullptr;
  check(strata_dbsr_from_csr(d.indptr.data(), d.indices.data(), d.values.data(), csr.rows, csr.cols,
                             csr.nnz, b, nullptr, &h));
  std::unique_ptr<strata_dbsr, int (*)(strata_dbsr*)> hold(h, strata_dbsr_destroy);
  int64_t mb = 0, nb = 0, bb = 0, nstored = 0, nblocks = 0, pad = 0;
  check(strata_dbsr_info(h, &mb, &nb, &bb, &nstored, &nblocks, &pad));
  IntArray io(std::max<int64_t>(nstored, 1)), jp(nstored + 1), jx(std::max<int64_t>(nblocks, 1));
  std::vector<float> v(std::max<int64_t>(nblocks * b * b, 1));
  check(strata_dbsr_read(h, io.data(), jp.data(), jx.data(), v.data()));
  io.resize(nstored);
  jx.resize(nblocks);
  v.resize(nblocks * b * b);
  TensorStorage t;
  t.kind = FormatKind::Dbsr;
  t.rows = mb * b;
  t.cols = nb * b;
  t.nnz = csr.nnz;
  t.block = b;
  t.pad_slots = pad;
  t.aux[prefix + "IO_indptr"] = {0, static_cast<int32_t>(nstored)};
  t.aux[prefix + "IO_indices"] = std::move(io);
  t.aux[prefix + "JO_indptr"] = std::move(jp);
  t.aux[prefix + "JO_indices"] = std::move(jx);
  t.values = std::move(v);
  return t;
}

// csr_to_srbcrs (storage.cpp:372-440): t-row tiles, distinct columns grouped by g (the last
// group padded with its last column), values slot-major [groups * g][t], on the device.
inline TensorStorage csr_to_srbcrs(const TensorStorage& csr, int64_t t, int64_t g,
                                   const std::string& prefix = "") {
  if (t < 1 || g < 1) fail(ErrKind::Usage, "SR-BCRS requires t >= 1 and g >= 1");
  DeviceCsr d(csr);
  strata_srbcrs* h = nullptr;
  check(strata_srbcrs_from_csr(d.indptr.data(), d.indices.data(), d.values.data(), csr.rows,
                               csr.cols, csr.nnz, t, g, nullptr, &h));
  std::unique_ptr<strata_srbcrs, int (*)(strata_srbcrs*)> hold(h, strata_srbcrs_destroy);
  int64_t mb = 0, tt = 0, gg = 0, groups = 0, pad = 0;
  check(strata_srbcrs_info(h, &mb, &tt, &gg, &groups, &pad));
  IntArray gp(mb + 1), jx(std::max<int64_t>(groups * g, 1));
  std::vector<float> v(std::max<int64_t>(groups * g * t, 1));
  check(strata_srbcrs_read(h, gp.data(), jx.data(), v.data()));
  jx.resize(groups * g);
  v.resize(groups * g * t);
  TensorStorage s;
  s.kind = FormatKind::SrBcrs;
  s.rows = mb * t;
  s.cols = csr.cols;
  s.nnz = csr.nnz;
  s.block = t;
  s.group = g;
  s.pad_slots = pad;
  s.aux[prefix + "G_indptr"] = std::move(gp);
  s.aux[prefix + "JT_indices"] = std::move(jx);
  s.values = std::move(v);
  return s;
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

// ---- Matrix Market (mmio.hpp:22-26) ---------------------------------------------------------
// read_matrix_market parses the entry lines on the device (strata_mtx_parse); the triplets come
// back as the reference's value-type CooMatrix.  write_matrix_market is the host writer
// (sorted triplets, precision 17, mmio.cpp:63-72).
class DeviceCoo {  // the parsed triplets resident in HBM (int32 row / col, f64 and f32 values)
 public:
  explicit DeviceCoo(strata_mtx* h) : h_(h) { check(strata_mtx_info(h, &rows, &cols, &ntriplets)); }
  const strata_mtx* get() const { return h_.get(); }
  CooMatrix host() const {
    std::vector<int64_t> r(ntriplets), c(ntriplets);
    std::vector<double> v(ntriplets);
    check(strata_mtx_read(h_.get(), r.data(), c.data(), v.data()));
    CooMatrix m;
    m.rows = rows;
    m.cols = cols;
    m.triplets.resize(ntriplets);
    for (int64_t i = 0; i < ntriplets; ++i) m.triplets[i] = {r[i], c[i], v[i]};
    return m;
  }
  int64_t rows = 0, cols = 0, ntriplets = 0;

 private:
  struct Del {
    void operator()(strata_mtx* h) const { strata_mtx_destroy(h); }
  };
  std::unique_ptr<strata_mtx, Del> h_;
};

inline DeviceCoo read_matrix_market_device(const std::string& text, cudaStream_t s = nullptr) {
  strata_mtx* h = nullptr;
  check(strata_mtx_parse(text.data(), static_cast<int64_t>(text.size()), &h, s));
  return DeviceCoo(h);
}
inline CooMatrix read_matrix_market(std::istream& in) {
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return read_matrix_market_device(text).host();
}
inline CooMatrix read_matrix_market_file(const std::string& path) {
  strata_mtx* h = nullptr;
  check(strata_mtx_read_file(path.c_str(), &h, nullptr));
  return DeviceCoo(h).host();
}
inline void write_matrix_market(std::ostream& out, const CooMatrix& m) {
  out << "%%MatrixMarket matrix coordinate real general\n";
  std::vector<Triplet> t = m.triplets;
  std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  out << m.rows << " " << m.cols << " " << t.size() << "\n";
  out.precision(17);
  for (const auto& e : t) out << e.row + 1 << " " << e.col + 1 << " " << e.value << "\n";
}
inline void write_matrix_market_file(const std::string& path, const CooMatrix& m) {
  std::ofstream f(path);
  if (!f) fail(ErrKind::Usage, "cannot open " + path + " for writing");
  write_matrix_market(f, m);
}

// ---- dtypes, bindings, interpret (common.hpp:22-31, storage.hpp:33-43, interp.hpp:25-63) ----
enum class DType { I32, F32, F64 };
inline const char* dtype_name(DType t) {
  switch (t) {
    case DType::I32: return "i32";
    case DType::F32: return "f32";
    case DType::F64: return "f64";
  }
  return "?";
}

struct TensorData {
  DType dtype = DType::F64;
  std::vector<int32_t> i32;
  std::vector<float> f32;
  std::vector<double> f64;

  static TensorData zeros(DType t, size_t n) {
    TensorData d;
    d.dtype = t;
    if (t == DType::I32) d.i32.assign(n, 0);
    else if (t == DType::F32) d.f32.assign(n, 0.f);
    else d.f64.assign(n, 0.0);
    return d;
  }
  size_t size() const {
    return dtype == DType::I32 ? i32.size() : dtype == DType::F32 ? f32.size() : f64.size();
  }
  double get(size_t i) const {
    return dtype == DType::I32 ? static_cast<double>(i32[i])
                               : dtype == DType::F32 ? static_cast<double>(f32[i]) : f64[i];
  }
  void set(size_t i, double v) {
    if (dtype == DType::I32) i32[i] = static_cast<int32_t>(v);
    else if (dtype == DType::F32) f32[i] = static_cast<float>(v);
    else f64[i] = v;
  }
  // Convenience (not in the reference): a TensorData of dtype t holding v.
  static TensorData of(const std::vector<double>& v, DType t = DType::F64) {
    TensorData d = zeros(t, v.size());
    for (size_t i = 0; i < v.size(); ++i) d.set(i, v[i]);
    return d;
  }
  std::vector<double> values() const {
    std::vector<double> out(size());
    for (size_t i = 0; i < out.size(); ++i) out[i] = get(i);
    return out;
  }
};

struct Bindings {
  std::map<std::string, TensorData> buffers;
  std::map<std::string, int64_t> scalars;
};

enum class ExecMode { Checked, Release };
struct ExecStats {
  int64_t loads = 0, stores = 0, flops = 0;
};
struct ExecReport {
  Bindings outputs;
  ExecStats stats;
  std::vector<std::string> violations;
  double device_ms = 0.0;  // not in the reference: CUDA-event time of the kernels
  bool ok() const { return violations.empty(); }
};
struct ExecOptions {
  ExecMode mode = ExecMode::Release;
  bool skip_copy_blocks = false;
  int threads = 1;
  cudaStream_t stream = nullptr;  // not in the reference: the stream the kernels run on
};

// ---- pipelines (kernels.hpp:22-31, driver.hpp:25-91) ---------------------------------------
enum class KernelOp { SpMM, SDDMM, RGMS };

struct KernelSpec {
  KernelOp op = KernelOp::SpMM;
  int64_t m = 0, n = 0;
  int64_t d = 0;
  int64_t d_in = 0, d_out = 0;
  int64_t relations = 1;
  DType dtype = DType::F32;
};

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
  std::string str() const {  // driver.cpp:56-64
    std::ostringstream os;
    os << kind;
    if (kind == "bsr" || kind == "dbsr") os << ":b=" << b;
    if (kind == "ell" && w > 0) os << ":w=" << w;
    if (kind == "srbcrs") os << ":t=" << t << ",g=" << g;
    if (kind == "hyb") os << ":c=" << c << ",k=" << k;
    return os.str();
  }
};

struct PipelineOptions {
  std::string schedule_script;  // accepted; the device kernels carry their own schedule
  bool preconverted = true;
  ExecMode mode = ExecMode::Release;
  int threads = 1;
};

// FormatRewriteRule (transform.hpp:33-48), as far as callers read it: the rule name, the
// converted buffer's name and the converted storage (kind, dims, nnz, pad_slots and, for
// ELL buckets, the width; its aux arrays are read back from the device by rule_storage()).
struct FormatRewriteRule {
  std::string name, new_buffer;
  TensorStorage storage;
};

// ---- rule generators (transform.hpp:92-103, transform.cpp:432-557) --------------------------
// The converted storage (device conversion, arrays read back under the reference's aux names)
// with the reference's rule / buffer names: rule `name`, buffer "A_" + name, arrays prefixed
// name + "_".  (The IR fields of the reference's rules — axes, index maps — belong to the
// lowering passes, which are out of scope.)
inline FormatRewriteRule identity_rule(const TensorStorage& csr, const std::string& name = "csr") {
  FormatRewriteRule r;
  r.name = name;
  r.new_buffer = "A_" + name;
  r.storage = csr;  // build_csr(csr_to_coo(csr), name + "_"): the same arrays, renamed
  r.storage.aux.clear();
  for (const auto& [key, arr] : csr.aux) {
    for (const char* base : {"J_indptr", "J_indices"}) {
      const std::string b(base);
      if (key.size() >= b.size() && key.compare(key.size() - b.size(), b.size(), b) == 0)
        r.storage.aux[name + "_" + b] = arr;
    }
  }
  return r;
}

inline FormatRewriteRule ell_rule(const TensorStorage& csr, int64_t w, const std::string& name = "ell") {
  FormatRewriteRule r;
  r.name = name;
  r.new_buffer = "A_" + name;
  r.storage = csr_to_ell(csr, w, name + "_");
  return r;
}

inline FormatRewriteRule bsr_rule(const TensorStorage& csr, int64_t b, const std::string& name = "bsr") {
  FormatRewriteRule r;
  r.name = name;
  r.new_buffer = "A_" + name;
  r.storage = csr_to_bsr(csr, b, name + "_");
  return r;
}

// c * (k + 1) rules, one per (partition, bucket) ELL sub-matrix, empty buckets included
// (build_ell_bucket with no segments: I_indptr {0, 0}, empty arrays).
inline std::vector<FormatRewriteRule> hyb_rules(const TensorStorage& csr, int c, int k,
                                                const std::string& name = "hyb") {
  HybDecomposition h = decompose_hyb(csr, c, k, name + "_");
  std::vector<FormatRewriteRule> rules;
  for (int p = 0; p < c; ++p) {
    for (int b = 0; b <= k; ++b) {
      FormatRewriteRule r;
      r.name = name + "_p" + std::to_string(p) + "_b" + std::to_string(b);
      r.new_buffer = "A_" + r.name;
      const EllBucketPart* part = nullptr;
      for (const auto& q : h.parts)
        if (q.partition == p && q.bucket == b) part = &q;
      if (part) {
        r.storage = part->ell;
      } else {
        const std::string pre = name + "_hyb_p" + std::to_string(p) + "_b" + std::to_string(b) + "_";
        r.storage.kind = FormatKind::EllBucket;
        r.storage.rows = csr.rows;
        r.storage.cols = csr.cols;
        r.storage.width = int64_t{1} << b;
        r.storage.aux[pre + "I_indptr"] = {0, 0};
        r.storage.aux[pre + "I_indices"] = {};
        r.storage.aux[pre + "J_indices"] = {};
      }
      rules.push_back(std::move(r));
    }
  }
  return rules;
}

// verify_coverage (transform.hpp:85-90, transform.cpp:396-426): every original non-zero is
// claimed by exactly one rule and the rule storages add up to the original (toy sizes: dense).
inline std::vector<std::string> verify_coverage(const TensorStorage& original,
                                                const std::vector<FormatRewriteRule>& rules) {
  std::vector<std::string> out;
  const DenseMatrix orig = reconstruct_dense(original);
  DenseMatrix sum(orig.rows, orig.cols);
  std::vector<int> claims(static_cast<size_t>(orig.rows * orig.cols), 0);
  for (const auto& rule : rules) {
    for_each_stored_cell(rule.storage, [&](int64_t i, int64_t j, double v) {
      if (i < orig.rows && j < orig.cols) {
        sum.at(i, j) += v;
        claims[i * orig.cols + j] += 1;
      } else if (v != 0.0) {
        out.push_back(rule.name + ": non-zero value in padding region");
      }
    });
  }
  for (int64_t i = 0; i < orig.rows; ++i)
    for (int64_t j = 0; j < orig.cols; ++j) {
      if (sum.at(i, j) != orig.at(i, j)) {
        out.push_back("value mismatch at (" + std::to_string(i) + ", " + std::to_string(j) + ")");
        return out;
      }
      if (orig.at(i, j) != 0.0 && claims[i * orig.cols + j] != 1) {
        out.push_back("non-zero (" + std::to_string(i) + ", " + std::to_string(j) + ") claimed by " +
                      std::to_string(claims[i * orig.cols + j]) + " rules");
        return out;
      }
    }
  return out;
}

// bind_storage (interp.hpp:63, interp.cpp:554-562): aux arrays as I32 buffers under their own
// names, the values under buffer_name.
inline void bind_storage(Bindings& b, const std::string& buffer_name, const TensorStorage& s) {
  for (const auto& [key, arr] : s.aux) {
    TensorData d;
    d.dtype = DType::I32;
    d.i32 = arr;
    b.buffers[key] = std::move(d);
  }
  TensorData v;
  v.dtype = DType::F32;
  v.f32 = s.values;
  b.buffers[buffer_name] = std::move(v);
}

// ---- RelSparse (kernels.hpp:33-43, kernels.cpp:19-83): the RGMS operand -------------------
// Relation-major: I_indptr[R+1] over the rows active in each relation, I_indices those rows,
// J_indptr / J_indices their neighbours (ascending columns), values in the same order.
struct RelSparse {
  int64_t relations = 0, rows = 0, cols = 0, nnz = 0;
  std::map<std::string, IntArray> aux;
  TensorData values;
};

inline RelSparse build_rel_sparse(const std::vector<CooMatrix>& per_relation, DType dtype) {
  if (per_relation.empty()) fail(ErrKind::Usage, "need at least one relation");
  RelSparse r;
  r.relations = static_cast<int64_t>(per_relation.size());
  r.rows = per_relation[0].rows;
  r.cols = per_relation[0].cols;
  IntArray i_indptr = {0}, i_indices, j_indptr = {0}, j_indices;
  std::vector<double> vals;
  for (const auto& m : per_relation) {
    if (m.rows != r.rows || m.cols != r.cols) fail(ErrKind::Usage, "all relations must share dims");
    std::vector<Triplet> t = m.triplets;
    std::sort(t.begin(), t.end(), [](const Triplet& a, const Triplet& b) {
      return a.row != b.row ? a.row < b.row : a.col < b.col;
    });
    for (size_t q = 0; q < t.size();) {
      const int64_t row = t[q].row;
      i_indices.push_back(static_cast<int32_t>(row));
      for (; q < t.size() && t[q].row == row; ++q) {
        j_indices.push_back(static_cast<int32_t>(t[q].col));
        vals.push_back(t[q].value);
      }
      j_indptr.push_back(static_cast<int32_t>(j_indices.size()));
    }
    i_indptr.push_back(static_cast<int32_t>(i_indices.size()));
  }
  r.nnz = static_cast<int64_t>(vals.size());
  r.aux["I_indptr"] = std::move(i_indptr);
  r.aux["I_indices"] = std::move(i_indices);
  r.aux["J_indptr"] = std::move(j_indptr);
  r.aux["J_indices"] = std::move(j_indices);
  r.values = TensorData::of(vals, dtype);
  return r;
}

inline void bind_rel_sparse(Bindings& b, const std::string& buffer_name, const RelSparse& r) {
  for (const auto& [key, arr] : r.aux) {
    TensorData d;
    d.dtype = DType::I32;
    d.i32 = arr;
    b.buffers[key] = std::move(d);
  }
  b.buffers[buffer_name] = r.values;
}

inline DenseMatrix relation_dense(const RelSparse& r, int64_t rel) {
  DenseMatrix d(r.rows, r.cols);
  const IntArray& ip = r.aux.at("I_indptr");
  const IntArray& ii = r.aux.at("I_indices");
  const IntArray& jp = r.aux.at("J_indptr");
  const IntArray& ji = r.aux.at("J_indices");
  for (int32_t q = ip[rel]; q < ip[rel + 1]; ++q)
    for (int32_t e = jp[q]; e < jp[q + 1]; ++e) d.at(ii[q], ji[e]) += r.values.get(e);
  return d;
}

enum class Stage { I, II, III };
inline const char* stage_name(Stage s) { return s == Stage::I ? "I" : s == Stage::II ? "II" : "III"; }

namespace detail {

// The device execution plan a Program stands for: the sparse operand converted once and
// resident in HBM, plus the op's binding contract.  interpret() runs it.
struct DevicePlan {
  KernelOp op = KernelOp::SpMM;
  FormatRequest fmt;
  int64_t m = 0, n = 0, d = 0, d_in = 0, d_out = 0, relations = 1;
  int64_t work_slots = 0;  // stored slots the kernel executes (padding included)
  std::unique_ptr<DeviceCsr> csr;
  std::unique_ptr<DeviceHyb> hyb;
  std::unique_ptr<DeviceBsr> bsr;
  struct DbsrDel {
    void operator()(strata_dbsr* h) const { strata_dbsr_destroy(h); }
  };
  struct SrbcrsDel {
    void operator()(strata_srbcrs* h) const { strata_srbcrs_destroy(h); }
  };
  struct RgmsDel {
    void operator()(strata_rgms* h) const { strata_rgms_destroy(h); }
  };
  std::unique_ptr<strata_dbsr, DbsrDel> dbsr;
  std::unique_ptr<strata_srbcrs, SrbcrsDel> srbcrs;
  std::unique_ptr<strata_rgms, RgmsDel> rgms;
  DeviceArray<int32_t> rel_ptr, rel_dst, rel_src;
  DeviceArray<float> rel_a;

  static const TensorData& bound(const Bindings& b, const std::string& name, size_t n_expected) {
    auto it = b.buffers.find(name);  // interp.cpp:572-582
    if (it == b.buffers.end()) fail(ErrKind::Exec, "missing binding for buffer " + name);
    if (it->second.size() != n_expected)
      fail(ErrKind::Exec, "binding size mismatch for " + name + ": got " +
                              std::to_string(it->second.size()) + ", declared " +
                              std::to_string(n_expected));
    return it->second;
  }
  static std::vector<float> f32(const TensorData& t) {
    std::vector<float> v(t.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = static_cast<float>(t.get(i));
    return v;
  }
  static std::vector<uint16_t> bf16(const TensorData& t) {
    std::vector<uint16_t> v(t.size());
    for (size_t i = 0; i < v.size(); ++i) v[i] = to_bf16(static_cast<float>(t.get(i)));
    return v;
  }

  // Kernels between two events on the caller's stream; returns the output values.
  template <class F>
  static std::vector<float> timed(cudaStream_t s, size_t nout, double& ms, F&& launch) {
    DeviceArray<float> out(std::max<size_t>(nout, 1));
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0));
    cuda_check(cudaEventCreate(&e1));
    cuda_check(cudaEventRecord(e0, s));
    launch(out.data());
    cuda_check(cudaEventRecord(e1, s));
    cuda_check(cudaEventSynchronize(e1));
    float t = 0.f;
    cuda_check(cudaEventElapsedTime(&t, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    ms = t;
    std::vector<float> h = out.host();
    h.resize(nout);
    return h;
  }

  ExecReport run(const Bindings& b, const ExecOptions& o, const std::string& out_name) const {
    ExecReport rep;
    const cudaStream_t s = o.stream;
    std::vector<float> y;
    if (op == KernelOp::SpMM) {
      const TensorData& x = bound(b, "X", static_cast<size_t>(n * d));
      if (fmt.kind == "bsr" || fmt.kind == "dbsr" || fmt.kind == "srbcrs") {  // bf16 tensor cores
        DeviceArray<uint16_t> X(bf16(x));
        y = timed(s, static_cast<size_t>(m * d), rep.device_ms, [&](float* Y) {
          if (bsr) bsr->spmm_bf16(X.data(), Y, d, s);
          else if (dbsr) check(strata_dbsr_spmm_bf16(dbsr.get(), X.data(), Y, d, s));
          else check(strata_srbcrs_spmm_bf16(srbcrs.get(), X.data(), Y, d, s));
        });
      } else {
        DeviceArray<float> X(f32(x));
        y = timed(s, static_cast<size_t>(m * d), rep.device_ms, [&](float* Y) {
          if (hyb) hyb->spmm(X.data(), Y, d, s);
          else check(strata_spmm_csr_f32(csr->indptr.data(), csr->indices.data(), csr->values.data(),
                                         X.data(), Y, m, n, d, s));
        });
      }
      rep.stats.flops = 2 * work_slots * d;
      rep.stats.loads = work_slots * (d + 2);
      rep.stats.stores = m * d;
    } else if (op == KernelOp::SDDMM) {
      const TensorData& x = bound(b, "X", static_cast<size_t>(m * d));
      const TensorData& yd = bound(b, "Y", static_cast<size_t>(d * n));
      DeviceArray<float> X(f32(x)), Yd(f32(yd));
      y = timed(s, static_cast<size_t>(csr->nnz), rep.device_ms, [&](float* B) {
        check(strata_sddmm_csr_f32(csr->indptr.data(), csr->indices.data(), csr->values.data(),
                                   X.data(), Yd.data(), B, m, n, csr->nnz, d, s));
      });
      rep.stats.flops = csr->nnz * (2 * d + 1);
      rep.stats.loads = csr->nnz * (2 * d + 2);
      rep.stats.stores = csr->nnz;
    } else {
      const TensorData& x = bound(b, "X", static_cast<size_t>(n * d_in));
      const TensorData& w = bound(b, "W", static_cast<size_t>(relations * d_in * d_out));
      DeviceArray<uint16_t> X(bf16(x)), W(bf16(w));
      y = timed(s, static_cast<size_t>(m * d_out), rep.device_ms, [&](float* Y) {
        check(strata_rgms_run_bf16(rgms.get(), X.data(), W.data(), Y, d_in, d_out, s));
      });
      rep.stats.flops = 2 * work_slots * d_in * d_out;
      rep.stats.loads = work_slots * (d_in + 2);
      rep.stats.stores = m * d_out;
    }
    TensorData out = TensorData::zeros(DType::F32, y.size());
    out.f32 = std::move(y);
    rep.outputs.buffers[out_name] = std::move(out);
    return rep;
  }
};

inline void require_f32(DType dtype) {
  if (dtype != DType::F32)
    fail(ErrKind::Usage, std::string("dtype ") + dtype_name(dtype) +
                             " is not served by the B200 kernels (f32 storage; the tensor-core "
                             "formats compute in bf16 with f32 accumulation)");
}

// pad_for_format (driver.cpp:69-78)
inline CooMatrix pad_for_format(const CooMatrix& m, const FormatRequest& fmt) {
  CooMatrix out = m;
  if (fmt.kind == "bsr" || fmt.kind == "dbsr") {
    out.rows = (m.rows + fmt.b - 1) / fmt.b * fmt.b;
    out.cols = (m.cols + fmt.b - 1) / fmt.b * fmt.b;
  } else if (fmt.kind == "srbcrs") {
    out.rows = (m.rows + fmt.t - 1) / fmt.t * fmt.t;
  }
  return out;
}

inline int64_t max_row_length(const TensorStorage& csr) {
  const IntArray& ip = csr.arr("J_indptr");
  int64_t w = 0;
  for (size_t i = 0; i + 1 < ip.size(); ++i) w = std::max<int64_t>(w, ip[i + 1] - ip[i]);
  return std::max<int64_t>(w, 1);
}

}  // namespace detail

// A stage-III program.  On this path it stands for the device plan of its pipeline (there is
// no IR to walk: interpret() dispatches to the kernels the plan was built for).
struct Program {
  Stage stage = Stage::III;
  std::shared_ptr<const detail::DevicePlan> plan;
};

// interpret (interp.hpp:57, interp.cpp:564-622): same contract — inputs read from the
// bindings by name with the reference's Exec errors, outputs returned in report.outputs —
// executed by the B200 kernels.
inline ExecReport interpret(const Program& p, const Bindings& b, const ExecOptions& opts = {}) {
  if (p.stage != Stage::III)
    fail(ErrKind::Exec, std::string("interpret expects a stage-III program (got stage ") +
                            stage_name(p.stage) + ")");
  if (!p.plan) fail(ErrKind::Exec, "program has no device plan (not built by a pipeline)");
  const char* out = p.plan->op == KernelOp::SDDMM ? "B" : "Y";
  return p.plan->run(b, opts, out);
}

struct Pipeline {
  KernelSpec spec;
  Program stage1, stage2, stage3;
  Bindings bindings;
  ExecOptions exec_opts;
  std::vector<FormatRewriteRule> rules;
  std::string output_buffer;
  int64_t out_rows = 0, out_cols = 0;
  std::optional<TensorStorage> output_pattern;  // SDDMM: B shares A's structure

  // driver.cpp:146-171: interpret stage3, read the output back as a dense matrix.
  DenseMatrix run_dense() {
    ExecReport report = interpret(stage3, bindings, exec_opts);
    if (!report.ok()) {
      std::string msg = "execution violations:";
      for (const auto& v : report.violations) msg += "\n  " + v;
      fail(ErrKind::Exec, msg);
    }
    auto it = report.outputs.buffers.find(output_buffer);
    if (it == report.outputs.buffers.end())
      fail(ErrKind::Exec, "pipeline output " + output_buffer + " missing from report");
    const TensorData& data = it->second;
    if (output_pattern) {
      TensorStorage view = *output_pattern;
      view.values.resize(data.size());
      for (size_t i = 0; i < data.size(); ++i) view.values[i] = static_cast<float>(data.get(i));
      return reconstruct_dense(view);
    }
    DenseMatrix d(out_rows, out_cols);
    for (int64_t i = 0; i < out_rows * out_cols; ++i) d.v[i] = data.get(i);
    return d;
  }

  // Host copy of rule i's converted storage (aux arrays included), read back from the device.
  TensorStorage rule_storage(size_t i) const {
    const detail::DevicePlan& pl = *stage3.plan;
    const FormatRewriteRule& r = rules.at(i);
    if (pl.hyb) {
      HybDecomposition h = pl.hyb->host();
      for (auto& part : h.parts)
        if (r.name == "hyb_p" + std::to_string(part.partition) + "_b" + std::to_string(part.bucket))
          return part.ell;
      return r.storage;  // an empty bucket: no arrays
    }
    if (pl.bsr) return pl.bsr->host(r.name + "_");
    return r.storage;
  }

  const detail::DevicePlan& plan() const { return *stage3.plan; }
};

namespace detail {
inline void finish_pipeline(Pipeline& pl, std::shared_ptr<DevicePlan> plan, const PipelineOptions& opts) {
  pl.stage3.stage = Stage::III;
  pl.stage3.plan = plan;
  pl.stage1 = Program{Stage::I, plan};
  pl.stage2 = Program{Stage::II, plan};
  pl.exec_opts.mode = opts.mode;
  pl.exec_opts.skip_copy_blocks = opts.preconverted;
  pl.exec_opts.threads = opts.threads;
}
}  // namespace detail

// build_matrix_pipeline (driver.hpp:63-64, driver.cpp:173-217): pad for the format, build the
// CSR, convert on the device, name the rules like rules_for (driver.cpp:80-104).
inline Pipeline build_matrix_pipeline(KernelOp op, const CooMatrix& m_in, int64_t d, DType dtype,
                                      const FormatRequest& fmt, const PipelineOptions& opts) {
  detail::require_f32(dtype);
  if (op == KernelOp::RGMS) fail(ErrKind::Usage, "RGMS pipelines come from build_rgms_pipeline");
  Pipeline pl;
  CooMatrix m = detail::pad_for_format(m_in, fmt);
  TensorStorage csr = build_csr(m);
  pl.spec.op = op;
  pl.spec.m = m.rows;
  pl.spec.n = m.cols;
  pl.spec.d = d;
  pl.spec.dtype = dtype;
  auto plan = std::make_shared<detail::DevicePlan>();
  plan->op = op;
  plan->fmt = fmt;
  plan->m = m.rows;
  plan->n = m.cols;
  plan->d = d;
  plan->csr = std::make_unique<DeviceCsr>(csr);
  plan->work_slots = csr.nnz;
  if (op == KernelOp::SpMM) {
    pl.output_buffer = "Y";
    pl.out_rows = m.rows;
    pl.out_cols = d;
  } else {
    pl.output_buffer = "B";
    pl.out_rows = m.rows;
    pl.out_cols = m.cols;
  }
  auto rule = [&](const std::string& name, FormatKind kind) {
    FormatRewriteRule r;
    r.name = name;
    r.new_buffer = "A_" + name;
    r.storage.kind = kind;
    r.storage.rows = m.rows;
    r.storage.cols = m.cols;
    pl.rules.push_back(r);
    return &pl.rules.back();
  };
  if (fmt.kind == "csr") {
  } else if (fmt.kind == "hyb") {
    const int k = fmt.k >= 0 ? fmt.k : hyb_auto_k(csr);
    if (fmt.c < 1 || k < 0) fail(ErrKind::Usage, "hyb requires c >= 1 and k >= 0");
    plan->hyb = std::make_unique<DeviceHyb>(*plan->csr, fmt.c, k);
    plan->work_slots = 0;
    int np = 0;
    check(strata_hyb_num_parts(plan->hyb->get(), &np));
    std::map<std::pair<int, int>, int> present;
    for (int i = 0; i < np; ++i) {
      int p = 0, bb = 0;
      int64_t w = 0, nr = 0, nz = 0, pad = 0, lo = 0, hi = 0;
      check(strata_hyb_part_info(plan->hyb->get(), i, &p, &bb, &w, &nr, &nz, &pad, &lo, &hi));
      present[{p, bb}] = i;
      plan->work_slots += nr * w;
    }
    // hyb_rules (transform.cpp:525-557): c * (k + 1) rules, empty buckets included.
    for (int p = 0; p < fmt.c; ++p)
      for (int bb = 0; bb <= k; ++bb) {
        FormatRewriteRule* r = rule("hyb_p" + std::to_string(p) + "_b" + std::to_string(bb),
                                    FormatKind::EllBucket);
        r->storage.width = int64_t{1} << bb;
        auto it = present.find({p, bb});
        if (it != present.end()) {
          int pp = 0, b2 = 0;
          int64_t w = 0, nr = 0, nz = 0, pad = 0, lo = 0, hi = 0;
          check(strata_hyb_part_info(plan->hyb->get(), it->second, &pp, &b2, &w, &nr, &nz, &pad, &lo, &hi));
          r->storage.nnz = nz;
          r->storage.pad_slots = pad;
        }
      }
  } else if (fmt.kind == "bsr") {
    if (op != KernelOp::SpMM) fail(ErrKind::Usage, "format bsr is not served for SDDMM");
    plan->bsr = std::make_unique<DeviceBsr>(*plan->csr, fmt.b);
    plan->work_slots = plan->bsr->nblocks * fmt.b * fmt.b;
    FormatRewriteRule* r = rule("bsr", FormatKind::Bsr);
    r->storage.block = fmt.b;
    r->storage.nnz = csr.nnz;
    r->storage.pad_slots = plan->bsr->pad_slots;
  } else if (fmt.kind == "dbsr") {
    if (op != KernelOp::SpMM) fail(ErrKind::Usage, "format dbsr is not served for SDDMM");
    strata_dbsr* h = nullptr;
    check(strata_dbsr_from_csr(plan->csr->indptr.data(), plan->csr->indices.data(),
                               plan->csr->values.data(), plan->csr->rows, plan->csr->cols,
                               plan->csr->nnz, fmt.b, nullptr, &h));
    plan->dbsr.reset(h);
    int64_t mb = 0, nb = 0, b = 0, nstored = 0, nblocks = 0, pad = 0;
    check(strata_dbsr_info(h, &mb, &nb, &b, &nstored, &nblocks, &pad));
    plan->work_slots = nblocks * b * b;
    FormatRewriteRule* r = rule("dbsr", FormatKind::Dbsr);
    r->storage.block = fmt.b;
    r->storage.nnz = csr.nnz;
    r->storage.pad_slots = pad;
  } else if (fmt.kind == "srbcrs") {
    if (op != KernelOp::SpMM) fail(ErrKind::Usage, "format srbcrs is not served for SDDMM");
    strata_srbcrs* h = nullptr;
    check(strata_srbcrs_from_csr(plan->csr->indptr.data(), plan->csr->indices.data(),
                                 plan->csr->values.data(), plan->csr->rows, plan->csr->cols,
                                 plan->csr->nnz, fmt.t, fmt.g, nullptr, &h));
    plan->srbcrs.reset(h);
    int64_t mb = 0, t = 0, g = 0, ngroups = 0, pad = 0;
    check(strata_srbcrs_info(h, &mb, &t, &g, &ngroups, &pad));
    plan->work_slots = ngroups * t * g;
    FormatRewriteRule* r = rule("srbcrs", FormatKind::SrBcrs);
    r->storage.nnz = csr.nnz;
    r->storage.pad_slots = pad;
  } else if (fmt.kind == "ell") {
    // csr_to_ell (w = max row length by default, driver.cpp:86-93): the capacity check runs on
    // the device; the ELL product is the CSR one (pads multiply by 0), so the row-split CSR
    // kernel executes it.
    const int64_t w = fmt.w > 0 ? fmt.w : detail::max_row_length(csr);
    TensorStorage ell = csr_to_ell(csr, w, "ell_");
    FormatRewriteRule* r = rule("ell", FormatKind::Ell);
    r->storage = std::move(ell);
    plan->work_slots = m.rows * w;
  } else {
    fail(ErrKind::Usage, "no rules for format " + fmt.kind);
  }
  if (op == KernelOp::SDDMM) pl.output_pattern = csr;
  detail::finish_pipeline(pl, std::move(plan), opts);
  return pl;
}

// Former four-argument form (F32, default options).
inline Pipeline build_matrix_pipeline(KernelOp op, const CooMatrix& m, int64_t d,
                                      const FormatRequest& fmt) {
  return build_matrix_pipeline(op, m, d, DType::F32, fmt, PipelineOptions{});
}

// build_rgms_pipeline (driver.hpp:67-71, driver.cpp:241-314): relations padded for the format,
// relation-major edges (build_rel_sparse, kernels.cpp:19-62), X then W drawn from
// mt19937(seed) uniform_int(-3, 3) unless overridden (x_override: cols x d_in; w_override:
// one d_in x d_out matrix per relation).  "hyb" decomposes every relation on the device and
// plans from the parts (strata_rgms_plan_hyb); the other formats compute the same product from
// the relation-major CSR edges; both execute the two-pass tcgen05 RGMS.
inline Pipeline build_rgms_pipeline(const std::vector<CooMatrix>& relations, int64_t d_in,
                                    int64_t d_out, DType dtype, const FormatRequest& fmt,
                                    const PipelineOptions& opts,
                                    const std::vector<DenseMatrix>* w_override = nullptr,
                                    const DenseMatrix* x_override = nullptr, uint64_t seed = 7) {
  detail::require_f32(dtype);
  if (relations.empty()) fail(ErrKind::Usage, "need at least one relation");
  Pipeline pl;
  auto plan = std::make_shared<detail::DevicePlan>();
  std::vector<CooMatrix> rels;
  for (const auto& r : relations) rels.push_back(detail::pad_for_format(r, fmt));
  const int64_t R = static_cast<int64_t>(rels.size());
  const int64_t m = rels[0].rows, n = rels[0].cols;
  std::vector<int32_t> rp{0}, dst, src;
  std::vector<float> a;
  for (const auto& r : rels) {
    if (r.rows != m || r.cols != n) fail(ErrKind::Usage, "all relations must share dims");
    TensorStorage s = build_csr(r);  // sorted, validated like the reference's per-slice CSR
    const IntArray& ip = s.arr("J_indptr");
    const IntArray& ix = s.arr("J_indices");
    for (int64_t i = 0; i < m; ++i)
      for (int32_t q = ip[i]; q < ip[i + 1]; ++q) {
        dst.push_back(static_cast<int32_t>(i));
        src.push_back(ix[q]);
        a.push_back(s.values[q]);
      }
    rp.push_back(static_cast<int32_t>(src.size()));
  }
  pl.spec.op = KernelOp::RGMS;
  pl.spec.m = m;
  pl.spec.n = n;
  pl.spec.d_in = d_in;
  pl.spec.d_out = d_out;
  pl.spec.relations = R;
  pl.spec.dtype = dtype;
  pl.output_buffer = "Y";
  pl.out_rows = m;
  pl.out_cols = d_out;

  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_int_distribution<int> val(-3, 3);
  TensorData xd = TensorData::zeros(dtype, static_cast<size_t>(n * d_in));
  if (x_override) {
    if (x_override->rows * x_override->cols != n * d_in)
      fail(ErrKind::Usage, "x_override must be cols x d_in");
    for (size_t i = 0; i < xd.size(); ++i) xd.set(i, x_override->v[i]);
  } else {
    for (size_t i = 0; i < xd.size(); ++i) xd.set(i, val(rng));
  }
  TensorData wd = TensorData::zeros(dtype, static_cast<size_t>(R * d_in * d_out));
  if (w_override && static_cast<int64_t>(w_override->size()) != R)
    fail(ErrKind::Usage, "w_override needs one matrix per relation");
  for (int64_t r = 0; r < R; ++r)
    for (int64_t k = 0; k < d_in; ++k)
      for (int64_t l = 0; l < d_out; ++l)
        wd.set((r * d_in + k) * d_out + l, w_override ? (*w_override)[r].at(k, l) : val(rng));
  pl.bindings.buffers["X"] = std::move(xd);
  pl.bindings.buffers["W"] = std::move(wd);

  if (fmt.kind != "csr") {
    for (int64_t r = 0; r < R; ++r) {
      FormatRewriteRule rule;
      rule.name = "r" + std::to_string(r) + "_" + fmt.kind;
      rule.new_buffer = "A_" + rule.name;
      rule.storage.rows = m;
      rule.storage.cols = n;
      rule.storage.nnz = rp[r + 1] - rp[r];
      rule.storage.kind = fmt.kind == "hyb" ? FormatKind::EllBucket
                          : fmt.kind == "ell" ? FormatKind::Ell : FormatKind::Bsr;
      pl.rules.push_back(rule);
    }
  }
  plan->op = KernelOp::RGMS;
  plan->fmt = fmt;
  plan->m = m;
  plan->n = n;
  plan->d_in = d_in;
  plan->d_out = d_out;
  plan->relations = R;
  plan->work_slots = static_cast<int64_t>(src.size());
  strata_rgms* h = nullptr;
  if (fmt.kind == "hyb") {
    // per-relation hyb rules (driver.cpp:294-300: k = hyb_auto_k of each slice unless given),
    // decomposed on the device and read in place by strata_rgms_plan_hyb
    std::vector<std::unique_ptr<DeviceCsr>> dcsr;
    std::vector<std::unique_ptr<DeviceHyb>> dhyb;
    std::vector<const strata_hyb*> hp;
    for (const auto& r : rels) {
      TensorStorage sl = build_csr(r);
      dcsr.push_back(std::make_unique<DeviceCsr>(sl));
      const int k = fmt.k >= 0 ? fmt.k : hyb_auto_k(sl);
      if (fmt.c < 1 || k < 0) fail(ErrKind::Usage, "hyb requires c >= 1 and k >= 0");
      dhyb.push_back(std::make_unique<DeviceHyb>(*dcsr.back(), fmt.c, k));
      hp.push_back(dhyb.back()->get());
    }
    check(strata_rgms_plan_hyb(hp.data(), R, &h, nullptr));  // synchronous: parts may go
  } else {
    plan->rel_ptr = DeviceArray<int32_t>(rp);
    plan->rel_dst = DeviceArray<int32_t>(dst);
    plan->rel_src = DeviceArray<int32_t>(src);
    plan->rel_a = DeviceArray<float>(a);
    check(strata_rgms_plan(plan->rel_ptr.data(), plan->rel_dst.data(), plan->rel_src.data(),
                           plan->rel_a.data(), R, m, n, static_cast<int64_t>(src.size()), &h, nullptr));
  }
  plan->rgms.reset(h);
  detail::finish_pipeline(pl, std::move(plan), opts);
  return pl;
}

// Former form (F32, csr, default options).
inline Pipeline build_rgms_pipeline(const std::vector<CooMatrix>& relations, int64_t d_in,
                                    int64_t d_out, uint64_t seed = 7) {
  return build_rgms_pipeline(relations, d_in, d_out, DType::F32, FormatRequest{}, PipelineOptions{},
                             nullptr, nullptr, seed);
}

// ---- verification (driver.hpp:73-81, driver.cpp:316-363) -----------------------------------
struct VerifyResult {
  bool pass = true;
  std::string detail;
};

namespace detail {
inline VerifyResult compare(const DenseMatrix& got, const DenseMatrix& want, double rel_tol) {
  VerifyResult out;
  if (got.rows != want.rows || got.cols != want.cols) {
    out.pass = false;
    out.detail = "shape mismatch";
    return out;
  }
  for (int64_t i = 0; i < got.rows; ++i)
    for (int64_t j = 0; j < got.cols; ++j) {
      const double x = got.at(i, j), y = want.at(i, j);
      const double denom = std::max({std::fabs(x), std::fabs(y), 1.0});
      if (std::fabs(x - y) > rel_tol * denom) {
        out.pass = false;
        std::ostringstream os;
        os << "first divergence at (" << i << ", " << j << "): got " << x << ", expected " << y;
        out.detail = os.str();
        return out;
      }
    }
  return out;
}
}  // namespace detail

// Runs the pipeline on the device and compares it with the reference's dense oracle (f64,
// the padded matrix's stored entries): SpMM Y = A X; SDDMM B = A .* (X Y) on the pattern.
inline VerifyResult verify_pipeline(KernelOp op, const CooMatrix& m, int64_t d, DType dtype,
                                    const FormatRequest& fmt, const PipelineOptions& opts,
                                    uint64_t seed) {
  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_int_distribution<int> val(-3, 3);
  Pipeline pl = build_matrix_pipeline(op, m, d, dtype, fmt, opts);
  // The oracle walks the padded matrix's triplets in (row, col) order with their f64 values,
  // i.e. the stored entries of the reference's dense_from_coo(padded).
  CooMatrix padded = detail::pad_for_format(m, fmt);
  std::sort(padded.triplets.begin(), padded.triplets.end(), [](const Triplet& p, const Triplet& q) {
    return p.row != q.row ? p.row < q.row : p.col < q.col;
  });
  const double tol = dtype == DType::I32 ? 0.0 : 1e-5;
  if (op == KernelOp::SpMM) {
    DenseMatrix x(pl.spec.n, d);
    for (auto& v : x.v) v = val(rng);
    pl.bindings.buffers["X"] = TensorData::of(x.v, dtype);
    DenseMatrix got = pl.run_dense();
    DenseMatrix want(padded.rows, d);
    for (const Triplet& e : padded.triplets)
      if (e.value != 0.0)
        for (int64_t k = 0; k < d; ++k) want.at(e.row, k) += e.value * x.at(e.col, k);
    return detail::compare(got, want, tol);
  }
  DenseMatrix x(pl.spec.m, d), y(d, pl.spec.n);
  for (auto& v : x.v) v = val(rng);
  for (auto& v : y.v) v = val(rng);
  pl.bindings.buffers["X"] = TensorData::of(x.v, dtype);
  pl.bindings.buffers["Y"] = TensorData::of(y.v, dtype);
  DenseMatrix got = pl.run_dense();
  DenseMatrix want(padded.rows, padded.cols);
  for (const Triplet& e : padded.triplets) {
    if (e.value == 0.0) continue;
    double acc = 0;
    for (int64_t k = 0; k < d; ++k) acc += x.at(e.row, k) * y.at(k, e.col);
    want.at(e.row, e.col) = e.value * acc;
  }
  return detail::compare(got, want, tol);
}

// ---- tuner (tune.hpp, tune.cpp:19-190) -------------------------------------------------------
struct SearchSpace {
  std::vector<std::string> formats;
  std::vector<std::string> schedules;
  static SearchSpace hyb_c_grid(int k0 = -1, bool scan_k = false, bool include_csr = true) {
    SearchSpace s;
    if (include_csr) s.formats.push_back("csr");
    for (int c : {1, 2, 4, 8, 16}) {
      if (scan_k && k0 >= 0) {
        for (int off : {-1, 0, 1})
          s.formats.push_back("hyb:c=" + std::to_string(c) + ",k=" + std::to_string(std::max(0, k0 + off)));
      } else if (k0 >= 0) {
        s.formats.push_back("hyb:c=" + std::to_string(c) + ",k=" + std::to_string(k0));
      } else {
        s.formats.push_back("hyb:c=" + std::to_string(c));
      }
    }
    s.schedules.push_back("");
    return s;
  }
};

struct SearchPoint {
  int id = 0;
  std::string format, schedule;
};

struct TrialResult {
  SearchPoint point;
  double median_ns = 0.0;
  int64_t flops = 0, loads = 0;
  bool valid = false, correct = false;
  double padding = 0.0, balance = 1.0;
  std::string error;
};

struct TuneReport {
  std::vector<TrialResult> trials;
  int best = -1;
};

inline std::vector<SearchPoint> enumerate(const SearchSpace& space) {
  std::vector<SearchPoint> out;
  const std::vector<std::string> formats =
      space.formats.empty() ? std::vector<std::string>{"csr"} : space.formats;
  const std::vector<std::string> schedules =
      space.schedules.empty() ? std::vector<std::string>{""} : space.schedules;
  int id = 0;
  for (const auto& f : formats)
    for (const auto& s : schedules) out.push_back({id++, f, s});
  return out;
}

// run_trials: the reference's loop (build, verify gate, warmup + repeats of interpret, median)
// with the repeats timed on the device (CUDA events around the kernels; conversion untimed as
// `preconverted` asks) and flush_cache writing a 256 MB device buffer (larger than L2).
inline TuneReport run_trials(KernelOp op, const CooMatrix& m, int64_t d, DType dtype,
                             const SearchSpace& space, int repeats = 100, int warmup = 10,
                             bool flush_cache = false, uint64_t seed = 1) {
  if (repeats < 1) fail(ErrKind::Usage, "repeats must be >= 1");
  TuneReport report;
  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_int_distribution<int> val(-3, 3);
  DenseMatrix x(m.cols, d);
  for (auto& v : x.v) v = val(rng);
  std::unique_ptr<DeviceArray<uint8_t>> junk;
  if (flush_cache) junk = std::make_unique<DeviceArray<uint8_t>>(size_t{256} << 20);
  for (const SearchPoint& pt : enumerate(space)) {
    TrialResult tr;
    tr.point = pt;
    try {
      FormatRequest fmt = FormatRequest::parse(pt.format);
      PipelineOptions opts;
      opts.schedule_script = pt.schedule;
      opts.preconverted = true;
      Pipeline pl = build_matrix_pipeline(op, m, d, dtype, fmt, opts);
      pl.bindings.buffers["X"] = TensorData::of(x.v, dtype);  // as tune.cpp:112-114
      VerifyResult v = verify_pipeline(op, m, d, dtype, fmt, opts, seed + 17);
      tr.correct = v.pass;
      if (!v.pass) tr.error = v.detail;
      int64_t pads = 0, slots = 0;
      for (const auto& r : pl.rules) {  // storage_padding (tune.cpp:86-95)
        pads += r.storage.pad_slots;
        slots += r.storage.nnz + r.storage.pad_slots;
      }
      tr.padding = slots == 0 ? 0.0 : static_cast<double>(pads) / static_cast<double>(slots);
      if (pl.plan().hyb) check(strata_hyb_row_work_balance(pl.plan().hyb->get(), &tr.balance, nullptr));
      std::vector<double> samples;
      for (int rep = 0; rep < warmup + repeats; ++rep) {
        if (junk) cuda_check(cudaMemset(junk->data(), rep & 0xff, junk->size()));
        ExecReport er = interpret(pl.stage3, pl.bindings, pl.exec_opts);
        if (rep == 0) {
          tr.flops = er.stats.flops;
          tr.loads = er.stats.loads;
        }
        if (rep >= warmup) samples.push_back(er.device_ms * 1e6);
      }
      std::sort(samples.begin(), samples.end());
      tr.median_ns = samples[samples.size() / 2];
      tr.valid = true;
    } catch (const Error& e) {
      tr.valid = false;
      tr.error = e.what();
    }
    report.trials.push_back(std::move(tr));
  }
  for (size_t i = 0; i < report.trials.size(); ++i) {
    const TrialResult& tr = report.trials[i];
    if (!tr.valid || !tr.correct) continue;
    if (report.best < 0 || tr.median_ns < report.trials[report.best].median_ns)
      report.best = static_cast<int>(i);
  }
  if (report.best < 0) fail(ErrKind::Usage, "tuner: no valid point in the search space");
  return report;
}

// report_json (tune.cpp:171-197): the same fields, two-space indentation.
inline std::string report_json(const TuneReport& report) {
  auto esc = [](const std::string& s) {
    std::string o;
    for (char ch : s) {
      if (ch == '"' || ch == '\\') { o += '\\'; o += ch; }
      else if (ch == '\n') o += "\\n";
      else o += ch;
    }
    return o;
  };
  auto num = [](double v) {
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
  };
  std::ostringstream j;
  j << "{\n  \"best_point\": " << (report.best >= 0 ? report.trials[report.best].point.id : -1)
    << ",\n  \"trials\": [";
  for (size_t i = 0; i < report.trials.size(); ++i) {
    const TrialResult& t = report.trials[i];
    j << (i ? ",\n" : "\n") << "    {\n";
    j << "      \"best\": " << (static_cast<int>(i) == report.best ? "true" : "false") << ",\n";
    j << "      \"correct\": " << (t.correct ? "true" : "false") << ",\n";
    if (!t.error.empty()) j << "      \"error\": \"" << esc(t.error) << "\",\n";
    j << "      \"flops\": " << t.flops << ",\n";
    j << "      \"loads\": " << t.loads << ",\n";
    j << "      \"median_ns\": " << num(t.median_ns) << ",\n";
    j << "      \"padding_ratio\": " << num(t.padding) << ",\n";
    j << "      \"params\": {\n        \"format\": \"" << esc(t.point.format)
      << "\",\n        \"schedule\": \"" << esc(t.point.schedule) << "\"\n      },\n";
    j << "      \"point\": " << t.point.id << ",\n";
    j << "      \"row_work_balance\": " << num(t.balance) << ",\n";
    j << "      \"valid\": " << (t.valid ? "true" : "false") << "\n    }";
  }
  j << (report.trials.empty() ? "]\n}" : "\n  ]\n}");
  return j.str();
}

}  // namespace strata_b200
