// ref_shim.cpp — extern "C" access to the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// This file is ours; it only calls the reference's public API (proj/include/strata/*.hpp)
// so that pytest (ctypes) can use the reference itself as the parity oracle and as the
// CPU baseline.  Built by oracle/Makefile into oracle/_ref/libstrata_ref.so together with
// the reference's own translation units compiled in place from /root/reference/proj/src.
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// load this library.  The product path never does.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include <sstream>

#include "strata/driver.hpp"
#include "strata/mmio.hpp"
#include "strata/interp.hpp"
#include "strata/kernels.hpp"
#include "strata/storage.hpp"
#include "strata/transform.hpp"

using namespace strata;

namespace {
thread_local std::string g_err;
thread_local int g_kind = 0;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    g_kind = static_cast<int>(e.kind) + 1;  // 0 = OK, else ErrKind ordinal + 1
    return g_kind;
  } catch (const std::exception& e) {
    g_err = e.what();
    g_kind = static_cast<int>(ErrKind::Internal) + 1;
    return g_kind;
  }
}

DType dt(int code) { return code == 0 ? DType::I32 : code == 1 ? DType::F32 : DType::F64; }

struct PipelineH {
  Pipeline pl;
};
}  // namespace

extern "C" {

const char* sref_last_error() { return g_err.c_str(); }

// ---- COO -----------------------------------------------------------------------------
// driver.cpp:365-416 generate_matrix
int sref_generate(const char* kind, int64_t n, int64_t m, double density, int64_t band,
                  int64_t block, double avg_degree, uint64_t seed, void** out) {
  return guard([&] {
    *out = new CooMatrix(generate_matrix(kind, n, m, density, band, block, avg_degree, seed));
  });
}

int sref_coo_from_arrays(int64_t rows, int64_t cols, int64_t nnz, const int64_t* r,
                         const int64_t* c, const double* v, void** out) {
  return guard([&] {
    auto* m = new CooMatrix();
    m->rows = rows;
    m->cols = cols;
    m->triplets.resize(nnz);
    for (int64_t i = 0; i < nnz; ++i) m->triplets[i] = {r[i], c[i], v[i]};
    *out = m;
  });
}

void sref_coo_info(void* h, int64_t* rows, int64_t* cols, int64_t* nnz) {
  auto* m = static_cast<CooMatrix*>(h);
  *rows = m->rows;
  *cols = m->cols;
  *nnz = static_cast<int64_t>(m->triplets.size());
}

void sref_coo_triplets(void* h, int64_t* r, int64_t* c, double* v) {
  auto* m = static_cast<CooMatrix*>(h);
  for (size_t i = 0; i < m->triplets.size(); ++i) {
    r[i] = m->triplets[i].row;
    c[i] = m->triplets[i].col;
    v[i] = m->triplets[i].value;
  }
}

void sref_coo_free(void* h) { delete static_cast<CooMatrix*>(h); }

// mmio.cpp:17-55 read_matrix_market over an in-memory stream, and :63-72 write_matrix_market.
int sref_read_matrix_market(const char* text, int64_t len, void** out) {
  return guard([&] {
    std::istringstream in(std::string(text, static_cast<size_t>(len)));
    *out = new CooMatrix(read_matrix_market(in));
  });
}

// Writes into buf (capacity cap); returns the full text length (call again with a larger buf).
int64_t sref_write_matrix_market(void* coo, char* buf, int64_t cap) {
  std::ostringstream os;
  write_matrix_market(os, *static_cast<CooMatrix*>(coo));
  const std::string s = os.str();
  if (static_cast<int64_t>(s.size()) <= cap) memcpy(buf, s.data(), s.size());
  return static_cast<int64_t>(s.size());
}

// strata_cli.cpp:70-82 split_relations lives in the CLI (not the library, and the CLI needs the
// absent CLI11), so this is a two-line restatement of it: triplet t goes to relation
// mt19937(seed)() % R, in triplet order.
int sref_split_relations(void* coo, int64_t relations, uint64_t seed, void** outs) {
  return guard([&] {
    auto* m = static_cast<CooMatrix*>(coo);
    std::vector<CooMatrix*> rels(relations);
    for (auto& r : rels) {
      r = new CooMatrix();
      r->rows = m->rows;
      r->cols = m->cols;
      r->value_dtype = m->value_dtype;
    }
    std::mt19937 rng(static_cast<uint32_t>(seed));
    for (const auto& t : m->triplets) rels[rng() % relations]->triplets.push_back(t);
    for (int64_t i = 0; i < relations; ++i) outs[i] = rels[i];
  });
}

// tune.cpp:108-111 / driver.cpp:320-321: dense operand, mt19937(seed), uniform_int(-3,3),
// row-major.
void sref_dense_int(int64_t count, uint64_t seed, double* out) {
  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_int_distribution<int> val(-3, 3);
  for (int64_t i = 0; i < count; ++i) out[i] = val(rng);
}

// ---- storages ------------------------------------------------------------------------
int sref_build_csr(void* coo, int dtype, void** out) {
  return guard([&] {
    CooMatrix m = *static_cast<CooMatrix*>(coo);
    m.value_dtype = dt(dtype);
    *out = new TensorStorage(build_csr(m));
  });
}

int sref_csr_to_bsr(void* csr, int64_t b, void** out) {
  return guard([&] { *out = new TensorStorage(csr_to_bsr(*static_cast<TensorStorage*>(csr), b)); });
}

int sref_csr_to_ell(void* csr, int64_t w, void** out) {
  return guard([&] { *out = new TensorStorage(csr_to_ell(*static_cast<TensorStorage*>(csr), w)); });
}

int sref_csr_to_dbsr(void* csr, int64_t b, void** out) {
  return guard([&] { *out = new TensorStorage(csr_to_dbsr(*static_cast<TensorStorage*>(csr), b)); });
}

int sref_csr_to_srbcrs(void* csr, int64_t t, int64_t g, void** out) {
  return guard([&] {
    *out = new TensorStorage(csr_to_srbcrs(*static_cast<TensorStorage*>(csr), t, g));
  });
}

int sref_hyb_auto_k(void* csr) { return hyb_auto_k(*static_cast<TensorStorage*>(csr)); }

// info: rows, cols, nnz, pad_slots, block, nvalues, orig_rows, orig_cols
void sref_storage_info(void* h, int64_t* info) {
  auto* s = static_cast<TensorStorage*>(h);
  info[0] = s->rows;
  info[1] = s->cols;
  info[2] = s->nnz;
  info[3] = s->pad_slots;
  info[4] = s->block;
  info[5] = static_cast<int64_t>(s->values.size());
  info[6] = s->orig_rows;
  info[7] = s->orig_cols;
}

// Returns the aux array length (or -1 if absent); copies up to cap entries.
int64_t sref_storage_aux(void* h, const char* name, int32_t* out, int64_t cap) {
  auto* s = static_cast<TensorStorage*>(h);
  auto it = s->aux.find(name);
  if (it == s->aux.end()) return -1;
  int64_t n = static_cast<int64_t>(it->second.size());
  if (out) std::memcpy(out, it->second.data(), sizeof(int32_t) * std::min(n, cap));
  return n;
}

void sref_storage_values(void* h, double* out) {
  auto* s = static_cast<TensorStorage*>(h);
  for (size_t i = 0; i < s->values.size(); ++i) out[i] = s->values.get(i);
}

int sref_padding_ratio(void* h, double* out) {
  return guard([&] { *out = padding_ratio(*static_cast<TensorStorage*>(h)); });
}

int sref_validate_storage(void* h) {
  return static_cast<int>(validate_storage(*static_cast<TensorStorage*>(h)).size());
}

void sref_storage_free(void* h) { delete static_cast<TensorStorage*>(h); }

// ---- hyb -----------------------------------------------------------------------------
int sref_decompose_hyb(void* csr, int c, int k, const char* prefix, void** out) {
  return guard([&] {
    *out = new HybDecomposition(decompose_hyb(*static_cast<TensorStorage*>(csr), c, k, prefix));
  });
}

int sref_hyb_num_parts(void* h) { return static_cast<int>(static_cast<HybDecomposition*>(h)->parts.size()); }

double sref_hyb_padding(void* h) { return static_cast<HybDecomposition*>(h)->padding_ratio; }

// info: partition, bucket, width, nrows, nnz, pad_slots, col_lo, col_hi
void sref_hyb_part_info(void* h, int i, int64_t* info) {
  const EllBucketPart& p = static_cast<HybDecomposition*>(h)->parts[i];
  const Axis& ia = p.ell.axes.at(p.ell.buffer_axes[1]);
  info[0] = p.partition;
  info[1] = p.bucket;
  info[2] = p.width;
  info[3] = static_cast<int64_t>(p.ell.arr(ia.indices_name).size());
  info[4] = p.ell.nnz;
  info[5] = p.ell.pad_slots;
  info[6] = p.col_lo;
  info[7] = p.col_hi;
}

// Arrays by the reference's binding names (prefix + "hyb_p{p}_b{b}_" + I_indptr/I_indices/J_indices).
void* sref_hyb_part_storage(void* h, int i) {
  return &static_cast<HybDecomposition*>(h)->parts[i].ell;
}

void sref_hyb_free(void* h) { delete static_cast<HybDecomposition*>(h); }

// transform.cpp:525-557 hyb_rules: writes "rule_name new_buffer arr1 arr2 arr3\n" per rule.
int sref_hyb_rules(void* csr, int c, int k, const char* name, char* buf, int64_t cap) {
  return guard([&] {
    auto rules = hyb_rules(*static_cast<TensorStorage*>(csr), c, k, name);
    std::string s;
    for (const auto& r : rules) {
      s += r.name + " " + r.new_buffer;
      for (const auto& [an, arr] : r.storage.aux) s += " " + an + ":" + std::to_string(arr.size());
      s += " " + std::to_string(r.storage.values.size()) + "\n";
    }
    std::strncpy(buf, s.c_str(), cap - 1);
    buf[cap - 1] = 0;
  });
}

// ---- pipelines (driver.cpp:173-217, :241-314) + interpret (interp.cpp:564-622) ---------
// op: 0 SpMM, 1 SDDMM
int sref_pipeline_matrix(int op, void* coo, int64_t d, int dtype, const char* fmt, int threads,
                         void** out) {
  return guard([&] {
    PipelineOptions opts;
    opts.threads = threads;
    auto* h = new PipelineH();
    h->pl = build_matrix_pipeline(op == 0 ? KernelOp::SpMM : KernelOp::SDDMM,
                                  *static_cast<CooMatrix*>(coo), d, dt(dtype),
                                  FormatRequest::parse(fmt), opts);
    *out = h;
  });
}

int sref_pipeline_rgms(void** rels, int64_t R, int64_t d_in, int64_t d_out, int dtype,
                       const char* fmt, uint64_t seed, void** out) {
  return guard([&] {
    std::vector<CooMatrix> rs;
    for (int64_t r = 0; r < R; ++r) rs.push_back(*static_cast<CooMatrix*>(rels[r]));
    PipelineOptions opts;
    auto* h = new PipelineH();
    h->pl = build_rgms_pipeline(rs, d_in, d_out, dt(dtype), FormatRequest::parse(fmt), opts,
                                nullptr, nullptr, seed);
    *out = h;
  });
}

int sref_pipeline_set(void* h, const char* name, const double* data, int64_t n) {
  return guard([&] {
    auto* p = static_cast<PipelineH*>(h);
    TensorData d = TensorData::zeros(p->pl.spec.dtype, n);
    for (int64_t i = 0; i < n; ++i) d.set(i, data[i]);
    p->pl.bindings.buffers[name] = std::move(d);
  });
}

int64_t sref_pipeline_get(void* h, const char* name, double* out, int64_t cap) {
  auto* p = static_cast<PipelineH*>(h);
  auto it = p->pl.bindings.buffers.find(name);
  if (it == p->pl.bindings.buffers.end()) return -1;
  int64_t n = static_cast<int64_t>(it->second.size());
  if (out)
    for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = it->second.get(i);
  return n;
}

// Interpret stage III once; copy the positional output buffer (Y for SpMM/RGMS, B for SDDMM).
int sref_pipeline_run(void* h, double* out, int64_t cap, int64_t* n_out) {
  return guard([&] {
    auto* p = static_cast<PipelineH*>(h);
    ExecReport rep = interpret(p->pl.stage3, p->pl.bindings, p->pl.exec_opts);
    if (!rep.ok()) fail(ErrKind::Exec, "execution violations");
    const TensorData& o = rep.outputs.buffers.at(p->pl.output_buffer);
    int64_t n = static_cast<int64_t>(o.size());
    *n_out = n;
    if (out)
      for (int64_t i = 0; i < std::min(n, cap); ++i) out[i] = o.get(i);
  });
}

void sref_pipeline_free(void* h) { delete static_cast<PipelineH*>(h); }

}  // extern "C"
