// test_facade.cpp — the reference's own storage / kernel known-answer and property tests
// (proj/tests/test_storage.cpp, test_kernels.cpp, test_exec.cpp), rewritten against the
// device-backed strata_b200 façade (include/strata_b200.hpp).  Same scenarios, same expected
// values; every computation runs on the GPU through the C ABI.  Run by
// tests/test_gpu_cpp.py (needs a B200).
#include <cmath>
#include <cstdio>
#include <functional>
#include <sstream>
#include <random>
#include <string>
#include <vector>

#include "strata_b200.hpp"

using namespace strata_b200;

// ---- minimal test harness ----------------------------------------------------------------
namespace {
struct Case {
  const char* name;
  std::function<void()> fn;
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, std::function<void()> f) { cases().push_back({n, std::move(f)}); }
};
int g_fail = 0, g_checks = 0;
struct Abort {};
}  // namespace

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name) \
  static void CAT(tc_, __LINE__)(); static Reg CAT(reg_, __LINE__)(name, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()
#define CHECK(...) do { ++g_checks; if (!(__VA_ARGS__)) { ++g_fail; \
  std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); } } while (0)
#define REQUIRE(...) do { ++g_checks; if (!(__VA_ARGS__)) { ++g_fail; \
  std::printf("  FAILED %s:%d: %s\n", __FILE__, __LINE__, #__VA_ARGS__); throw Abort{}; } } while (0)
#define CHECK_THROWS_KIND(expr, k, substr) do { ++g_checks; bool ok_ = false; \
  try { (void)(expr); } catch (const Error& e_) { ok_ = e_.kind == (k) && \
    std::string(e_.what()).find(substr) != std::string::npos; } \
  if (!ok_) { ++g_fail; std::printf("  FAILED %s:%d: throws %s\n", __FILE__, __LINE__, #expr); } } while (0)

namespace {

// test_storage.cpp:18-25
CooMatrix example_m() {
  CooMatrix m;
  m.rows = m.cols = 4;
  m.triplets = {{0, 0, 1}, {0, 2, 2}, {1, 3, 3}, {2, 0, 4}, {2, 1, 5}, {2, 2, 6}, {2, 3, 7}};
  return m;
}

// testutil.cpp:17-33 semantics (values in [-4,4] \ {0}).
CooMatrix random_coo(std::mt19937& rng, int64_t rows, int64_t cols, double density) {
  CooMatrix m;
  m.rows = rows;
  m.cols = cols;
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::uniform_int_distribution<int> val(-4, 4);
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j)
      if (u(rng) < density) {
        int v = val(rng);
        m.triplets.push_back({i, j, double(v ? v : 1)});
      }
  return m;
}

DenseMatrix random_dense(std::mt19937& rng, int64_t r, int64_t c) {
  DenseMatrix d(r, c);
  std::uniform_int_distribution<int> val(-4, 4);
  for (auto& v : d.v) v = val(rng);
  return d;
}

DenseMatrix matmul(const DenseMatrix& a, const DenseMatrix& b) {
  DenseMatrix y(a.rows, b.cols);
  for (int64_t i = 0; i < a.rows; ++i)
    for (int64_t j = 0; j < a.cols; ++j)
      if (a.at(i, j) != 0.0)
        for (int64_t k = 0; k < b.cols; ++k) y.at(i, k) += a.at(i, j) * b.at(j, k);
  return y;
}

// reconstruct_dense of a hyb decomposition (storage.cpp:536-550), via the façade.
DenseMatrix reconstruct(const HybDecomposition& h) { return reconstruct_dense(h); }

DenseMatrix run_spmm(const CooMatrix& m, const DenseMatrix& x, const std::string& fmt) {
  Pipeline pl = build_matrix_pipeline(KernelOp::SpMM, m, x.cols, FormatRequest::parse(fmt));
  pl.bindings.buffers["X"] = TensorData::of(x.v);
  return pl.run_dense();
}

}  // namespace

// ---- storage (test_storage.cpp) -------------------------------------------------------------
TEST_CASE("build_csr matches the hand-derived layout") {  // :30-36
  TensorStorage s = build_csr(example_m());
  CHECK(s.arr("J_indptr") == IntArray{0, 2, 3, 7, 7});
  CHECK(s.arr("J_indices") == IntArray{0, 2, 3, 0, 1, 2, 3});
}

TEST_CASE("build_csr rejects duplicate coordinates") {  // :56-62
  CooMatrix m;
  m.rows = m.cols = 2;
  m.triplets = {{0, 0, 1}, {0, 0, 2}};
  CHECK_THROWS_KIND(build_csr(m), ErrKind::Validation, "duplicate");
}

TEST_CASE("csr_to_bsr tiles the example by hand") {  // :64-77
  TensorStorage bsr = csr_to_bsr(build_csr(example_m()), 2);
  CHECK(bsr.arr("JO_indptr") == IntArray{0, 2, 4});
  CHECK(bsr.arr("JO_indices") == IntArray{0, 1, 0, 1});
  CHECK(bsr.values[0] == 1 && bsr.values[1] == 0 && bsr.values[2] == 0 && bsr.values[3] == 0);
  CHECK(bsr.values[4] == 2 && bsr.values[7] == 3);
}

TEST_CASE("csr_to_bsr of all zeros stores no blocks") {  // :79-84
  CooMatrix m;
  m.rows = m.cols = 4;
  CHECK(csr_to_bsr(build_csr(m), 2).values.empty());
}

TEST_CASE("csr_to_bsr with b=1 mirrors CSR values") {  // :86-93
  TensorStorage csr = build_csr(example_m());
  TensorStorage bsr = csr_to_bsr(csr, 1);
  REQUIRE(bsr.values.size() == csr.values.size());
  CHECK(bsr.values == csr.values);
  CHECK(bsr.arr("JO_indices") == csr.arr("J_indices"));
}

TEST_CASE("csr_to_ell pads and errors per the capacity rule") {  // :95-113
  TensorStorage csr = build_csr(example_m());
  CHECK_THROWS_KIND(csr_to_ell(csr, 2), ErrKind::Capacity, "row 2");
  TensorStorage ell = csr_to_ell(csr, 4);
  const IntArray& ix = ell.arr("J_indices");
  CHECK(ix[0] == 0 && ix[1] == 2 && ix[2] == 2 && ix[3] == 2);
  CHECK(ix[12] == 0 && ix[15] == 0);
  CHECK(ell.values[2] == 0);
  CHECK(std::fabs(padding_ratio(ell) - 9.0 / 16.0) < 1e-12);
}

TEST_CASE("decompose_hyb buckets the example rows") {  // :122-134
  HybDecomposition h = decompose_hyb(build_csr(example_m()), 1, 2);
  REQUIRE(h.parts.size() == 3);
  CHECK(h.parts[0].bucket == 0);
  CHECK(h.parts[0].ell.arr("hyb_p0_b0_I_indices") == IntArray{1});
  CHECK(h.parts[1].ell.arr("hyb_p0_b1_I_indices") == IntArray{0});
  CHECK(h.parts[2].ell.arr("hyb_p0_b2_I_indices") == IntArray{2});
  CHECK(h.padding_ratio == 0.0);
}

TEST_CASE("decompose_hyb splits oversized rows into bucket k segments") {  // :136-146
  HybDecomposition h = decompose_hyb(build_csr(example_m()), 1, 1);
  const EllBucketPart* b1 = nullptr;
  for (const auto& p : h.parts)
    if (p.bucket == 1) b1 = &p;
  REQUIRE(b1 != nullptr);
  CHECK(b1->ell.arr("hyb_p0_b1_I_indices") == IntArray{0, 2, 2});
  CHECK(reconstruct(h).v == dense_from_coo(example_m()).v);
}

TEST_CASE("decompose_hyb of a zero matrix is empty") {  // :148-154
  CooMatrix m;
  m.rows = m.cols = 4;
  HybDecomposition h = decompose_hyb(build_csr(m), 2, 2);
  CHECK(h.parts.empty());
  CHECK(h.padding_ratio == 0.0);
}

TEST_CASE("decompose_hyb rejects c < 1 and k < 0") {  // storage.cpp:273
  CHECK_THROWS_KIND(decompose_hyb(build_csr(example_m()), 0, 1), ErrKind::Usage, "c >= 1");
  CHECK_THROWS_KIND(decompose_hyb(build_csr(example_m()), 1, -1), ErrKind::Usage, "k >= 0");
}

TEST_CASE("round trip: hyb and bsr reconstruct random matrices exactly") {  // :217-246
  std::mt19937 rng(42);
  for (int trial = 0; trial < 40; ++trial) {
    int64_t rows = 1 + static_cast<int64_t>(rng() % 64);
    int64_t cols = 1 + static_cast<int64_t>(rng() % 64);
    CooMatrix m = random_coo(rng, rows, cols, 0.25);
    TensorStorage csr = build_csr(m);
    CHECK(reconstruct(decompose_hyb(csr, 2, 2)).v == dense_from_coo(m).v);
    TensorStorage bsr = csr_to_bsr(csr, 2);
    DenseMatrix got(bsr.rows, bsr.cols);
    const IntArray& ip = bsr.arr("JO_indptr");
    const IntArray& ix = bsr.arr("JO_indices");
    for (int64_t br = 0; br < bsr.rows / 2; ++br)
      for (int32_t p = ip[br]; p < ip[br + 1]; ++p)
        for (int ii = 0; ii < 2; ++ii)
          for (int ji = 0; ji < 2; ++ji) got.at(br * 2 + ii, ix[p] * 2 + ji) += bsr.values[p * 4 + ii * 2 + ji];
    bool ok = true;
    DenseMatrix want = dense_from_coo(m);
    for (int64_t i = 0; i < got.rows; ++i)
      for (int64_t j = 0; j < got.cols; ++j)
        ok &= got.at(i, j) == ((i < rows && j < cols) ? want.at(i, j) : 0.0);
    CHECK(ok);
  }
}

TEST_CASE("indptr arrays are monotone and indices sorted per segment") {  // :319-331
  std::mt19937 rng(3);
  for (int trial = 0; trial < 10; ++trial) {
    CooMatrix m = random_coo(rng, 20, 20, 0.3);
    TensorStorage csr = build_csr(m);
    CHECK(validate_storage(csr).empty());
    CHECK(validate_storage(csr_to_bsr(csr, 2)).empty());
    for (const auto& p : decompose_hyb(csr, 2, 2).parts) CHECK(validate_storage(p.ell).empty());
    CHECK(reconstruct_dense(csr).v == dense_from_coo(m).v);
  }
  // corrupted storages are reported, not thrown
  TensorStorage bad = build_csr(example_m());
  bad.aux["J_indices"][1] = 0;  // row 0 holds columns {0, 2} -> {0, 0}
  auto msgs = validate_storage(bad);
  CHECK(!msgs.empty() && msgs[0] == "J: duplicate index inside segment");
  TensorStorage bad2 = build_csr(example_m());
  bad2.aux["J_indptr"][0] = 1;
  CHECK(!validate_storage(bad2).empty() && validate_storage(bad2)[0] == "J: indptr must start at 0");
}

TEST_CASE("hyb bucket uniformity and entry accounting") {  // :248-263
  std::mt19937 rng(11);
  for (int trial = 0; trial < 20; ++trial) {
    CooMatrix m = random_coo(rng, 32, 32, 0.3);
    HybDecomposition h = decompose_hyb(build_csr(m), 2, 2);
    int64_t entries = 0;
    for (const auto& p : h.parts) {
      CHECK(p.width == (int64_t{1} << p.bucket));
      entries += p.ell.nnz;
    }
    CHECK(entries == static_cast<int64_t>(m.triplets.size()));
  }
}

TEST_CASE("hyb padding ratio is always below one half") {  // :265-287
  std::mt19937 rng(5);
  for (int trial = 0; trial < 100; ++trial) {
    CooMatrix m = random_coo(rng, 24, 24, 0.2 + 0.01 * (trial % 30));
    HybDecomposition h = decompose_hyb(build_csr(m), 1 + trial % 3, trial % 4);
    CHECK(h.padding_ratio < 0.5);
  }
}

// ---- kernels (test_kernels.cpp, test_exec.cpp) -----------------------------------------------
TEST_CASE("SpMM with all-ones dense operand yields replicated row sums") {  // :33-41
  DenseMatrix ones(4, 2);
  for (auto& v : ones.v) v = 1;
  for (const char* fmt : {"csr", "hyb:c=1", "hyb:c=2,k=1"}) {
    DenseMatrix y = run_spmm(example_m(), ones, fmt);
    double sums[4] = {3, 3, 22, 0};
    for (int i = 0; i < 4; ++i)
      for (int k = 0; k < 2; ++k) CHECK(y.at(i, k) == sums[i]);
  }
}

TEST_CASE("SpMM identity operand reproduces the matrix") {  // :43-49
  DenseMatrix eye(4, 4);
  for (int i = 0; i < 4; ++i) eye.at(i, i) = 1;
  CHECK(run_spmm(example_m(), eye, "hyb:c=1,k=1").v == dense_from_coo(example_m()).v);
}

TEST_CASE("SpMM random instances equal the dense oracle in every format") {  // exec :86-102
  std::mt19937 rng(3);
  for (int trial = 0; trial < 20; ++trial) {
    CooMatrix a = random_coo(rng, 1 + rng() % 40, 1 + rng() % 40, 0.3);
    DenseMatrix x = random_dense(rng, a.cols, 8);
    DenseMatrix want = matmul(dense_from_coo(a), x);
    for (const char* fmt : {"csr", "ell", "hyb:c=1", "hyb:c=3,k=1", "hyb:c=1,k=0"})
      CHECK(run_spmm(a, x, fmt).v == want.v);
  }
}

TEST_CASE("tensor-core DBSR and SR-BCRS pipelines equal the dense oracle") {
  std::mt19937 rng(21);
  for (int trial = 0; trial < 4; ++trial) {
    CooMatrix a = random_coo(rng, 70 + rng() % 60, 50 + rng() % 40, 0.15);
    DenseMatrix x0 = random_dense(rng, a.cols, 64);  // integers: exact in bf16
    DenseMatrix want = matmul(dense_from_coo(a), x0);
    // dbsr pads rows and cols to multiples of b; srbcrs pads rows to multiples of t
    DenseMatrix xb(((a.cols + 31) / 32) * 32, 64);
    for (int64_t i = 0; i < x0.rows; ++i)
      for (int64_t j = 0; j < 64; ++j) xb.at(i, j) = x0.at(i, j);
    DenseMatrix gd = run_spmm(a, xb, "dbsr:b=32");
    DenseMatrix gs = run_spmm(a, x0, "srbcrs:t=8,g=32");
    bool ok = gd.rows == ((a.rows + 31) / 32) * 32 && gs.rows == ((a.rows + 7) / 8) * 8;
    for (const DenseMatrix* g : {&gd, &gs})
      for (int64_t i = 0; ok && i < g->rows; ++i)
        for (int64_t j = 0; j < 64; ++j) ok &= g->at(i, j) == (i < want.rows ? want.at(i, j) : 0.0);
    CHECK(ok);
  }
  FormatRequest f = FormatRequest::parse("srbcrs:t=8,g=32");
  CHECK(f.kind == "srbcrs" && f.t == 8 && f.g == 32);
  CHECK_THROWS_KIND(FormatRequest::parse("coo"), ErrKind::Usage, "unknown format: coo");
}

TEST_CASE("BSR tensor-core SpMM equals the dense oracle") {
  std::mt19937 rng(9);
  for (int trial = 0; trial < 5; ++trial) {
    CooMatrix a = random_coo(rng, 96, 64, 0.2);
    DenseMatrix x = random_dense(rng, 64, 64);  // integers: exact in bf16
    DenseMatrix want = matmul(dense_from_coo(a), x);
    DenseMatrix got = run_spmm(a, x, "bsr:b=32");
    CHECK(got.v == want.v);
  }
}

TEST_CASE("GNN layer step A*X*W equals the dense oracle in both associations") {  // §8f item 2
  std::mt19937 rng(23);
  CooMatrix a = generate_matrix("powerlaw", 900, 700, 0, 0, 0, 10.0, 5);
  TensorStorage csr = build_csr(a);
  DeviceCsr dc(csr);
  DeviceHyb h(dc, 1, hyb_auto_k(csr));
  for (auto [din, dout] : {std::pair<int64_t, int64_t>{64, 16}, {16, 64}}) {
    DenseMatrix x = random_dense(rng, a.cols, din), w = random_dense(rng, din, dout);
    DenseMatrix want = matmul(matmul(dense_from_coo(a), x), w);
    std::vector<float> xf(x.v.begin(), x.v.end()), wf(w.v.begin(), w.v.end());
    DeviceArray<float> X(xf), W(wf), Z(static_cast<size_t>(a.rows * dout)),
        work(static_cast<size_t>(h.gnn_layer_work_floats(din, dout)));
    h.gnn_layer(X.data(), W.data(), Z.data(), work.data(), din, dout);
    std::vector<float> z = Z.host();
    CHECK(std::vector<double>(z.begin(), z.end()) == want.v);
  }
}

TEST_CASE("SpMM is bitwise deterministic") {  // exec :135-157
  std::mt19937 rng(17);
  CooMatrix a = generate_matrix("powerlaw", 3000, 3000, 0, 0, 0, 40.0, 3);
  DenseMatrix x(a.cols, 32);
  std::normal_distribution<double> nd;
  for (auto& v : x.v) v = nd(rng);
  CHECK(run_spmm(a, x, "hyb:c=1,k=2").v == run_spmm(a, x, "hyb:c=1,k=2").v);
}

TEST_CASE("SDDMM: all-ones mask with identity factors picks the diagonal pattern") {  // :60-79
  CooMatrix a;
  a.rows = a.cols = 2;
  a.triplets = {{0, 0, 1}, {0, 1, 1}, {1, 0, 1}, {1, 1, 1}};
  Pipeline pl = build_matrix_pipeline(KernelOp::SDDMM, a, 2, FormatRequest{});
  pl.bindings.buffers["X"] = TensorData::of({1, 0, 0, 1});
  pl.bindings.buffers["Y"] = TensorData::of({1, 0, 0, 1});
  DenseMatrix b = pl.run_dense();
  CHECK(b.at(0, 0) == 1 && b.at(0, 1) == 0 && b.at(1, 0) == 0 && b.at(1, 1) == 1);
}

TEST_CASE("SDDMM random instances equal the dense oracle") {  // :81-97
  std::mt19937 rng(8);
  for (int trial = 0; trial < 20; ++trial) {
    CooMatrix a = random_coo(rng, 8, 8, 0.3);
    Pipeline pl = build_matrix_pipeline(KernelOp::SDDMM, a, 4, FormatRequest{});
    DenseMatrix x = random_dense(rng, 8, 4), y = random_dense(rng, 4, 8);
    pl.bindings.buffers["X"] = TensorData::of(x.v);
    pl.bindings.buffers["Y"] = TensorData::of(y.v);
    DenseMatrix got = pl.run_dense();
    DenseMatrix xy = matmul(x, y), ad = dense_from_coo(a), want(8, 8);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j) want.at(i, j) = ad.at(i, j) == 0 ? 0 : ad.at(i, j) * xy.at(i, j);
    REQUIRE(got.v == want.v);
  }
}

TEST_CASE("SDDMM of a zero mask is zero") {  // :99-103
  CooMatrix a;
  a.rows = a.cols = 4;
  Pipeline pl = build_matrix_pipeline(KernelOp::SDDMM, a, 2, FormatRequest{});
  pl.bindings.buffers["X"] = TensorData::of(std::vector<double>(8, 0.0));
  pl.bindings.buffers["Y"] = TensorData::of(std::vector<double>(8, 0.0));
  for (double v : pl.run_dense().v) CHECK(v == 0.0);
}

TEST_CASE("RGMS with one relation degenerates to SpMM of X*W") {  // :105-118
  std::mt19937 rng(12);
  CooMatrix a = random_coo(rng, 40, 40, 0.3);
  Pipeline pl = build_rgms_pipeline({a}, 16, 16);
  DenseMatrix got = pl.run_dense();
  DenseMatrix x(40, 16), w(16, 16);
  x.v = pl.bindings.buffers["X"].values();
  w.v = pl.bindings.buffers["W"].values();
  CHECK(got.v == matmul(dense_from_coo(a), matmul(x, w)).v);
}

TEST_CASE("RGMS random instances match the two-stage oracle") {  // :120-156
  std::mt19937 rng(21);
  std::uniform_real_distribution<double> u(0, 1);
  std::uniform_int_distribution<int> val(-3, 3);
  for (int trial = 0; trial < 25; ++trial) {
    int R = 1 + trial % 3;
    std::vector<CooMatrix> rels(R);
    for (auto& r : rels) {
      r.rows = r.cols = 48;
      for (int i = 0; i < 48; ++i)
        for (int j = 0; j < 48; ++j)
          if (u(rng) < 0.15) {
            int v = val(rng);
            r.triplets.push_back({i, j, double(v ? v : 1)});
          }
    }
    Pipeline pl = build_rgms_pipeline(rels, 16, 32, 100 + trial);
    DenseMatrix got = pl.run_dense();
    DenseMatrix x(48, 16), want(48, 32);
    x.v = pl.bindings.buffers["X"].values();
    for (int r = 0; r < R; ++r) {  // two_stage_rgms_oracle (kernels.cpp:169-193)
      DenseMatrix w(16, 32);
      const std::vector<double> wall = pl.bindings.buffers["W"].values();
      std::copy(wall.begin() + r * 512, wall.begin() + (r + 1) * 512, w.v.begin());
      DenseMatrix part = matmul(dense_from_coo(rels[r]), matmul(x, w));
      for (size_t i = 0; i < want.v.size(); ++i) want.v[i] += part.v[i];
    }
    REQUIRE(got.v == want.v);
  }
}

TEST_CASE("binding size mismatch is an Exec error") {  // interp.cpp:575-578
  Pipeline pl = build_matrix_pipeline(KernelOp::SpMM, example_m(), 2, FormatRequest::parse("hyb"));
  pl.bindings.buffers["X"] = TensorData::of(std::vector<double>(16, 1.0));
  CHECK_THROWS_KIND(pl.run_dense(), ErrKind::Exec, "binding size mismatch for X");
}

// ---- driver.hpp / interp.hpp / tune.hpp / mmio.hpp surface ------------------------------------

TEST_CASE("six-argument pipelines: dtype, options, stage-III interpret, rule names") {  // driver.hpp:63-64
  CooMatrix a = generate_matrix("powerlaw", 500, 400, 0, 0, 0, 12.0, 3);
  PipelineOptions opts;
  opts.schedule_script = "";
  Pipeline pl = build_matrix_pipeline(KernelOp::SpMM, a, 16, DType::F32, FormatRequest::parse("hyb:c=2,k=2"), opts);
  CHECK(pl.spec.m == 500 && pl.spec.n == 400 && pl.spec.d == 16 && pl.spec.dtype == DType::F32);
  CHECK(pl.output_buffer == "Y" && pl.out_rows == 500 && pl.out_cols == 16);
  REQUIRE(pl.rules.size() == 6);  // hyb_rules: c * (k + 1), empty buckets included
  CHECK(pl.rules[0].name == "hyb_p0_b0" && pl.rules[5].name == "hyb_p1_b2");
  CHECK(pl.rules[4].new_buffer == "A_hyb_p1_b1" && pl.rules[4].storage.width == 2);
  HybDecomposition h = decompose_hyb(build_csr(a), 2, 2);
  for (const auto& part : h.parts) {
    const std::string name = "hyb_p" + std::to_string(part.partition) + "_b" + std::to_string(part.bucket);
    for (size_t i = 0; i < pl.rules.size(); ++i)
      if (pl.rules[i].name == name) {
        TensorStorage got = pl.rule_storage(i);
        CHECK(got.aux == part.ell.aux && got.values == part.ell.values);
        CHECK(pl.rules[i].storage.nnz == part.ell.nnz && pl.rules[i].storage.pad_slots == part.ell.pad_slots);
      }
  }
  std::mt19937 rng(4);
  DenseMatrix x = random_dense(rng, 400, 16);
  pl.bindings.buffers["X"] = TensorData::of(x.v, DType::F32);
  ExecReport rep = interpret(pl.stage3, pl.bindings, pl.exec_opts);  // the tune.cpp:137 call
  REQUIRE(rep.ok() && rep.outputs.buffers.count("Y") == 1);
  CHECK(rep.outputs.buffers.at("Y").values() == matmul(dense_from_coo(a), x).v);
  CHECK(rep.stats.flops > 0 && rep.device_ms > 0);
  CHECK(pl.run_dense().v == matmul(dense_from_coo(a), x).v);
  CHECK_THROWS_KIND(interpret(pl.stage1, pl.bindings), ErrKind::Exec,
                    "interpret expects a stage-III program (got stage I)");
  Bindings empty;
  CHECK_THROWS_KIND(interpret(pl.stage3, empty), ErrKind::Exec, "missing binding for buffer X");
  CHECK_THROWS_KIND(build_matrix_pipeline(KernelOp::SpMM, a, 16, DType::F64, FormatRequest{}, opts),
                    ErrKind::Usage, "dtype f64 is not served");
  CHECK_THROWS_KIND(build_matrix_pipeline(KernelOp::SpMM, a, 16, DType::I32, FormatRequest{}, opts),
                    ErrKind::Usage, "dtype i32 is not served");
  CHECK(FormatRequest::parse("hyb:c=2,k=3").str() == "hyb:c=2,k=3");
  CHECK(FormatRequest::parse("bsr:b=4").str() == "bsr:b=4");
  CHECK(FormatRequest::parse("srbcrs:t=8,g=32").str() == "srbcrs:t=8,g=32");
}

TEST_CASE("verify_pipeline passes in every served format") {  // driver.cpp:316-363
  CooMatrix a = generate_matrix("powerlaw", 300, 260, 0, 0, 0, 9.0, 6);
  for (const char* f : {"csr", "hyb:c=1", "hyb:c=3,k=2", "ell", "bsr:b=32", "dbsr:b=32", "srbcrs:t=8,g=32"}) {
    VerifyResult v = verify_pipeline(KernelOp::SpMM, a, 64, DType::F32, FormatRequest::parse(f), PipelineOptions{}, 11);
    CHECK(v.pass);
    if (!v.pass) std::printf("    %s: %s\n", f, v.detail.c_str());
  }
  VerifyResult s = verify_pipeline(KernelOp::SDDMM, a, 16, DType::F32, FormatRequest{}, PipelineOptions{}, 12);
  CHECK(s.pass);
  CHECK_THROWS_KIND(verify_pipeline(KernelOp::SDDMM, a, 16, DType::F32, FormatRequest::parse("bsr:b=2"),
                                    PipelineOptions{}, 12), ErrKind::Usage, "not served for SDDMM");
}

TEST_CASE("build_rgms_pipeline: overrides and the reference's draw order") {  // driver.cpp:241-314
  std::mt19937 rng(31);
  std::vector<CooMatrix> rels(3);
  for (auto& r : rels) r = random_coo(rng, 40, 40, 0.2);
  DenseMatrix x = random_dense(rng, 40, 16);
  std::vector<DenseMatrix> w(3, DenseMatrix(16, 32));
  for (auto& m : w) m = random_dense(rng, 16, 32);
  // both overridden: Y = sum_r A_r X W_r
  Pipeline pl = build_rgms_pipeline(rels, 16, 32, DType::F32, FormatRequest::parse("hyb"),
                                    PipelineOptions{}, &w, &x, 5);
  DenseMatrix want(40, 32);
  for (int r = 0; r < 3; ++r) {
    DenseMatrix part = matmul(dense_from_coo(rels[r]), matmul(x, w[r]));
    for (size_t i = 0; i < want.v.size(); ++i) want.v[i] += part.v[i];
  }
  CHECK(pl.run_dense().v == want.v);
  CHECK(pl.rules.size() == 3 && pl.rules[1].name == "r1_hyb");
  // x overridden only: W takes the first draws of mt19937(seed)
  Pipeline p2 = build_rgms_pipeline(rels, 16, 32, DType::F32, FormatRequest{}, PipelineOptions{},
                                    nullptr, &x, 5);
  std::mt19937 r5(5);
  std::uniform_int_distribution<int> val(-3, 3);
  std::vector<double> wdraw(3 * 16 * 32);
  for (auto& v : wdraw) v = val(r5);
  CHECK(p2.bindings.buffers["W"].values() == wdraw);
  CHECK(p2.bindings.buffers["X"].values() == x.v);
  // neither: X first, then W (driver.cpp:270-288)
  Pipeline p3 = build_rgms_pipeline(rels, 16, 32, DType::F32, FormatRequest{}, PipelineOptions{});
  std::mt19937 r7(7);
  std::vector<double> xd(40 * 16), wd(3 * 16 * 32);
  for (auto& v : xd) v = val(r7);
  for (auto& v : wd) v = val(r7);
  CHECK(p3.bindings.buffers["X"].values() == xd && p3.bindings.buffers["W"].values() == wd);
  CHECK_THROWS_KIND(build_rgms_pipeline(rels, 16, 32, DType::F64, FormatRequest{}, PipelineOptions{}),
                    ErrKind::Usage, "dtype f64");
}

TEST_CASE("run_trials over the hyb c-grid reaches the device and picks a correct point") {  // tune.cpp:100-165
  CooMatrix a = generate_matrix("powerlaw", 2000, 2000, 0, 0, 0, 16.0, 1);
  SearchSpace sp = SearchSpace::hyb_c_grid(-1, false, true);
  CHECK(sp.formats.size() == 6 && sp.formats[0] == "csr" && sp.formats[2] == "hyb:c=2");
  CHECK(enumerate(SearchSpace::hyb_c_grid(3, true, false)).size() == 15);
  TuneReport rep = run_trials(KernelOp::SpMM, a, 32, DType::F32, sp, 5, 2, true, 1);
  REQUIRE(rep.trials.size() == 6);
  for (const auto& t : rep.trials) CHECK(t.valid && t.correct && t.median_ns > 0 && t.flops > 0);
  CHECK(rep.best >= 0 && rep.trials[1].padding > 0 && rep.trials[1].balance >= 1.0);
  const std::string js = report_json(rep);
  CHECK(js.find("\"best_point\": " + std::to_string(rep.trials[rep.best].point.id)) != std::string::npos);
  CHECK(js.find("\"format\": \"hyb:c=16\"") != std::string::npos);
  // SDDMM points fail their binding (the reference's run_trials binds only X) -> no valid point
  CHECK_THROWS_KIND(run_trials(KernelOp::SDDMM, a, 32, DType::F32, sp, 2, 1), ErrKind::Usage,
                    "tuner: no valid point");
}

TEST_CASE("matrix market round trip") {  // test_storage.cpp:333-345
  CooMatrix m = example_m();
  std::ostringstream os;
  write_matrix_market(os, m);
  CHECK(os.str().find("%%MatrixMarket matrix coordinate real general") == 0);
  std::istringstream is(os.str());
  CooMatrix back = read_matrix_market(is);
  CHECK(back.rows == m.rows);
  CHECK(back.cols == m.cols);
  CHECK(dense_from_coo(back).v == dense_from_coo(m).v);
  std::istringstream bad("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1\n3 1 1\n");
  CHECK_THROWS_KIND(read_matrix_market(bad), ErrKind::Usage, "matrix market entry out of range: 3 1 1");
  CHECK_THROWS_KIND(read_matrix_market_file("/nonexistent.mtx"), ErrKind::Usage, "cannot open /nonexistent.mtx");
}

TEST_CASE("sharded SpMM / SDDMM through the C ABI with an NCCL communicator (world 1)") {  // §8b/§8e
  CooMatrix a = generate_matrix("powerlaw", 6000, 5000, 0, 0, 0, 11.0, 8);
  TensorStorage csr = build_csr(a);
  DeviceCsr dc(csr);
  char id[STRATA_NCCL_ID_BYTES];
  check(strata_nccl_unique_id(id));
  void* comm = nullptr;  // an ncclComm_t
  check(strata_nccl_comm_init(id, 1, 0, &comm));
  std::mt19937 rng(3);
  const int64_t d = 32;
  DenseMatrix x = random_dense(rng, a.cols, d);
  std::vector<float> xf(x.v.begin(), x.v.end());
  DeviceArray<float> X(xf), Y(static_cast<size_t>(a.rows * d)), Yref(static_cast<size_t>(a.rows * d));
  DeviceHyb h(dc, 1, hyb_auto_k(csr));
  h.spmm(X.data(), Yref.data(), d);
  for (int chunks : {1, 4}) {
    strata_shard_plan* p = nullptr;
    check(strata_shard_plan_create(dc.indptr.data(), dc.indices.data(), dc.values.data(), dc.rows,
                                   dc.cols, 0, 1, chunks, 1, hyb_auto_k(csr), &p, nullptr));
    check(strata_spmm_hyb_f32_sharded(p, X.data(), Y.data(), d, &comm, 1, nullptr));
    CHECK(Y.host() == Yref.host());
    DenseMatrix xs = random_dense(rng, a.rows, 16), yd = random_dense(rng, 16, a.cols);
    std::vector<float> xsf(xs.v.begin(), xs.v.end()), ydf(yd.v.begin(), yd.v.end());
    DeviceArray<float> Xs(xsf), Yd(ydf), B(static_cast<size_t>(csr.nnz)), Bref(static_cast<size_t>(csr.nnz));
    check(strata_sddmm_csr_f32(dc.indptr.data(), dc.indices.data(), dc.values.data(), Xs.data(),
                               Yd.data(), Bref.data(), a.rows, a.cols, csr.nnz, 16, nullptr));
    check(strata_sddmm_csr_f32_sharded(p, Xs.data(), Yd.data(), B.data(), 16, 1, &comm, 1, nullptr));
    CHECK(B.host() == Bref.host());
    int64_t r0 = -1, r1 = -1;
    check(strata_shard_plan_rows(p, 0, -1, &r0, &r1));
    CHECK(r0 == 0 && r1 == a.rows);
    CHECK(strata_spmm_hyb_f32_sharded(p, X.data(), Y.data(), d, &comm, 2, nullptr) == STRATA_ERR_USAGE);
    check(strata_shard_plan_destroy(p));
  }
  check(strata_nccl_comm_destroy(&comm));
}

// test_storage.cpp:156-237: DBSR / SR-BCRS builders (device conversion, host read-back).
TEST_CASE("csr_to_dbsr keeps only non-empty block rows") {  // :156-165
  CooMatrix m;
  m.rows = m.cols = 6;
  m.triplets = {{0, 0, 1}, {4, 2, 2}};
  TensorStorage dbsr = csr_to_dbsr(build_csr(m), 2);
  CHECK(dbsr.arr("IO_indices") == IntArray{0, 2});
  CHECK(validate_storage(dbsr).empty());
  CHECK(reconstruct_dense(dbsr).v == dense_from_coo(m).v);
}

TEST_CASE("csr_to_dbsr equals bsr reconstruction when no row is empty") {  // :167-172
  std::mt19937 rng(7);
  CooMatrix m = random_coo(rng, 8, 8, 0.6);
  TensorStorage csr = build_csr(m);
  CHECK(reconstruct_dense(csr_to_dbsr(csr, 2)).v == reconstruct_dense(csr_to_bsr(csr, 2)).v);
}

TEST_CASE("csr_to_dbsr of a zero matrix stores nothing") {  // :174-179
  CooMatrix m;
  m.rows = m.cols = 4;
  TensorStorage dbsr = csr_to_dbsr(build_csr(m), 2);
  CHECK(dbsr.arr("IO_indices").empty());
}

TEST_CASE("csr_to_srbcrs of a zero matrix stores nothing") {
  CooMatrix m;
  m.rows = m.cols = 4;
  TensorStorage s = csr_to_srbcrs(build_csr(m), 2, 2);
  CHECK(s.arr("G_indptr") == IntArray({0, 0, 0}));
  CHECK(s.arr("JT_indices").empty() && s.values.empty());
  CHECK(validate_storage(s).empty());
  CHECK(padding_ratio(s) == 0.0);
}

TEST_CASE("csr_to_srbcrs single full column tile") {  // :181-191
  CooMatrix m;
  m.rows = 2;
  m.cols = 3;
  m.triplets = {{0, 1, 1}, {1, 1, 2}};
  TensorStorage s = csr_to_srbcrs(build_csr(m), 2, 1);
  CHECK(s.arr("G_indptr") == IntArray{0, 1});
  CHECK(s.arr("JT_indices") == IntArray{1});
  CHECK(s.values.size() == 2);
  CHECK(padding_ratio(s) == 0.0);
}

TEST_CASE("csr_to_srbcrs groups tiles and pads the tail") {  // :193-204
  CooMatrix m;
  m.rows = 2;
  m.cols = 8;
  m.triplets = {{0, 1, 1}, {0, 4, 2}, {1, 6, 3}};
  TensorStorage s = csr_to_srbcrs(build_csr(m), 2, 2);
  CHECK(s.arr("G_indptr") == IntArray{0, 2});
  CHECK(s.values.size() == 2 * 2 * 2);
  CHECK(s.pad_slots == 8 - 3);
  CHECK(reconstruct_dense(s).v == dense_from_coo(m).v);
  CHECK(validate_storage(s).empty());
}

TEST_CASE("srbcrs reconstruction pads rows to a multiple of t") {  // :206-215
  TensorStorage s = csr_to_srbcrs(build_csr(example_m()), 3, 2);
  DenseMatrix d = reconstruct_dense(s);
  CHECK(d.rows == 6);
  DenseMatrix orig = dense_from_coo(example_m());
  for (int64_t i = 0; i < 4; ++i)
    for (int64_t j = 0; j < 4; ++j) CHECK(d.at(i, j) == orig.at(i, j));
  for (int64_t i = 4; i < 6; ++i)
    for (int64_t j = 0; j < 4; ++j) CHECK(d.at(i, j) == 0.0);
}

TEST_CASE("round trip: DBSR and SR-BCRS reconstruct random matrices exactly") {  // :217-237
  std::mt19937 rng(42);
  for (int trial = 0; trial < 40; ++trial) {
    const int64_t rows = 1 + static_cast<int64_t>(rng() % 64);
    const int64_t cols = 1 + static_cast<int64_t>(rng() % 64);
    CooMatrix m = random_coo(rng, rows, cols, 0.25);
    const DenseMatrix want = dense_from_coo(m);
    TensorStorage csr = build_csr(m);
    auto check_padded = [&](const DenseMatrix& got) {
      for (int64_t i = 0; i < got.rows; ++i)
        for (int64_t j = 0; j < got.cols; ++j) {
          const double expect = (i < rows && j < cols) ? want.at(i, j) : 0.0;
          if (got.at(i, j) != expect) return false;
        }
      return got.rows >= rows && got.cols >= cols;
    };
    const TensorStorage dbsr = csr_to_dbsr(csr, 3), sr = csr_to_srbcrs(csr, 2, 2);
    CHECK(check_padded(reconstruct_dense(dbsr)));
    CHECK(check_padded(reconstruct_dense(sr)));
    CHECK(validate_storage(dbsr).empty());
    CHECK(validate_storage(sr).empty());
  }
}

// storage.cpp:16-26 / :126-136, kernels.cpp:19-83 host helpers.
TEST_CASE("format names, csr_to_coo, RelSparse") {
  CHECK(std::string(format_kind_name(FormatKind::EllBucket)) == "ell_bucket");
  CHECK(std::string(format_kind_name(FormatKind::SrBcrs)) == "srbcrs");
  const CooMatrix m = example_m();
  const CooMatrix back = csr_to_coo(build_csr(m));
  CHECK(dense_from_coo(back).v == dense_from_coo(m).v && back.triplets.size() == m.triplets.size());
  // two relations of the 4 x 4 example: the reference's relation-major layout
  CooMatrix r0, r1;
  r0.rows = r1.rows = r0.cols = r1.cols = 4;
  r0.triplets = {{2, 3, 7}, {0, 2, 2}, {2, 0, 4}};
  r1.triplets = {{1, 3, 3}, {0, 0, 1}};
  const RelSparse rs = build_rel_sparse({r0, r1}, DType::F32);
  CHECK(rs.aux.at("I_indptr") == IntArray({0, 2, 4}));
  CHECK(rs.aux.at("I_indices") == IntArray({0, 2, 0, 1}));
  CHECK(rs.aux.at("J_indptr") == IntArray({0, 1, 3, 4, 5}));
  CHECK(rs.aux.at("J_indices") == IntArray({2, 0, 3, 0, 3}));
  CHECK(rs.values.dtype == DType::F32 && rs.values.f32 == std::vector<float>({2, 4, 7, 1, 3}));
  CHECK(relation_dense(rs, 0).v == dense_from_coo(r0).v);
  CHECK(relation_dense(rs, 1).v == dense_from_coo(r1).v);
  Bindings b;
  bind_rel_sparse(b, "A", rs);
  CHECK(b.buffers.at("A").f32 == rs.values.f32 && b.buffers.at("J_indices").i32 == rs.aux.at("J_indices"));
  CooMatrix bad = r1;
  bad.rows = 5;
  CHECK_THROWS_KIND(build_rel_sparse({r0, bad}, DType::F32), ErrKind::Usage, "share dims");
}

// transform.hpp:92-103 rule generators + bind_storage (interp.cpp:554-562): names, buffer
// names and array sizes equal the reference's (golden.npz "rules/example_c2_k2").
TEST_CASE("rule generators and bind_storage") {
  const TensorStorage csr = build_csr(example_m());
  const std::vector<std::string> want = {
      "hyb_p0_b0|A_hyb_p0_b0|hyb_hyb_p0_b0_I_indices:1,hyb_hyb_p0_b0_I_indptr:2,hyb_hyb_p0_b0_J_indices:1",
      "hyb_p0_b1|A_hyb_p0_b1|hyb_hyb_p0_b1_I_indices:1,hyb_hyb_p0_b1_I_indptr:2,hyb_hyb_p0_b1_J_indices:2",
      "hyb_p0_b2|A_hyb_p0_b2|hyb_hyb_p0_b2_I_indices:0,hyb_hyb_p0_b2_I_indptr:2,hyb_hyb_p0_b2_J_indices:0",
      "hyb_p1_b0|A_hyb_p1_b0|hyb_hyb_p1_b0_I_indices:2,hyb_hyb_p1_b0_I_indptr:2,hyb_hyb_p1_b0_J_indices:2",
      "hyb_p1_b1|A_hyb_p1_b1|hyb_hyb_p1_b1_I_indices:1,hyb_hyb_p1_b1_I_indptr:2,hyb_hyb_p1_b1_J_indices:2",
      "hyb_p1_b2|A_hyb_p1_b2|hyb_hyb_p1_b2_I_indices:0,hyb_hyb_p1_b2_I_indptr:2,hyb_hyb_p1_b2_J_indices:0"};
  const auto rules = hyb_rules(csr, 2, 2, "hyb");
  REQUIRE(rules.size() == want.size());
  for (size_t i = 0; i < rules.size(); ++i) {
    std::string got = rules[i].name + "|" + rules[i].new_buffer + "|";
    bool first = true;
    for (const auto& [key, arr] : rules[i].storage.aux) {  // std::map: sorted like the golden
      got += (first ? "" : ",") + key + ":" + std::to_string(arr.size());
      first = false;
    }
    CHECK(got == want[i]);
  }
  const FormatRewriteRule b = bsr_rule(csr, 2);
  CHECK(b.name == "bsr" && b.new_buffer == "A_bsr" && b.storage.kind == FormatKind::Bsr);
  CHECK(b.storage.aux.count("bsr_JO_indptr") == 1 && b.storage.aux.count("bsr_JO_indices") == 1);
  CHECK(b.storage.arr("bsr_JO_indptr") == csr_to_bsr(csr, 2, "x_").arr("x_JO_indptr"));
  const FormatRewriteRule e = ell_rule(csr, 4);
  CHECK(e.new_buffer == "A_ell" && e.storage.aux.count("ell_J_indices") == 1);
  CHECK(e.storage.values.size() == 16);
  const FormatRewriteRule id = identity_rule(csr);
  CHECK(id.new_buffer == "A_csr" && id.storage.arr("csr_J_indptr") == csr.arr("J_indptr"));
  CHECK(id.storage.arr("csr_J_indices") == csr.arr("J_indices") && id.storage.values == csr.values);
  // verify_coverage (transform.cpp:396-426): hyb / bsr / ell / identity rules each cover
  // the matrix exactly; two copies of a rule claim every non-zero twice
  CHECK(verify_coverage(csr, rules).empty());
  CHECK(verify_coverage(csr, {b}).empty());
  CHECK(verify_coverage(csr, {e}).empty());
  CHECK(verify_coverage(csr, {id}).empty());
  const auto twice = verify_coverage(csr, {id, id});
  CHECK(twice.size() == 1 && twice[0].find("value mismatch") == 0);
  Bindings bb;
  bind_storage(bb, "A_bsr", b.storage);
  CHECK(bb.buffers.at("A_bsr").dtype == DType::F32 && bb.buffers.at("A_bsr").f32 == b.storage.values);
  CHECK(bb.buffers.at("bsr_JO_indices").dtype == DType::I32 &&
        bb.buffers.at("bsr_JO_indices").i32 == b.storage.arr("bsr_JO_indices"));
}

int main() {
  int failed_cases = 0;
  for (auto& c : cases()) {
    const int before = g_fail;
    try {
      c.fn();
    } catch (const Abort&) {
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  EXCEPTION in '%s': %s\n", c.name, e.what());
    }
    if (g_fail != before) {
      ++failed_cases;
      std::printf("[FAIL] %s\n", c.name);
    }
  }
  std::printf("cases: %zu  failed: %d  checks: %d\n", cases().size(), failed_cases, g_checks);
  return failed_cases ? 1 : 0;
}
