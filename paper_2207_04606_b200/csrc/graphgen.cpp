// graphgen.cpp — synthetic inputs for the benchmark configs, emitted directly as CSR.
//
// Restates generate_matrix (driver.cpp:365-416) + build_csr (storage.cpp:89-124) of the
// reference.  The graph must be *identical* to the reference's, and the reference draws from
// libstdc++'s mt19937 / uniform_int_distribution / uniform_real_distribution / std::shuffle,
// so this file makes exactly the same <random> calls in exactly the same order.  What changes
// is the data structure: the reference inserts columns into a std::set per row and then sorts
// 24-byte triplets (74.8 s + 16.8 s at Reddit shape); here a per-row bitmap reproduces the
// same draw sequence (a draw that is already present is discarded exactly as std::set::insert
// discards it) and rows are written straight into their CSR slot (the permutation is known
// before any column is drawn), so the whole thing is one pass with no sort of triplets.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "capi_internal.h"

namespace strata_b200 {

namespace {

int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Triple {
  int64_t row, col;
  float val;
};

// Build CSR from triplets produced in (row, col)-sorted order (random/banded/blocksparse
// already emit row-major order per block row; sort to be safe — those generators are small).
void triplets_to_csr(CsrHost& out, std::vector<Triple>& t) {
  std::stable_sort(t.begin(), t.end(), [](const Triple& a, const Triple& b) {
    return a.row != b.row ? a.row < b.row : a.col < b.col;
  });
  out.indptr.assign(out.rows + 1, 0);
  out.indices.resize(t.size());
  out.values.resize(t.size());
  for (size_t i = 0; i < t.size(); ++i) {
    out.indptr[t[i].row + 1]++;
    out.indices[i] = static_cast<int32_t>(t[i].col);
    out.values[i] = t[i].val;
  }
  for (int64_t r = 0; r < out.rows; ++r) out.indptr[r + 1] += out.indptr[r];
}

}  // namespace

void generate_csr(const std::string& kind, int64_t n, int64_t m, double density, int64_t band,
                  int64_t block, double avg_degree, uint64_t seed, CsrHost& out) {
  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_real_distribution<double> u(0.0, 1.0);
  std::uniform_int_distribution<int> val(1, 9);
  out.rows = n;
  out.cols = m;
  std::vector<Triple> t;
  if (kind == "random") {
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = 0; j < m; ++j)
        if (u(rng) < density) t.push_back({i, j, float(val(rng))});
    triplets_to_csr(out, t);
  } else if (kind == "banded") {
    if (band >= m) throw ApiError(STRATA_ERR_USAGE, "band width must be smaller than the matrix");
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = std::max<int64_t>(0, i - band); j <= std::min<int64_t>(m - 1, i + band); ++j)
        t.push_back({i, j, float(val(rng))});
    triplets_to_csr(out, t);
  } else if (kind == "blocksparse") {
    int64_t nb = ceil_div(n, block), mb = ceil_div(m, block);
    for (int64_t bi = 0; bi < nb; ++bi)
      for (int64_t bj = 0; bj < mb; ++bj) {
        if (u(rng) >= density) continue;
        for (int64_t i = bi * block; i < std::min(n, (bi + 1) * block); ++i)
          for (int64_t j = bj * block; j < std::min(m, (bj + 1) * block); ++j)
            t.push_back({i, j, float(val(rng))});
      }
    triplets_to_csr(out, t);
  } else if (kind == "powerlaw") {
    // Degree sequence: Zipf(0.9) weights summed in index order (driver.cpp:394-399).
    std::vector<double> weight(n);
    double sum = 0;
    for (int64_t i = 0; i < n; ++i) {
      weight[i] = 1.0 / std::pow(double(i + 1), 0.9);
      sum += weight[i];
    }
    std::vector<int64_t> rows(n);
    for (int64_t i = 0; i < n; ++i) rows[i] = i;
    std::shuffle(rows.begin(), rows.end(), rng);  // :402, first RNG consumer
    out.row_order.assign(rows.begin(), rows.end());
    double total_edges = avg_degree * double(n);
    std::vector<int64_t> deg(n);
    for (int64_t i = 0; i < n; ++i)
      deg[i] = std::min<int64_t>(m, std::max<int64_t>(0, llround(total_edges * weight[i] / sum)));
    // CSR row rows[i] holds the columns drawn for index i.
    out.indptr.assign(n + 1, 0);
    for (int64_t i = 0; i < n; ++i) out.indptr[rows[i] + 1] = static_cast<int32_t>(deg[i]);
    int64_t total = 0;
    for (int64_t r = 0; r < n; ++r) {
      total += out.indptr[r + 1];
      if (total > INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "nnz exceeds int32 indptr");
      out.indptr[r + 1] = static_cast<int32_t>(total);
    }
    out.indices.resize(total);
    out.values.resize(total);
    std::vector<uint64_t> bits(ceil_div(std::max<int64_t>(m, 1), 64), 0);
    std::vector<int32_t> drawn;
    for (int64_t i = 0; i < n; ++i) {
      // :407-410 — `while (cols.size() < deg) cols.insert(cd(rng));` then ascending order,
      // one val(rng) per column.
      std::uniform_int_distribution<int64_t> cd(0, m - 1);
      drawn.clear();
      while (static_cast<int64_t>(drawn.size()) < deg[i]) {
        int64_t c = cd(rng);
        uint64_t& w = bits[c >> 6];
        uint64_t bit = uint64_t{1} << (c & 63);
        if (!(w & bit)) {
          w |= bit;
          drawn.push_back(static_cast<int32_t>(c));
        }
      }
      int32_t* dst = out.indices.data() + out.indptr[rows[i]];
      if (deg[i] * 16 > m) {  // dense-ish row: read the bitmap in order, clearing it
        int64_t o = 0;
        for (size_t wi = 0; wi < bits.size(); ++wi) {
          uint64_t w = bits[wi];
          while (w) {
            int b = __builtin_ctzll(w);
            dst[o++] = static_cast<int32_t>(wi * 64 + b);
            w &= w - 1;
          }
          bits[wi] = 0;
        }
      } else {
        std::sort(drawn.begin(), drawn.end());
        for (size_t o = 0; o < drawn.size(); ++o) {
          dst[o] = drawn[o];
          bits[drawn[o] >> 6] = 0;
        }
      }
      float* vdst = out.values.data() + out.indptr[rows[i]];
      for (int64_t o = 0; o < deg[i]; ++o) vdst[o] = float(val(rng));
    }
  } else {
    throw ApiError(STRATA_ERR_USAGE, "unknown generator kind: " + kind);
  }
  out.nnz = static_cast<int64_t>(out.indices.size());
}

void dense_int(int64_t count, uint64_t seed, float* out) {
  std::mt19937 rng(static_cast<uint32_t>(seed));
  std::uniform_int_distribution<int> val(-3, 3);
  for (int64_t i = 0; i < count; ++i) out[i] = static_cast<float>(val(rng));
}

}  // namespace strata_b200
