// hyb_build.cu — device construction of the hyb(c, k) decomposition.
//
// Restates decompose_hyb (storage.cpp:271-334) + build_ell_bucket (storage.cpp:229-269) as a
// stable multi-bin partition of rows, i.e. one pass of an LSD radix sort keyed by
// bin = (partition p, bucket b):
//   1. hyb_count_kernel   per 256-row tile: segments and entries per bin (smem histogram)
//   2. cub::DeviceScan     exclusive scan in (bin-major, tile) order -> global positions.
//                          Bin-major order IS the reference's part order (partition-major,
//                          bucket ascending, empty bins occupying nothing), tile order and
//                          the in-tile rank are row order, so positions are bit-exact.
//   3. hyb_scatter_kernel  per tile, per bin: CTA-wide exclusive scan of segment counts ->
//                          I_indices[pos] = row plus a (source offset, length) descriptor per
//                          segment; split rows (l > 2^k) emit ceil(l / 2^k) consecutive
//                          segments (storage.cpp:301-309), cooperatively for long rows.
//   4. hyb_fill_kernel     one thread per ELL slot: real slot -> (col, val); pad slot ->
//                          (last real column of that segment, 0) (storage.cpp:253-261).
// Then the SpMM schedule: rows-per-chunk per part and, for the bucket-k part (the only one
// whose I_indices may repeat), the list of split runs that cross chunk boundaries.
// The only host synchronisation is the D2H of the per-bin totals needed to size allocations.
#include <cub/cub.cuh>

#include <algorithm>

#include "capi_internal.h"
#include "common.cuh"

namespace strata_b200 {

namespace {

constexpr int kTile = 256;
constexpr int kSlotsPerChunk = 256;  // SpMM work unit: ~256 ELL slots per virtual warp

__device__ __forceinline__ int ceil_log2_dev(int64_t x) {
  return x <= 1 ? 0 : 64 - __clzll(static_cast<unsigned long long>(x - 1));
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* __restrict__ a, int64_t lo,
                                                   int64_t hi, int64_t v) {
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

struct RowPart {
  int64_t q0, l;
};

// Entries of row i inside partition p (storage.cpp:284-297; the row is sorted so they are
// one contiguous run of the CSR row).
__device__ __forceinline__ RowPart row_part(const int32_t* __restrict__ indptr,
                                            const int32_t* __restrict__ indices, int64_t i,
                                            int p, int c, int64_t part_w, int64_t cols) {
  int64_t a = indptr[i], b = indptr[i + 1];
  if (c == 1) return {a, b - a};
  int64_t lo = static_cast<int64_t>(p) * part_w;
  int64_t hi = min64(cols, lo + part_w);
  int64_t q0 = lower_bound_i32(indices, a, b, lo);
  int64_t q1 = lower_bound_i32(indices, q0, b, hi);
  return {q0, q1 - q0};
}

__global__ void __launch_bounds__(kTile)
hyb_count_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                 int64_t rows, int c, int k, int64_t part_w, int64_t cols, int64_t ntiles,
                 long long* __restrict__ cnt, unsigned long long* __restrict__ nnz_bin) {
  extern __shared__ unsigned long long s_hist[];  // [2 * nbins]
  const int nbins = c * (k + 1) + 1;              // last bin: rows with no entry at all
  for (int i = threadIdx.x; i < 2 * nbins; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kTile + threadIdx.x;
  if (i < rows) {
    const int64_t cap = int64_t{1} << k;
    bool any = false;
    for (int p = 0; p < c; ++p) {
      RowPart rp = row_part(indptr, indices, i, p, c, part_w, cols);
      if (rp.l == 0) continue;
      any = true;
      int bin;
      unsigned long long nseg;
      if (rp.l > cap) {
        bin = p * (k + 1) + k;
        nseg = static_cast<unsigned long long>((rp.l + cap - 1) >> k);
      } else {
        bin = p * (k + 1) + ceil_log2_dev(rp.l);
        nseg = 1;
      }
      atomicAdd(&s_hist[bin], nseg);
      atomicAdd(&s_hist[nbins + bin], static_cast<unsigned long long>(rp.l));
    }
    if (!any) atomicAdd(&s_hist[nbins - 1], 1ull);
  }
  __syncthreads();
  for (int bin = threadIdx.x; bin < nbins; bin += blockDim.x) {
    cnt[static_cast<int64_t>(bin) * ntiles + blockIdx.x] = static_cast<long long>(s_hist[bin]);
    if (s_hist[nbins + bin]) atomicAdd(&nnz_bin[bin], s_hist[nbins + bin]);
  }
}

struct QueueEntry {
  long long base, q0, l;
  int row;
};

__global__ void __launch_bounds__(kTile)
hyb_scatter_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                   int64_t rows, int c, int k, int64_t part_w, int64_t cols, int64_t ntiles,
                   const long long* __restrict__ cnt, const long long* __restrict__ off,
                   int32_t* __restrict__ seg_row, long long* __restrict__ seg_src,
                   int32_t* __restrict__ seg_len, int32_t* __restrict__ empty_rows,
                   long long empty_base) {
  using Scan = cub::BlockScan<long long, kTile>;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ QueueEntry queue[kTile];
  __shared__ int qn;
  const int nbins = c * (k + 1) + 1;
  const int64_t t = blockIdx.x;
  const int64_t i = t * kTile + threadIdx.x;
  const bool valid = i < rows;
  const int64_t cap = int64_t{1} << k;
  bool any = false;
  if (threadIdx.x == 0) qn = 0;
  __syncthreads();
  for (int p = 0; p < c; ++p) {
    RowPart rp{0, 0};
    if (valid) rp = row_part(indptr, indices, i, p, c, part_w, cols);
    any |= rp.l > 0;
    int mybin = -1;
    long long nseg = 0;
    if (rp.l > 0) {
      mybin = rp.l > cap ? k : ceil_log2_dev(rp.l);
      nseg = rp.l > cap ? (rp.l + cap - 1) >> k : 1;
    }
    for (int bb = 0; bb <= k; ++bb) {
      const int bin = p * (k + 1) + bb;
      if (cnt[static_cast<int64_t>(bin) * ntiles + t] == 0) continue;  // CTA-uniform
      long long v = mybin == bb ? nseg : 0, rank;
      Scan(scan_tmp).ExclusiveSum(v, rank);
      if (v) {
        const long long base = off[static_cast<int64_t>(bin) * ntiles + t] + rank;
        if (v <= 8) {
          for (long long s = 0; s < v; ++s) {
            seg_row[base + s] = static_cast<int32_t>(i);
            seg_src[base + s] = rp.q0 + (s << k);
            seg_len[base + s] = static_cast<int32_t>(min64(cap, rp.l - (s << k)));
          }
        } else {  // long row: hand it to the whole CTA
          int slot = atomicAdd(&qn, 1);
          queue[slot] = {base, rp.q0, rp.l, static_cast<int>(i)};
        }
      }
      __syncthreads();
      const int nq = qn;
      for (int e = 0; e < nq; ++e) {
        const QueueEntry q = queue[e];
        const long long ns = (q.l + cap - 1) >> k;
        for (long long s = threadIdx.x; s < ns; s += kTile) {
          seg_row[q.base + s] = q.row;
          seg_src[q.base + s] = q.q0 + (s << k);
          seg_len[q.base + s] = static_cast<int32_t>(min64(cap, q.l - (s << k)));
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) qn = 0;
      __syncthreads();
    }
  }
  const int ebin = nbins - 1;
  if (cnt[static_cast<int64_t>(ebin) * ntiles + t] != 0) {
    long long v = (valid && !any) ? 1 : 0, rank;
    Scan(scan_tmp).ExclusiveSum(v, rank);
    if (v) empty_rows[off[static_cast<int64_t>(ebin) * ntiles + t] - empty_base + rank] =
        static_cast<int32_t>(i);
  }
}

struct FillPart {
  long long slot_off, row_off, nslots;
  int b;
};

__global__ void __launch_bounds__(256)
hyb_fill_kernel(const int32_t* __restrict__ indices, const float* __restrict__ values,
                const long long* __restrict__ seg_src, const int32_t* __restrict__ seg_len,
                int32_t* __restrict__ J, float* __restrict__ V, long long total_slots,
                const FillPart* __restrict__ parts, int nparts) {
  extern __shared__ FillPart sp[];  // [nparts]
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) sp[p] = parts[p];
  __syncthreads();
  for (long long slot = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       slot < total_slots; slot += static_cast<long long>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = nparts - 1;
    while (lo < hi) {  // last part with slot_off <= slot
      int mid = (lo + hi + 1) >> 1;
      if (sp[mid].slot_off <= slot) lo = mid; else hi = mid - 1;
    }
    const FillPart P = sp[lo];
    const long long local = slot - P.slot_off;
    if (local >= P.nslots) continue;  // alignment gap after a part (never read)
    const long long r = P.row_off + (local >> P.b);
    const int s = static_cast<int>(local & ((1ll << P.b) - 1));
    const long long src = seg_src[r];
    const int len = seg_len[r];
    if (s < len) {
      J[slot] = indices[src + s];
      V[slot] = values[src + s];
    } else {
      J[slot] = indices[src + len - 1];
      V[slot] = 0.0f;
    }
  }
}

// Chunk c of a split part "crosses" into c+1 when the last row of c and the first row of c+1
// are segments of the same source row.  A crossing run = one source row's chain of crossing
// boundaries; start = its first chunk, end = its last chunk.
__global__ void cross_flags_kernel(const int32_t* __restrict__ I, long long nrows, int rpc_log2,
                                   long long nchunks, unsigned char* __restrict__ fstart,
                                   unsigned char* __restrict__ fend) {
  const long long c = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= nchunks) return;
  auto cross = [&](long long cc) -> bool {
    if (cc < 0 || cc + 1 >= nchunks) return false;
    const long long r = (cc + 1) << rpc_log2;
    return r < nrows && I[r - 1] == I[r];
  };
  // A run passes *through* chunk c only if c holds a single source row (uniform); a chunk that
  // ends one split row and starts another is the end of one run and the start of the next.
  const long long r0 = c << rpc_log2, r1 = min64((c + 1) << rpc_log2, nrows);
  const bool uniform = I[r0] == I[r1 - 1];
  const bool xc = cross(c), xp = cross(c - 1);
  fstart[c] = xc && !(xp && uniform);
  fend[c] = xp && !(xc && uniform);
}

}  // namespace

void hyb_decompose_device(strata_hyb_impl& h, const int32_t* indptr, const int32_t* indices,
                          const float* values, cudaStream_t s) {
  const int c = h.c, k = h.k;
  const int64_t rows = h.rows, cols = h.cols;
  const int nbins = c * (k + 1) + 1;
  const int64_t ntiles = (rows + kTile - 1) / kTile;
  const int64_t part_w = (cols + c - 1) / c;  // storage.cpp:280

  h.parts.clear();
  h.n_empty = 0;
  h.padding_ratio = 0.0;
  if (rows == 0) return;

  DevBuf<long long> cnt(static_cast<size_t>(nbins) * ntiles + 1), off(cnt.n);
  DevBuf<unsigned long long> nnz_bin(nbins);
  STRATA_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, cnt.n * sizeof(long long), s));
  STRATA_CUDA_CHECK(cudaMemsetAsync(nnz_bin.p, 0, nnz_bin.n * sizeof(unsigned long long), s));
  hyb_count_kernel<<<static_cast<unsigned>(ntiles), kTile, 2 * nbins * sizeof(unsigned long long),
                     s>>>(indptr, indices, rows, c, k, part_w, cols, ntiles, cnt.p, nnz_bin.p);
  STRATA_CUDA_CHECK(cudaGetLastError());

  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, off.p, static_cast<int64_t>(cnt.n), s);
  DevBuf<unsigned char> tmp(tmp_bytes);
  cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, off.p, static_cast<int64_t>(cnt.n), s);
  STRATA_CUDA_CHECK(cudaGetLastError());

  // Per-bin start positions (bin * ntiles), plus the grand total at index nbins * ntiles.
  std::vector<long long> bin_start(nbins + 1);
  std::vector<unsigned long long> bin_nnz(nbins);
  STRATA_CUDA_CHECK(cudaMemcpy2DAsync(bin_start.data(), sizeof(long long), off.p,
                                      ntiles * sizeof(long long), sizeof(long long), nbins + 1,
                                      cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaMemcpyAsync(bin_nnz.data(), nnz_bin.p, nbins * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));

  const long long total_segs = bin_start[nbins - 1];  // empty bin is last
  h.n_empty = bin_start[nbins] - bin_start[nbins - 1];

  // Part table (storage.cpp:316-331): non-empty bins in bin order.
  int64_t slot_cursor = 0, pads = 0, slots = 0;
  for (int bin = 0; bin < nbins - 1; ++bin) {
    const long long nseg = bin_start[bin + 1] - bin_start[bin];
    if (nseg == 0) continue;
    HybPart P;
    P.partition = bin / (k + 1);
    P.bucket = bin % (k + 1);
    P.width = int64_t{1} << P.bucket;
    P.nrows = nseg;
    P.nnz = static_cast<int64_t>(bin_nnz[bin]);
    P.pad_slots = P.nrows * P.width - P.nnz;
    P.col_lo = static_cast<int64_t>(P.partition) * part_w;
    P.col_hi = std::min<int64_t>(cols, (P.partition + 1) * part_w);
    P.row_off = bin_start[bin];
    if (P.nrows * P.width > INT32_MAX - 256)  // the SpMM keeps part-local slot indices in 32 bits
      throw ApiError(STRATA_ERR_CAPACITY, "hyb part exceeds 2^31 ELL slots");
    P.slot_off = slot_cursor;  // multiple of 8 slots: the SpMM reads 8-slot tiles as int4 pairs
    slot_cursor += (P.nrows * P.width + 7) & ~int64_t{7};
    pads += P.pad_slots;
    slots += P.nrows * P.width;
    h.parts.push_back(P);
  }
  h.padding_ratio = slots == 0 ? 0.0 : static_cast<double>(pads) / static_cast<double>(slots);

  h.I.alloc(total_segs);
  h.J.alloc(slot_cursor);
  h.V.alloc(slot_cursor);
  h.empty_rows.alloc(h.n_empty);
  DevBuf<long long> seg_src(total_segs);
  DevBuf<int32_t> seg_len(total_segs);
  if (ntiles > 0) {
    hyb_scatter_kernel<<<static_cast<unsigned>(ntiles), kTile, 0, s>>>(
        indptr, indices, rows, c, k, part_w, cols, ntiles, cnt.p, off.p, h.I.p, seg_src.p,
        seg_len.p, h.empty_rows.p, bin_start[nbins - 1]);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }
  if (slot_cursor > 0) {
    std::vector<FillPart> fp;
    for (const auto& P : h.parts) fp.push_back({P.slot_off, P.row_off, P.nrows * P.width, P.bucket});
    DevBuf<FillPart> dfp(fp.size());
    STRATA_CUDA_CHECK(cudaMemcpyAsync(dfp.p, fp.data(), fp.size() * sizeof(FillPart),
                                      cudaMemcpyHostToDevice, s));
    const long long blocks = std::min<long long>((slot_cursor + 255) / 256, 148LL * 64);
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(hyb_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(std::max<size_t>(fp.size() * sizeof(FillPart), 1))));
    hyb_fill_kernel<<<static_cast<unsigned>(blocks), 256, fp.size() * sizeof(FillPart), s>>>(
        indices, values, seg_src.p, seg_len.p, h.J.p, h.V.p, slot_cursor, dfp.p,
        static_cast<int>(fp.size()));
    STRATA_CUDA_CHECK(cudaGetLastError());
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));  // dfp / seg_* are freed on return
  }

  // SpMM schedule.
  std::vector<FixTile> tiles;
  std::vector<FixRun> runs;
  h.fix_ranges.clear();
  int64_t carry_chunks = 0, l2_slots = 0;
  for (auto& P : h.parts) {
    P.rpc_log2 = std::max(0, 8 - P.bucket);  // kSlotsPerChunk = 256 slots per chunk
    static_assert(kSlotsPerChunk == 256, "rpc rule assumes 256-slot chunks");
    P.nchunks = (P.nrows + (int64_t{1} << P.rpc_log2) - 1) >> P.rpc_log2;
    P.may_split = (P.bucket == k);  // only bucket k may hold several segments of one row
    P.nruns = 0;
    P.carry_off = 0;
    if (h.fix_ranges.empty() || h.fix_ranges.back().partition != P.partition)
      h.fix_ranges.push_back({P.partition, (long long)tiles.size(), (long long)tiles.size(),
                              (long long)runs.size(), (long long)runs.size()});
    if (!P.may_split || P.nchunks < 2) continue;
    DevBuf<unsigned char> fs(P.nchunks), fe(P.nchunks);
    cross_flags_kernel<<<static_cast<unsigned>((P.nchunks + 255) / 256), 256, 0, s>>>(
        h.I.p + P.row_off, P.nrows, P.rpc_log2, P.nchunks, fs.p, fe.p);
    STRATA_CUDA_CHECK(cudaGetLastError());
    DevBuf<long long> rs(P.nchunks), re(P.nchunks);
    DevBuf<long long> nsel(2);
    cub::CountingInputIterator<long long> it(0);
    size_t tb = 0, tb2 = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, it, fs.p, rs.p, nsel.p, P.nchunks, s);
    cub::DeviceSelect::Flagged(nullptr, tb2, it, fe.p, re.p, nsel.p + 1, P.nchunks, s);
    DevBuf<unsigned char> t2(std::max(tb, tb2));
    cub::DeviceSelect::Flagged(t2.p, tb, it, fs.p, rs.p, nsel.p, P.nchunks, s);
    cub::DeviceSelect::Flagged(t2.p, tb2, it, fe.p, re.p, nsel.p + 1, P.nchunks, s);
    STRATA_CUDA_CHECK(cudaGetLastError());
    long long hn[2];
    STRATA_CUDA_CHECK(cudaMemcpyAsync(hn, nsel.p, sizeof(hn), cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    if (hn[0] != hn[1]) throw ApiError(STRATA_ERR_INTERNAL, "hyb: unbalanced split runs");
    P.nruns = hn[0];
    P.carry_off = carry_chunks;
    carry_chunks += P.nchunks;
    if (!P.nruns) continue;
    std::vector<long long> a(P.nruns), b(P.nruns);
    std::vector<int32_t> Ih(P.nrows);
    STRATA_CUDA_CHECK(cudaMemcpy(a.data(), rs.p, P.nruns * sizeof(long long), cudaMemcpyDeviceToHost));
    STRATA_CUDA_CHECK(cudaMemcpy(b.data(), re.p, P.nruns * sizeof(long long), cudaMemcpyDeviceToHost));
    STRATA_CUDA_CHECK(cudaMemcpy(Ih.data(), h.I.p + P.row_off, P.nrows * sizeof(int32_t),
                                 cudaMemcpyDeviceToHost));
    for (long long j = 0; j < P.nruns; ++j) {
      // Run j: chunks a[j]..b[j]; contributions in order = tail carry of a[j], then the head
      // carries of a[j]+1 .. b[j].  Its output row is the last row of chunk a[j].
      const long long ca = a[j], n = b[j] - a[j] + 1;
      const long long row = Ih[((ca + 1) << P.rpc_log2) - 1];
      const long long nt = (n + kFixTile - 1) / kFixTile;
      for (long long u = 0; u < nt; ++u) {
        FixTile t;
        t.carry0 = P.carry_off + ca + u * kFixTile;
        t.count = static_cast<int>(std::min<long long>(kFixTile, n - u * kFixTile));
        t.first_slot = u == 0 ? 1 : 0;
        t.out = nt == 1 ? row : -(l2_slots + u + 1);
        tiles.push_back(t);
      }
      if (nt > 1) {
        runs.push_back({l2_slots, row, static_cast<int>(nt), 0});
        l2_slots += nt;
      }
    }
    h.fix_ranges.back().tile_end = static_cast<long long>(tiles.size());
    h.fix_ranges.back().run_end = static_cast<long long>(runs.size());
  }
  h.total_chunks_carry = carry_chunks;
  h.l2_slots = l2_slots;
  h.fix_tiles.alloc(tiles.size());
  h.fix_runs.alloc(runs.size());
  if (!tiles.empty())
    STRATA_CUDA_CHECK(cudaMemcpy(h.fix_tiles.p, tiles.data(), tiles.size() * sizeof(FixTile),
                                 cudaMemcpyHostToDevice));
  if (!runs.empty())
    STRATA_CUDA_CHECK(cudaMemcpy(h.fix_runs.p, runs.data(), runs.size() * sizeof(FixRun),
                                 cudaMemcpyHostToDevice));
}


// ---- row-work balance (tune.cpp:46-76 hyb_balance) ---------------------------------------
namespace {
// Per ELL row of one part: real (non-padding) slots; per part the max and the sum.
__global__ void row_work_kernel(const int32_t* __restrict__ J, long long nrows, int w,
                                unsigned long long* __restrict__ out /* [max, sum] */) {
  unsigned long long mx = 0, sum = 0;
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < nrows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int32_t* row = J + r * w;
    unsigned long long real = 1;
    for (int k = 1; k < w; ++k) real += row[k] != row[k - 1];
    mx = max(mx, real);
    sum += real;
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, mx);
    atomicAdd(out + 1, sum);
  }
}
}  // namespace

double hyb_row_work_balance(const strata_hyb_impl& h, cudaStream_t s) {
  double worst = 1.0;
  if (h.parts.empty()) return worst;
  DevBuf<unsigned long long> acc(2 * h.parts.size());
  STRATA_CUDA_CHECK(cudaMemsetAsync(acc.p, 0, acc.n * sizeof(unsigned long long), s));
  for (size_t i = 0; i < h.parts.size(); ++i) {
    const HybPart& P = h.parts[i];
    if (P.nrows == 0) continue;
    const unsigned g = static_cast<unsigned>(std::min<long long>((P.nrows + 255) / 256, num_sms() * 8LL));
    row_work_kernel<<<g, 256, 0, s>>>(h.J.p + P.slot_off, P.nrows, static_cast<int>(P.width), acc.p + 2 * i);
  }
  STRATA_CUDA_CHECK(cudaGetLastError());
  std::vector<unsigned long long> hv(acc.n);
  STRATA_CUDA_CHECK(cudaMemcpyAsync(hv.data(), acc.p, acc.n * sizeof(unsigned long long),
                                    cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  for (size_t i = 0; i < h.parts.size(); ++i) {
    if (h.parts[i].nrows == 0 || hv[2 * i + 1] == 0) continue;
    const double mean = static_cast<double>(hv[2 * i + 1]) / static_cast<double>(h.parts[i].nrows);
    worst = std::max(worst, static_cast<double>(hv[2 * i]) / mean);
  }
  return worst;
}
}  // namespace strata_b200
