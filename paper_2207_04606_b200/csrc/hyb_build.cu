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
#include <cstdlib>

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

// ---- SpMM fix-up schedule, built on the device -------------------------------------------
// Per split part (bucket k), after the crossing runs are selected (rs[j], re[j]: first / last
// chunk of run j, j < nruns): a run of n = re - rs + 1 contributions needs ceil(n / kFixTile)
// level-1 tiles and, when that is more than one, a level-2 run entry with as many slots.
// Counts per run -> exclusive scans over all split parts in part order -> entries.  Runs of
// part pi live at [carry_off, carry_off + nchunks) of the concatenated per-chunk arrays.
__global__ void run_counts_kernel(const long long* __restrict__ rs, const long long* __restrict__ re,
                                  const long long* __restrict__ nsel, long long nchunks,
                                  long long* __restrict__ ntile, long long* __restrict__ nl2,
                                  long long* __restrict__ isrun) {
  const long long nruns = nsel[0];
  for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < nchunks;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long nt = 0;
    if (j < nruns) nt = (re[j] - rs[j] + 1 + kFixTile - 1) / kFixTile;
    ntile[j] = nt;
    nl2[j] = nt > 1 ? nt : 0;
    isrun[j] = nt > 1 ? 1 : 0;
  }
}

__global__ void fix_fill_kernel(const long long* __restrict__ rs, const long long* __restrict__ re,
                                const long long* __restrict__ nsel, const int32_t* __restrict__ I,
                                int rpc_log2, long long carry_off,
                                const long long* __restrict__ tile_off,
                                const long long* __restrict__ l2_off,
                                const long long* __restrict__ run_off, FixTile* __restrict__ tiles,
                                FixRun* __restrict__ runs) {
  const long long nruns = nsel[0];
  for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j < nruns;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    // Run j: chunks rs..re; contributions in order = tail carry of rs, then the head carries
    // of rs+1 .. re.  Its output row is the last row of chunk rs.
    const long long ca = rs[j], n = re[j] - ca + 1;
    const long long row = I[((ca + 1) << rpc_log2) - 1];
    const long long nt = (n + kFixTile - 1) / kFixTile;
    const long long t0 = tile_off[j], l2 = l2_off[j];
    for (long long u = 0; u < nt; ++u) {
      FixTile t;
      t.carry0 = carry_off + ca + u * kFixTile;
      t.count = static_cast<int>(min64(kFixTile, n - u * kFixTile));
      t.first_slot = u == 0 ? 1 : 0;
      t.out = nt == 1 ? row : -(l2 + u + 1);
      tiles[t0 + u] = t;
    }
    if (nt > 1) runs[run_off[j]] = FixRun{l2, row, static_cast<int>(nt), 0};
  }
}

unsigned grid_of(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, 148LL * 16)));
}

}  // namespace

// Two host synchronisations, both to size allocations: the per-bin totals (part table, ELL
// arrays) and the fix-up schedule totals.  Temporaries come from the stream-ordered pool and
// are released in stream order; the handle's arrays are pooled too (no cudaMalloc/cudaFree
// device-wide syncs), so a rebuilt plan of the same size reuses cached memory.
void hyb_decompose_device(strata_hyb_impl& h, const int32_t* indptr, const int32_t* indices,
                          const float* values, cudaStream_t s) {
  const int c = h.c, k = h.k;
  const int64_t rows = h.rows, cols = h.cols;
  const int nbins = c * (k + 1) + 1;
  const int64_t ntiles = (rows + kTile - 1) / kTile;
  const int64_t part_w = (cols + c - 1) / c;  // storage.cpp:280

  h.parts.clear();
  h.fix_ranges.clear();
  h.n_empty = 0;
  h.padding_ratio = 0.0;
  h.total_chunks_carry = 0;
  h.l2_slots = 0;
  if (rows == 0) return;

  DevBuf<long long> cnt(static_cast<size_t>(nbins) * ntiles + 1, s), off(cnt.n, s);
  DevBuf<unsigned long long> nnz_bin(nbins, s);
  STRATA_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, cnt.n * sizeof(long long), s));
  STRATA_CUDA_CHECK(cudaMemsetAsync(nnz_bin.p, 0, nnz_bin.n * sizeof(unsigned long long), s));
  hyb_count_kernel<<<static_cast<unsigned>(ntiles), kTile, 2 * nbins * sizeof(unsigned long long),
                     s>>>(indptr, indices, rows, c, k, part_w, cols, ntiles, cnt.p, nnz_bin.p);
  STRATA_CUDA_CHECK(cudaGetLastError());

  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt.p, off.p, static_cast<int64_t>(cnt.n), s);
  {
    DevBuf<unsigned char> tmp(tmp_bytes, s);
    cub::DeviceScan::ExclusiveSum(tmp.p, tmp_bytes, cnt.p, off.p, static_cast<int64_t>(cnt.n), s);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }

  // Sync 1: per-bin start positions (bin * ntiles) + the grand total, and per-bin entries.
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

  static const bool pooled = getenv("STRATA_HYB_POOL") && atoi(getenv("STRATA_HYB_POOL")) == 1;  // A/B knob
  if (pooled) {
    h.I.alloc_async(total_segs, s, true);
    h.J.alloc_async(slot_cursor, s, true);
    h.V.alloc_async(slot_cursor, s, true);
    h.empty_rows.alloc_async(h.n_empty, s, true);
  } else {
    h.I.alloc(total_segs);
    h.J.alloc(slot_cursor);
    h.V.alloc(slot_cursor);
    h.empty_rows.alloc(h.n_empty);
  }
  DevBuf<long long> seg_src(total_segs, s);
  DevBuf<int32_t> seg_len(total_segs, s);
  if (ntiles > 0) {
    hyb_scatter_kernel<<<static_cast<unsigned>(ntiles), kTile, 0, s>>>(
        indptr, indices, rows, c, k, part_w, cols, ntiles, cnt.p, off.p, h.I.p, seg_src.p,
        seg_len.p, h.empty_rows.p, bin_start[nbins - 1]);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }
  if (slot_cursor > 0) {
    std::vector<FillPart> fp;
    for (const auto& P : h.parts) fp.push_back({P.slot_off, P.row_off, P.nrows * P.width, P.bucket});
    DevBuf<FillPart> dfp(fp.size(), s);
    STRATA_CUDA_CHECK(cudaMemcpyAsync(dfp.p, fp.data(), fp.size() * sizeof(FillPart),
                                      cudaMemcpyHostToDevice, s));
    const size_t smem = std::max<size_t>(fp.size() * sizeof(FillPart), 1);
    if (smem > 48 * 1024)
      STRATA_CUDA_CHECK(cudaFuncSetAttribute(hyb_fill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem)));
    const long long blocks = std::min<long long>((slot_cursor + 255) / 256, 148LL * 64);
    hyb_fill_kernel<<<static_cast<unsigned>(blocks), 256, smem, s>>>(
        indices, values, seg_src.p, seg_len.p, h.J.p, h.V.p, slot_cursor, dfp.p,
        static_cast<int>(fp.size()));
    STRATA_CUDA_CHECK(cudaGetLastError());
    // (a pageable-source cudaMemcpyAsync returns once `fp` is staged: no sync needed for it)
  }

  // SpMM schedule: rows per chunk per part; the bucket-k part (the only one whose I_indices
  // may repeat) gets its crossing runs, selected and expanded into fix-up tiles on the device.
  std::vector<size_t> split;  // indices of split parts with >= 2 chunks
  int64_t carry_chunks = 0;
  for (size_t pi = 0; pi < h.parts.size(); ++pi) {
    HybPart& P = h.parts[pi];
    P.rpc_log2 = std::max(0, 8 - P.bucket);  // kSlotsPerChunk = 256 slots per chunk
    static_assert(kSlotsPerChunk == 256, "rpc rule assumes 256-slot chunks");
    P.nchunks = (P.nrows + (int64_t{1} << P.rpc_log2) - 1) >> P.rpc_log2;
    P.may_split = (P.bucket == k);
    P.nruns = 0;
    P.carry_off = 0;
    if (!P.may_split || P.nchunks < 2) continue;
    P.carry_off = carry_chunks;
    carry_chunks += P.nchunks;
    split.push_back(pi);
  }
  h.total_chunks_carry = carry_chunks;

  DevBuf<long long> rs, re, nsel, ntile, nl2, isrun, tile_off, l2_off, run_off;
  if (!split.empty()) {
    const size_t tot = static_cast<size_t>(carry_chunks);
    rs.alloc_async(tot, s);
    re.alloc_async(tot, s);
    nsel.alloc_async(2 * split.size(), s);
    ntile.alloc_async(tot + 1, s);
    nl2.alloc_async(tot + 1, s);
    isrun.alloc_async(tot + 1, s);
    tile_off.alloc_async(tot + 1, s);
    l2_off.alloc_async(tot + 1, s);
    run_off.alloc_async(tot + 1, s);
    DevBuf<unsigned char> fs(tot, s), fe(tot, s);
    cub::CountingInputIterator<long long> it(0);
    size_t tb = 0;
    for (size_t si = 0; si < split.size(); ++si) {
      const HybPart& P = h.parts[split[si]];
      size_t t1 = 0;
      cub::DeviceSelect::Flagged(nullptr, t1, it, fs.p, rs.p, nsel.p, P.nchunks, s);
      tb = std::max(tb, t1);
    }
    DevBuf<unsigned char> t2(tb, s);
    for (size_t si = 0; si < split.size(); ++si) {
      const HybPart& P = h.parts[split[si]];
      const long long o = P.carry_off;
      cross_flags_kernel<<<grid_of(P.nchunks), 256, 0, s>>>(h.I.p + P.row_off, P.nrows, P.rpc_log2,
                                                            P.nchunks, fs.p + o, fe.p + o);
      size_t t1 = tb;
      cub::DeviceSelect::Flagged(t2.p, t1, it, fs.p + o, rs.p + o, nsel.p + 2 * si, P.nchunks, s);
      t1 = tb;
      cub::DeviceSelect::Flagged(t2.p, t1, it, fe.p + o, re.p + o, nsel.p + 2 * si + 1, P.nchunks, s);
      run_counts_kernel<<<grid_of(P.nchunks), 256, 0, s>>>(rs.p + o, re.p + o, nsel.p + 2 * si,
                                                           P.nchunks, ntile.p + o, nl2.p + o,
                                                           isrun.p + o);
    }
    STRATA_CUDA_CHECK(cudaGetLastError());
    for (DevBuf<long long>* a : {&ntile, &nl2, &isrun})
      STRATA_CUDA_CHECK(cudaMemsetAsync(a->p + tot, 0, sizeof(long long), s));
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, ntile.p, tile_off.p, static_cast<int64_t>(tot + 1), s);
    DevBuf<unsigned char> t3(sb, s);
    for (auto [in, out] : {std::pair{&ntile, &tile_off}, {&nl2, &l2_off}, {&isrun, &run_off}}) {
      size_t sb2 = sb;
      cub::DeviceScan::ExclusiveSum(t3.p, sb2, in->p, out->p, static_cast<int64_t>(tot + 1), s);
    }
    STRATA_CUDA_CHECK(cudaGetLastError());
    // Sync 2: per split part its run counts (selected starts / ends) and the scan positions
    // at its first chunk, plus the totals.
    std::vector<long long> hsel(2 * split.size());
    STRATA_CUDA_CHECK(cudaMemcpyAsync(hsel.data(), nsel.p, hsel.size() * sizeof(long long),
                                      cudaMemcpyDeviceToHost, s));
    std::vector<long long> tb_h(split.size() + 1), rb_h(split.size() + 1), l2_h(split.size() + 1);
    for (size_t si = 0; si <= split.size(); ++si) {
      const long long o = si < split.size() ? h.parts[split[si]].carry_off : carry_chunks;
      STRATA_CUDA_CHECK(cudaMemcpyAsync(&tb_h[si], tile_off.p + o, sizeof(long long), cudaMemcpyDeviceToHost, s));
      STRATA_CUDA_CHECK(cudaMemcpyAsync(&rb_h[si], run_off.p + o, sizeof(long long), cudaMemcpyDeviceToHost, s));
      STRATA_CUDA_CHECK(cudaMemcpyAsync(&l2_h[si], l2_off.p + o, sizeof(long long), cudaMemcpyDeviceToHost, s));
    }
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    for (size_t si = 0; si < split.size(); ++si) {
      if (hsel[2 * si] != hsel[2 * si + 1]) throw ApiError(STRATA_ERR_INTERNAL, "hyb: unbalanced split runs");
      h.parts[split[si]].nruns = hsel[2 * si];
    }
    h.l2_slots = l2_h[split.size()];
    h.fix_tiles.alloc_async(tb_h[split.size()], s, true);
    h.fix_runs.alloc_async(rb_h[split.size()], s, true);
    for (size_t si = 0; si < split.size(); ++si) {
      const HybPart& P = h.parts[split[si]];
      if (!P.nruns) continue;
      const long long o = P.carry_off;
      fix_fill_kernel<<<grid_of(P.nruns), 256, 0, s>>>(rs.p + o, re.p + o, nsel.p + 2 * si,
                                                       h.I.p + P.row_off, P.rpc_log2, o,
                                                       tile_off.p + o, l2_off.p + o, run_off.p + o,
                                                       h.fix_tiles.p, h.fix_runs.p);
    }
    STRATA_CUDA_CHECK(cudaGetLastError());
    // per column partition, in partition order: its split part's tiles / runs (empty ranges
    // for partitions without one)
    size_t si = 0;
    for (const auto& P : h.parts) {
      if (!h.fix_ranges.empty() && h.fix_ranges.back().partition == P.partition) continue;
      while (si < split.size() && h.parts[split[si]].partition < P.partition) ++si;
      const bool has = si < split.size() && h.parts[split[si]].partition == P.partition;
      const size_t b0 = si, b1 = has ? si + 1 : si;
      h.fix_ranges.push_back({P.partition, tb_h[b0], tb_h[b1], rb_h[b0], rb_h[b1]});
    }
  } else {
    for (const auto& P : h.parts)
      if (h.fix_ranges.empty() || h.fix_ranges.back().partition != P.partition)
        h.fix_ranges.push_back({P.partition, 0, 0, 0, 0});
  }
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
