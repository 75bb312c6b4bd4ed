// rgms.cu — RGMS / RGCN aggregation on tcgen05 tensor cores.
//
// Reference op (kernels.cpp:138-167, driver.cpp:241-314):
//   Y[i, l] = sum_r sum_j A[r, i, j] * sum_k X[j, k] * W[r, k, l]
// over the RelSparse layout (kernels.cpp:19-62): relation-major edges, rows ascending inside a
// relation.  Flattened here to rel_ptr[R+1] / dst / src / A.
//
// Two passes, no atomics, deterministic:
//   plan   (once, like build_rgms_pipeline's decomposition): per-relation 128-edge tiles;
//          message *runs* (consecutive edges of one relation with one destination inside a
//          32-edge warp group) get rows of T in destination order (stable radix sort, so a row's
//          runs stay in relation order) and the row pointer dptr.
//   pass 1 rgms_edge_gemm_kernel — warp-specialised, mbarrier-pipelined: producers gather the
//          tile's 128 X rows (cp.async into the swizzled K-major A operand) and TMA-load W_r and
//          the index block; one thread issues tcgen05.mma M = 128 edges, N = d_out, K = d_in
//          into a double-buffered TMEM accumulator; four epilogue warps scale by A, sum runs and
//          write one message row per run.
//   pass 2 rgms_row_sum_kernel — Y[i] = sum_{q in [dptr i, dptr i+1)} T[q] (contiguous rows,
//          streamed once; empty rows write 0 as the reference's zero-initialised Y); rows with
//          more than kLong runs go through fixed-shape chunk partials (long_chunk / finish).
// Why not scatter with atomics: the 5.7M x d_out red.global.add into a Y larger than L2 was
// the bottleneck of the first version (3.7 ms at C4); T costs 2 * runs * d_out * 4 bytes of
// streaming traffic instead.
// Numerics: f32 products / tensor-core f32 accumulation over k, one f32 multiply by A, f32
// run and row sums in relation order — exact on the reference's integer operands.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <cuda_bf16.h>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

using namespace strata_b200;

struct strata_rgms {
  int device = 0;
  int64_t R = 0, m = 0, n = 0, nnz = 0;
  int64_t ntiles = 0;            // 128-edge tiles (tiles never straddle relations)
  int64_t nruns = 0;             // message runs (see run_heads_kernel)
  int64_t trows = 0;             // T rows: the runs of rows with >= 2 runs (the sole run of a
                                 // row goes straight to Y from pass 1: a "direct" row)
  DevBuf<uint32_t> dbits;        // [ceil(m/32)] bit r of word b: row 32b + r is direct
  DevBuf<int32_t> edges;         // [ntiles][kTileWords] per-tile edge blocks (see below)
  DevBuf<int32_t> dptr;          // [m+1] row pointer into the destination-sorted order
  int nlong = 0, nchunks = 0;     // rows with > kLong edges and their kChunk-edge chunks
  DevBuf<int32_t> long_rows;     // [nlong] ascending
  DevBuf<int32_t> chunk_off;     // [nlong+1] first chunk of long row li
  // Pass 2's work list: the rows it writes (>= 2 runs, or no edge at all), ascending, and
  // their T-row pointer (cptr[j] = dptr[rowlist[j]], cptr[nlist] = trows).
  int64_t nlist = 0;
  DevBuf<int32_t> rowlist, cptr;
};

namespace {

constexpr int kEdges = 128;  // UMMA M

__global__ void rel_tiles_kernel(const int32_t* __restrict__ rel_ptr, long long R,
                                 long long* __restrict__ ntiles) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < R) ntiles[r] = (rel_ptr[r + 1] - rel_ptr[r] + kEdges - 1) / kEdges;
  if (r == R) ntiles[R] = 0;
}

__global__ void tile_rel_kernel(const long long* __restrict__ tile_start, long long R,
                                int32_t* __restrict__ tile_rel) {
  const long long r = blockIdx.x;
  for (long long t = tile_start[r] + threadIdx.x; t < tile_start[r + 1]; t += blockDim.x)
    tile_rel[t] = static_cast<int32_t>(r);
}

__global__ void iota_kernel(int32_t* __restrict__ v, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    v[i] = static_cast<int32_t>(i);
}

// pos[order[q]] = q: edge e's slot in the destination-sorted order.
__global__ void invert_kernel(const int32_t* __restrict__ order, long long n,
                              int32_t* __restrict__ pos) {
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
       q += static_cast<long long>(gridDim.x) * blockDim.x)
    pos[order[q]] = static_cast<int32_t>(q);
}

// dptr[i] = first q with sorted_dst[q] >= i (i = 0..m).
__global__ void row_ptr_kernel(const int32_t* __restrict__ sorted_dst, long long nnz, long long m,
                               int32_t* __restrict__ dptr) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i <= m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (sorted_dst[mid] < i) lo = mid + 1; else hi = mid;
    }
    dptr[i] = static_cast<int32_t>(lo);
  }
}

// Per-tile edge block in HBM (built by the plan; tile-padded so every block is 16-byte aligned
// and one tile's indices are 97 contiguous 16-byte chunks):
//   [0..3] header {relation r, edges ne, 0, 0}; [4..131] src; [132..259] pos (-1 = pad);
//   [260..387] A (f32 bits).
constexpr int kTileWords = 4 + 3 * kEdges;
constexpr int kTileChunks = kTileWords / 4;  // 97

// Message runs: consecutive edges of one relation with the same destination inside one 32-edge
// warp group of a tile are summed in pass 1's epilogue and leave one T row (a "run").  head[e]
// marks the first edge of a run.
__global__ void run_heads_kernel(const int32_t* __restrict__ rel_ptr,
                                 const long long* __restrict__ tile_start,
                                 const int32_t* __restrict__ tile_rel, long long ntiles,
                                 const int32_t* __restrict__ dst, int32_t* __restrict__ head) {
  for (long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       s < ntiles * kEdges; s += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = s / kEdges;
    const int i = static_cast<int>(s % kEdges);
    const int r = tile_rel[t];
    const long long e = rel_ptr[r] + (t - tile_start[r]) * kEdges + i;
    if (e < rel_ptr[r + 1]) head[e] = (i % 32 == 0 || dst[e] != dst[e - 1]) ? 1 : 0;
  }
}

// run_dst[run of e] = dst[e] for run heads (run = inclusive-scan(head)[e] - 1).
__global__ void run_dst_kernel(const int32_t* __restrict__ head, const int32_t* __restrict__ incl,
                               const int32_t* __restrict__ dst, long long nnz,
                               int32_t* __restrict__ run_dst) {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += static_cast<long long>(gridDim.x) * blockDim.x)
    if (head[e]) run_dst[incl[e] - 1] = dst[e];
}

// Direct rows: a row with exactly one run needs no T row — pass 1 writes its sum to Y.
// dflag[q] = 1 when the run at destination-sorted position q is its row's only run.
__global__ void direct_flags_kernel(const int32_t* __restrict__ keys, long long nr,
                                    const int32_t* __restrict__ dptr, int32_t* __restrict__ dflag) {
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q <= nr;
       q += static_cast<long long>(gridDim.x) * blockDim.x)
    dflag[q] = q < nr && dptr[keys[q] + 1] - dptr[keys[q]] == 1 ? 1 : 0;
}

// Run r's pos word: -(3 + row) for a direct run, else its compacted T row.
__global__ void direct_pos_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ dflag,
                                  const int32_t* __restrict__ dbefore, long long nr,
                                  int32_t* __restrict__ run_pos) {
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r < nr;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int q = run_pos[r];
    run_pos[r] = dflag[q] ? -3 - keys[q] : q - dbefore[q];
  }
}

// Direct-row bitmask (from the uncompacted dptr), then dptr[i] -= direct runs before it.
__global__ void direct_bits_kernel(const int32_t* __restrict__ dptr, long long m,
                                   uint32_t* __restrict__ dbits) {
  const long long nw = (m + 31) / 32 * 32;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nw;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool d = i < m && dptr[i + 1] - dptr[i] == 1;
    const unsigned w = __ballot_sync(0xffffffffu, d);
    if ((threadIdx.x & 31) == 0) dbits[i / 32] = w;
  }
}

__global__ void compact_dptr_kernel(const int32_t* __restrict__ dbefore, long long m,
                                    int32_t* __restrict__ dptr) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i <= m;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    dptr[i] -= dbefore[dptr[i]];
}

__global__ void nondirect_flags_kernel(const uint32_t* __restrict__ dbits, long long m,
                                       uint8_t* __restrict__ flag) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    flag[i] = ((dbits[i >> 5] >> (i & 31)) & 1u) ? 0 : 1;
}

__global__ void list_ptr_kernel(const int32_t* __restrict__ rowlist, const int32_t* __restrict__ dptr,
                                long long n, long long m, int32_t* __restrict__ cptr) {
  for (long long j = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; j <= n;
       j += static_cast<long long>(gridDim.x) * blockDim.x)
    cptr[j] = dptr[j < n ? rowlist[j] : m];
}

// Per-tile edge blocks; the pos word of an edge is its run's T row for a run head (or
// -(3 + row) for a direct row's run), -2 for a run continuation and -1 for padding.
__global__ void tile_edges_kernel(const int32_t* __restrict__ rel_ptr, long long R,
                                  const long long* __restrict__ tile_start,
                                  const int32_t* __restrict__ tile_rel, long long ntiles,
                                  const int32_t* __restrict__ src, const int32_t* __restrict__ head,
                                  const int32_t* __restrict__ incl, const int32_t* __restrict__ run_pos,
                                  const float* __restrict__ A, int32_t* __restrict__ ed) {
  for (long long s = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
       s < ntiles * kEdges; s += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long t = s / kEdges;
    const int i = static_cast<int>(s % kEdges);
    const int r = tile_rel[t];
    const long long base = rel_ptr[r] + (t - tile_start[r]) * kEdges;
    const long long e = base + i;
    const bool valid = e < rel_ptr[r + 1];
    int32_t* blk = ed + t * kTileWords;
    blk[4 + i] = valid ? src[e] : 0;
    blk[4 + kEdges + i] = valid ? (head[e] ? run_pos[incl[e] - 1] : -2) : -1;
    blk[4 + 2 * kEdges + i] = valid ? __float_as_int(A[e]) : 0;
    if (i < 4)
      blk[i] = i == 0 ? static_cast<int>(r % R)
                      : (i == 1 ? static_cast<int>(min64(kEdges, rel_ptr[r + 1] - base)) : 0);
  }
}

// ---- pass 1: warp-specialised, mbarrier-pipelined tcgen05 tiles --------------------------
// Roles (224 threads):
//   warps 0-1 producers: index blocks kIdxAhead tiles ahead (1-D TMA bulk copies); per tile,
//           once its stage is free, W_r by d_out/8 TMA boxes {8 columns x d_in} into the
//           MN-major (SWIZZLE_NONE) B operand, and the 128 X rows by 16-byte cp.async chunks
//           written to their swizzled positions of the K-major A operand, completing on the
//           stage's mbarrier (cp.async.mbarrier.arrive.noinc).  (TMA tile::gather4 of the rows
//           works too — 4 rows per op — but measured 8 % slower at C4: 288 vs 266 us.)
//   warp 2  MMA issuer (lane 0): tcgen05.mma M = 128 edges, N = d_out, K = d_in into one of two
//           TMEM accumulators; tcgen05.commit frees the stage and publishes the accumulator;
//   warps 3-6 epilogue: tcgen05.ld of their 32 TMEM lanes, scale by A, per-warp swizzled
//           transpose through shared memory, one message row per run (st.global.cs), then
//           release the accumulator and the index block.
// Every hand-off is an mbarrier (TMA byte counts, tcgen05.commit or epilogue-warp arrivals), so
// the producer runs up to kStages tiles ahead of the MMA and the epilogue of tile j overlaps
// the MMA of tile j+1 — no CTA-wide barrier in the loop.
#ifndef STRATA_RGMS_PROD_WARPS  // A/B knob
#define STRATA_RGMS_PROD_WARPS 2
#endif
constexpr int kProdWarps = STRATA_RGMS_PROD_WARPS;  // warps 0 .. kProdWarps-1: producers
constexpr int kMmaWarp = kProdWarps;                // then the MMA issuer warp
#ifndef STRATA_RGMS_EPI_SETS  // A/B knob: epilogue warp sets (set e takes the tiles j = e mod sets)
#define STRATA_RGMS_EPI_SETS 1
#endif
constexpr int kEpiSets = STRATA_RGMS_EPI_SETS;
#ifndef STRATA_RGMS_CTAS  // A/B knob: cap on resident pass-1 CTAs per SM
#define STRATA_RGMS_CTAS 3
#endif
static_assert(kEpiSets == 1 || kEpiSets == 2, "one set per TMEM accumulator at most");
constexpr int kWsThreads = (kProdWarps + 1 + 4 * kEpiSets) * 32;  // then the epilogue warps
#ifndef STRATA_RGMS_WS_STAGES
#define STRATA_RGMS_WS_STAGES 4
#endif
constexpr int kStagesWs = STRATA_RGMS_WS_STAGES;
#ifndef STRATA_RGMS_EPI_PAD  // A/B knob: padded (1) or XOR-swizzled (0) epilogue transpose buffer
#define STRATA_RGMS_EPI_PAD 0  // (measured +1 % at C4: 0.347 vs 0.344 ms)
#endif
#ifndef STRATA_RGMS_EPI_NC  // A/B knob: accumulator columns per tcgen05.ld / epilogue pass
#define STRATA_RGMS_EPI_NC 32
#endif
constexpr int kIdxAheadWs = 3;
constexpr int kIdxSlotsWs = kIdxAheadWs + kStagesWs + 2;

template <int DIN, int DOUT>
struct RgmsWsSmem {
  static constexpr int kRowB = DIN * 2;              // A row bytes = swizzle width
  static constexpr int kABytes = kEdges * kRowB;
  static constexpr int kWBytes = DIN * DOUT * 2;
  static constexpr int kStage = kABytes + kWBytes;   // keeps every A region swizzle-atom aligned
  static constexpr int kIdxBytes = kTileWords * 4;   // 1552
  static constexpr int kNC = DOUT < STRATA_RGMS_EPI_NC ? DOUT : STRATA_RGMS_EPI_NC;  // epilogue column chunk
  // Epilogue transpose buffer per warp: 32 rows of kNC floats.  STRATA_RGMS_EPI_PAD: rows
  // padded by one float4 (conflict-free without the XOR swizzle, one IMAD per row address),
  // the pad column holding the warp's run table — the same bytes as swizzle + separate table.
  static constexpr int kRowF4 = kNC / 4 + (STRATA_RGMS_EPI_PAD ? 1 : 0);
  static constexpr int kEpiBytes = 4 * kEpiSets * 32 * kRowF4 * 16;
  static constexpr int kIdxOff = kStagesWs * kStage;
  static constexpr int kEpiOff = kIdxOff + kIdxSlotsWs * kIdxBytes;
  static constexpr int kRunOff = kEpiOff + kEpiBytes;        // per epilogue warp 32 int4 run records
  static constexpr int kBytes = kRunOff + (STRATA_RGMS_EPI_PAD ? 0 : 4 * kEpiSets * 32 * 16) + 1024;  // + alignment slack
  static constexpr int kAccCols = DOUT < 32 ? 32 : DOUT;
  static constexpr int kTmemCols = 2 * kAccCols <= 32 ? 32 : (2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : 256));
};

template <int DIN>
__device__ __forceinline__ uint64_t a_desc_kmajor(uint32_t saddr) {
  // K-major, swizzle width = one row (DIN * 2 bytes): 8-row atoms, SBO = 8 rows.
  if constexpr (DIN == 16) return tc::make_desc_sw32(saddr, 0, 8 * 32);
  else if constexpr (DIN == 32) return tc::make_desc_sw64(saddr, 0, 8 * 64);
  else return tc::make_desc_sw128(saddr, 0, 8 * 128);
}

template <int DIN, int DOUT>
__global__ void __launch_bounds__(kWsThreads, 1)
rgms_edge_gemm_kernel(const __grid_constant__ CUtensorMap wmap, const __nv_bfloat16* __restrict__ X,
                      const int32_t* __restrict__ ed, long long ntiles, float* __restrict__ T,
                      float* __restrict__ Y) {
  using SM = RgmsWsSmem<DIN, DOUT>;
  constexpr int kSboW = (DIN / 8) * 128;  // MN-major B (SWIZZLE_NONE): 8-column group stride
  constexpr uint32_t kIdesc = tc::make_idesc_bf16(kEdges, DOUT, /*A K-major*/ false, /*B MN-major*/ true);
  constexpr int kNC = SM::kNC;
  constexpr int kSPR = kNC / 4;    // float4 slots per row of a chunk
  static_assert(DIN == 16 || DIN == 32 || DIN == 64, "d_in");
  static_assert(DOUT % 16 == 0 && DOUT <= 128, "d_out");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[kStagesWs], empty[kStagesWs];
  __shared__ uint64_t idx_full[kIdxSlotsWs], idx_free[kIdxSlotsWs];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long G = gridDim.x;
  if (static_cast<long long>(blockIdx.x) >= ntiles) return;
  const long long nt = (ntiles - blockIdx.x + G - 1) / G;  // tiles of this CTA: b, b+G, ...

  if (warp == 0) tc::tmem_alloc<SM::kTmemCols>(&tmem_slot);
  if (threadIdx.x == 32 * kMmaWarp) {
    for (int i = 0; i < kStagesWs; ++i) {
      tc::mbar_init(&full[i], 32 * kProdWarps + 1);  // producer cp.async arrivals + W expect_tx
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kIdxSlotsWs; ++i) {
      tc::mbar_init(&idx_full[i], 1);
      tc::mbar_init(&idx_free[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 4);
    }
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  auto idx_slot = [&](long long j) {
    return reinterpret_cast<int32_t*>(smem + SM::kIdxOff + (j % kIdxSlotsWs) * SM::kIdxBytes);
  };

  if (warp < kProdWarps) {
    // ---------------- producers ----------------
    const int pt = threadIdx.x;  // 0 .. 32 * kProdWarps - 1
    if (pt == 0) tc::prefetch_tensormap(&wmap);
    auto issue_idx = [&](long long j) {  // thread 0
      const int k = static_cast<int>(j % kIdxSlotsWs);
      if (j >= kIdxSlotsWs) tc::mbar_wait(&idx_free[k], static_cast<uint32_t>((j / kIdxSlotsWs - 1) & 1));
      tc::mbar_arrive_expect_tx(&idx_full[k], SM::kIdxBytes);
      tc::bulk_copy_g2s(idx_slot(j), ed + (blockIdx.x + j * G) * kTileWords, SM::kIdxBytes, &idx_full[k]);
    };
    if (pt == 0)
      for (long long j = 0; j < kIdxAheadWs && j < nt; ++j) issue_idx(j);
    constexpr int kCpr = DIN / 8;                        // 16-byte chunks per X row
    constexpr int kPer = kEdges * kCpr / (32 * kProdWarps);
    constexpr int kSwzMask = SM::kRowB / 16 - 1;         // address bits [4:6] ^= bits [7:9]
    for (long long j = 0; j < nt; ++j) {
      if (pt == 0 && j + kIdxAheadWs < nt) issue_idx(j + kIdxAheadWs);
      const int s = static_cast<int>(j % kStagesWs);
      if (j >= kStagesWs) tc::mbar_wait(&empty[s], static_cast<uint32_t>((j / kStagesWs - 1) & 1));
      tc::mbar_wait(&idx_full[j % kIdxSlotsWs], static_cast<uint32_t>((j / kIdxSlotsWs) & 1));
      const int32_t* si = idx_slot(j);
      uint8_t* sA = smem + s * SM::kStage;
      uint8_t* sW = sA + SM::kABytes;
      if (pt == 0) {
        tc::mbar_arrive_expect_tx(&full[s], SM::kWBytes);
#pragma unroll
        for (int g = 0; g < DOUT / 8; ++g)  // W_r: one {8 columns x d_in rows} box per group
          tc::tma_load_2d(sW + g * kSboW, &wmap, g * 8, si[0] * DIN, &full[s]);
      }
      // X rows: 16-byte cp.async chunks written to their swizzled positions of the K-major
      // A operand; completion arrives on full[s] (cp.async.mbarrier.arrive.noinc).
      int32_t src[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) src[u] = si[4 + (pt + u * 32 * kProdWarps) / kCpr];
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int c = pt + u * 32 * kProdWarps;
        const int e = c / kCpr, kc = c % kCpr;
        const uint32_t o = e * SM::kRowB + kc * 16;
        tc::cp_async16(sA + (o ^ (((o >> 7) & kSwzMask) << 4)),
                       X + static_cast<long long>(src[u]) * DIN + kc * 8);
      }
      tc::cp_async_mbar_arrive_noinc(&full[s]);
    }
  } else if (warp == kMmaWarp) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      for (long long j = 0; j < nt; ++j) {
        const int s = static_cast<int>(j % kStagesWs);
        const int b = static_cast<int>(j & 1);
        tc::mbar_wait(&full[s], static_cast<uint32_t>((j / kStagesWs) & 1));
        if (j >= 2) tc::mbar_wait(&acc_empty[b], static_cast<uint32_t>((j / 2 - 1) & 1));
        tc::fence_proxy_async();  // cp.async (generic-proxy) writes -> tensor-core reads
        tc::fence_after_sync();
        const uint32_t a0 = tc::smem_u32(smem + s * SM::kStage);
        const uint32_t w0 = a0 + SM::kABytes;
#pragma unroll
        for (int kk = 0; kk < DIN / 16; ++kk)
          tc::mma_bf16(tmem + b * SM::kAccCols, a_desc_kmajor<DIN>(a0 + kk * 32),
                       tc::make_desc(w0 + kk * 256, 128, kSboW), kIdesc, kk > 0);
        tc::mma_commit(&empty[s]);
        tc::mma_commit(&acc_full[b]);
      }
    }
    __syncwarp();
  } else {
    // ---------------- epilogue (warps 3..: TMEM lanes 32 * (warp % 4) ..) ----------------
    // With two sets, set e owns accumulator e (tiles j = e mod 2): two tiles drain at once.
    const int q = warp & 3;
    const int ew = warp - kMmaWarp - 1;  // 0 .. 4 * kEpiSets - 1
    constexpr int kRow = SM::kRowF4;  // float4 per buffer row
    float4* epi = reinterpret_cast<float4*>(smem + SM::kEpiOff) + ew * (32 * kRow);
    // run table {r0, r1, T row, 0}: in the pad column of row k (padded), else its own array
    int4* runs = STRATA_RGMS_EPI_PAD ? reinterpret_cast<int4*>(epi + kSPR)
                                     : reinterpret_cast<int4*>(smem + SM::kRunOff) + ew * 32;
    constexpr int kRunStride = STRATA_RGMS_EPI_PAD ? kRow : 1;  // int4 between run records
    for (long long j = ew / 4; j < nt; j += kEpiSets) {
      const int b = static_cast<int>(j & 1);
      // The accumulator being published implies the producer saw this tile's index block land
      // (idx_full -> gathers -> full -> MMA -> commit), so the block is read only after it.
      tc::mbar_wait(&acc_full[b], static_cast<uint32_t>((j / 2) & 1));
      tc::fence_after_sync();
      const int32_t* si = idx_slot(j);
      const float a = __int_as_float(si[4 + 2 * kEdges + q * 32 + lane]);
      const int myword = si[4 + kEdges + q * 32 + lane];
      const bool is_head = myword >= 0 || myword <= -3;  // T row or direct Y row
      const unsigned heads = __ballot_sync(0xffffffffu, is_head);
      const unsigned pads = __ballot_sync(0xffffffffu, myword == -1);
      const int first_pad = pads ? __ffs(pads) - 1 : 32;
      const int nruns = __popc(heads);
      // Run table, once per tile: the head lane of the k-th run stores {r0, r1, T row} at k.
      if (is_head) {
        const unsigned later = heads & ~((2u << lane) - 1u);
        runs[__popc(heads & ((1u << lane) - 1u)) * kRunStride] =
            make_int4(lane, min(later ? __ffs(later) - 1 : 32, first_pad), myword, 0);
      }
#pragma unroll
      for (int c0 = 0; c0 < DOUT; c0 += kNC) {
        uint32_t v[kNC];
        tc::tmem_ld_32x32b<kNC>(tmem + b * SM::kAccCols + (static_cast<uint32_t>(q * 32) << 16) + c0, v);
        tc::tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < kSPR; ++u)
          epi[lane * kRow + (STRATA_RGMS_EPI_PAD ? u : (u ^ (lane & (kSPR - 1))))] =
              make_float4(a * __uint_as_float(v[4 * u]), a * __uint_as_float(v[4 * u + 1]),
                          a * __uint_as_float(v[4 * u + 2]), a * __uint_as_float(v[4 * u + 3]));
        __syncwarp();
        // (run, float4 column slot) items, kSPR per run, spread over the lanes: a run's rows
        // are summed in edge order, its slots leave as one contiguous kNC-float segment.
        for (int it = lane; it < nruns * kSPR; it += 32) {
          const int sl = it & (kSPR - 1);
          const int4 rn = runs[(it / kSPR) * kRunStride];
#if STRATA_RGMS_EPI_PAD
          const float4* er = epi + sl + rn.x * kRow;
          float4 acc = *er;
          for (int row = rn.x + 1; row < rn.y; ++row) acc = add4(acc, *(er += kRow));
#else
          float4 acc = epi[rn.x * kSPR + (sl ^ (rn.x & (kSPR - 1)))];
          for (int row = rn.x + 1; row < rn.y; ++row)
            acc = add4(acc, epi[row * kSPR + (sl ^ (row & (kSPR - 1)))]);
#endif
          if (rn.z >= 0) {
#if STRATA_RGMS_T_L2
            reinterpret_cast<float4*>(T + static_cast<long long>(rn.z) * DOUT + c0)[sl] = acc;
#else
            __stcs(reinterpret_cast<float4*>(T + static_cast<long long>(rn.z) * DOUT + c0) + sl, acc);
#endif
          } else {  // direct row: its only run is its sum (+0.f: the reference's 0 + x, no -0)
            acc.x += 0.f; acc.y += 0.f; acc.z += 0.f; acc.w += 0.f;
            __stcs(reinterpret_cast<float4*>(Y + static_cast<long long>(-3 - rn.z) * DOUT + c0) + sl, acc);
          }
        }
        __syncwarp();
      }
      tc::fence_before_sync();
      if (lane == 0) {
        tc::mbar_arrive(&acc_empty[b]);
        tc::mbar_arrive(&idx_free[j % kIdxSlotsWs]);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<SM::kTmemCols>(tmem);
}

// ---- pass 2: Y[i] = sum of T rows [dptr[i], dptr[i+1]) in order --------------------------
// A T row is read by kL lanes (float4 each, kF float4s per lane when DOUT > 128); kGrp = 32/kL
// lane groups per warp.  Rows longer than kLong edges (power-law hubs: at C4 2,973 rows hold
// 39 % of the edges, the longest 171,738) would serialise one lane group, so they are cut into
// kChunk-edge chunks summed by a whole warp (fixed strided split + fixed shuffle tree) into
// partials, and a finishing pass adds a row's partials in chunk order — deterministic.
#ifndef STRATA_RGMS_SUM_MINB  // A/B knobs of the row-sum pass
#define STRATA_RGMS_SUM_MINB 6
#endif
#ifndef STRATA_RGMS_SUM_KB
#define STRATA_RGMS_SUM_KB 4
#endif
#ifndef STRATA_RGMS_LONG
#define STRATA_RGMS_LONG 64
#endif
constexpr int kLong = STRATA_RGMS_LONG;
#ifndef STRATA_RGMS_SUM_WAVE  // A/B knob: cap on row-sum CTAs per SM in the grid
#define STRATA_RGMS_SUM_WAVE 32  // C4: 5 -> 0.380, 8 -> 0.375, 16 -> 0.367, 32 -> 0.365, 64 -> 0.373 ms
#endif
#ifndef STRATA_RGMS_CHUNK  // A/B knob: message rows per long-row chunk (128..1024 within 1 % at C4)
#define STRATA_RGMS_CHUNK 1024
#endif
constexpr int kChunk = STRATA_RGMS_CHUNK;
#ifndef STRATA_RGMS_COMPACT  // A/B knob: pass 2 walks the plan's compacted row list (1) or all rows (0)
#define STRATA_RGMS_COMPACT 1
#endif
#ifndef STRATA_RGMS_T_L2  // A/B knob: T rows written with the default L2 policy and dropped from L2
#define STRATA_RGMS_T_L2 0  // (discard.global.L2, no write-back) once pass 2 has summed them
#endif

// Pass 2 has consumed T row q: with STRATA_RGMS_T_L2 its 128-byte L2 lines are invalidated
// without write-back (the row is dead), one line per lane of the row's lane group.
template <int DOUT>
__device__ __forceinline__ void t_row_consumed(const float* T, long long q, int l) {
#if STRATA_RGMS_T_L2
  if constexpr ((DOUT * 4) % 128 == 0) {
    if (l < DOUT * 4 / 128)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(T + q * DOUT + l * 32) : "memory");
  }
#endif
}

template <int DOUT>
struct RowSumShape {
  static constexpr int kF4 = DOUT / 4;
  static constexpr int kL = kF4 < 32 ? kF4 : 32;
  static constexpr int kF = kF4 / kL;
  static constexpr int kGrp = 32 / kL;
};

// Short rows: a warp takes a block of 32 consecutive rows (bounds: one coalesced load, kept in
// smem); lane group g owns rows g*kRPV .. g*kRPV + kRPV - 1, whose T rows are contiguous, and
// walks that range in batches of 8 T rows issued together, flushing a row's sum when the walk
// crosses its end.  Long rows are stepped over (at most one wasted batch each).
// kCompact (the plan's compacted list of the rows pass 2 must write — rows with >= 2 runs and
// empty rows; the direct rows pass 1 wrote are absent): `m` is the list length, `dptr` the
// list's T-row pointer (cptr[j] = first T row of rowlist[j]) and Y row j is rowlist[j].
template <int DOUT, bool kCompact>
__device__ __forceinline__ void row_sum_body(const int32_t* __restrict__ dptr, const float* __restrict__ T,
                                             long long m, float* __restrict__ Y,
                                             const uint32_t* __restrict__ dbits,
                                             const int32_t* __restrict__ rowlist, long long blk,
                                             long long nblk) {
  using RS = RowSumShape<DOUT>;
  constexpr int kF4 = RS::kF4, kL = RS::kL, kF = RS::kF, kGrp = RS::kGrp;
  constexpr int kRPV = 32 / kGrp;  // rows per lane group per block
  constexpr int kB = STRATA_RGMS_SUM_KB;  // T rows in flight per lane group
  __shared__ int sbnd[8][33];
  __shared__ int srow[kCompact ? 8 : 1][32];
  const int lane = threadIdx.x & 31, l = lane % kL, g = lane / kL, w = threadIdx.x >> 5;
  int* bnd = sbnd[w];
  const long long nwarps = nblk * (blockDim.x >> 5);
  const float4* T4 = reinterpret_cast<const float4*>(T) + l;
  // The next block's bounds are loaded while this block's T rows stream (one DRAM latency
  // less on every block's dependency chain).
  long long b = blk * (blockDim.x >> 5) + w;
  int nb0 = 0, nb32 = 0, nrow = 0;
  uint32_t ndw = 0;  // direct rows of the block (written by pass 1, not here)
  if (b * 32 < m) {
    nb0 = __ldg(dptr + min64(b * 32 + lane, m));
    nb32 = __ldg(dptr + min64(b * 32 + 32, m));
    if constexpr (kCompact) nrow = __ldg(rowlist + min64(b * 32 + lane, m - 1));
    else ndw = __ldg(dbits + b);
  }
  for (; b * 32 < m; b += nwarps) {
    const long long i0 = b * 32;
    __syncwarp();
    bnd[lane] = nb0;
    if (lane == 0) bnd[32] = nb32;
    if constexpr (kCompact) srow[w][lane] = nrow;
    const uint32_t dw = ndw;
    __syncwarp();
    if ((b + nwarps) * 32 < m) {
      nb0 = __ldg(dptr + min64((b + nwarps) * 32 + lane, m));
      nb32 = __ldg(dptr + min64((b + nwarps) * 32 + 32, m));
      if constexpr (kCompact) nrow = __ldg(rowlist + min64((b + nwarps) * 32 + lane, m - 1));
      else ndw = __ldg(dbits + b + nwarps);
    }
    int r = g * kRPV;
    const int rend = static_cast<int>(min64(r + kRPV, m - i0));
    if (r >= rend) continue;
    int q = bnd[r], nb = bnd[r + 1];
    const int qend = bnd[rend];
    bool skip = nb - q > kLong;
    float4 acc[kF];
#pragma unroll
    for (int f = 0; f < kF; ++f) acc[f] = make_float4(0.f, 0.f, 0.f, 0.f);
    auto flush = [&] {
      if (!skip && (kCompact || !((dw >> r) & 1u))) {
        const long long yr = kCompact ? static_cast<long long>(srow[w][r]) : i0 + r;
#pragma unroll
        for (int f = 0; f < kF; ++f) {
          st_stream4(reinterpret_cast<float4*>(Y + yr * DOUT) + f * kL + l, acc[f]);
          acc[f] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      ++r;
      nb = r < rend ? bnd[r + 1] : qend;
      skip = r < rend && nb - bnd[r] > kLong;
    };
    while (q < qend) {
      if (skip) {  // long row: its T rows are summed by the chunk blocks (long_chunk_body)
        q = nb;
        flush();
        continue;
      }
      float4 u[kB][kF];
#pragma unroll
      for (int j = 0; j < kB; ++j)
#pragma unroll
        for (int f = 0; f < kF; ++f)
          u[j][f] = q + j < qend ? __ldcs(T4 + static_cast<long long>(q + j) * kF4 + f * kL)
                                 : make_float4(0.f, 0.f, 0.f, 0.f);
      int used = kB;
#pragma unroll
      for (int j = 0; j < kB; ++j) {
        if (used == kB) {
          const int qq = q + j;
          if (qq >= qend) {
            used = j;
          } else {
            while (qq >= nb) flush();
            if (skip) {
              used = j;  // qq starts a long row: the next round steps over it
            } else {
#pragma unroll
              for (int f = 0; f < kF; ++f) acc[f] = add4(acc[f], u[j][f]);
            }
          }
        }
      }
#if STRATA_RGMS_T_L2
#pragma unroll
      for (int j = 0; j < kB; ++j)
        if (j < used) t_row_consumed<DOUT>(T, q + j, l);
#endif
      q += used;
    }
    while (r < rend) flush();  // trailing rows (their sums, or zeros for empty rows)
  }
}

// Warp-wide fixed-order reduction of the kGrp lane groups' float4s (lane group 0 ends with it).
template <int kL>
__device__ __forceinline__ float4 reduce_groups(float4 v) {
#pragma unroll
  for (int off = 16; off >= kL; off >>= 1) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, off);
    v.y += __shfl_down_sync(0xffffffffu, v.y, off);
    v.z += __shfl_down_sync(0xffffffffu, v.z, off);
    v.w += __shfl_down_sync(0xffffffffu, v.w, off);
  }
  return v;
}

// One warp per chunk of a long row: partial[c] = sum of T rows [q0, q1).  Lane group g sums
// rows q0 + g, q0 + g + kGrp, ... (4 in flight), then the groups are combined.
template <int DOUT>
__device__ __forceinline__ void long_chunk_body(const int32_t* __restrict__ dptr,
                                                const int32_t* __restrict__ long_rows,
                                                const int32_t* __restrict__ chunk_off, int nlong,
                                                int nchunks, const float* __restrict__ T,
                                                float* __restrict__ partial, int blk, int nblk) {
  using RS = RowSumShape<DOUT>;
  constexpr int kF4 = RS::kF4, kL = RS::kL, kF = RS::kF, kGrp = RS::kGrp;
  const int lane = threadIdx.x & 31, l = lane % kL, grp = lane / kL;
  const int nwarps = nblk * (blockDim.x >> 5);
  for (int c = blk * (blockDim.x >> 5) + (threadIdx.x >> 5); c < nchunks; c += nwarps) {
    int lo = 0, hi = nlong;  // long row owning chunk c: last li with chunk_off[li] <= c
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(chunk_off + mid) <= c) lo = mid; else hi = mid;
    }
    const int row = __ldg(long_rows + lo);
    const int q0 = __ldg(dptr + row) + (c - __ldg(chunk_off + lo)) * kChunk;
    const int q1 = min(q0 + kChunk, __ldg(dptr + row + 1));
    float4 acc[kF];
#pragma unroll
    for (int g = 0; g < kF; ++g) acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    int q = q0 + grp;
    for (; q + 3 * kGrp < q1; q += 4 * kGrp) {
      float4 u[4][kF];
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int g = 0; g < kF; ++g)
          u[j][g] = __ldcs(reinterpret_cast<const float4*>(T) +
                           static_cast<long long>(q + j * kGrp) * kF4 + g * kL + l);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int g = 0; g < kF; ++g) acc[g] = add4(acc[g], u[j][g]);
#if STRATA_RGMS_T_L2
#pragma unroll
      for (int j = 0; j < 4; ++j) t_row_consumed<DOUT>(T, q + j * kGrp, l);
#endif
    }
    for (; q < q1; q += kGrp) {
#pragma unroll
      for (int g = 0; g < kF; ++g)
        acc[g] = add4(acc[g], __ldcs(reinterpret_cast<const float4*>(T) +
                                     static_cast<long long>(q) * kF4 + g * kL + l));
#if STRATA_RGMS_T_L2
      t_row_consumed<DOUT>(T, q, l);
#endif
    }
#pragma unroll
    for (int g = 0; g < kF; ++g) {
      const float4 v = reduce_groups<kL>(acc[g]);
      if (grp == 0) reinterpret_cast<float4*>(partial + static_cast<long long>(c) * DOUT)[g * kL + l] = v;
    }
  }
}

// Pass 2 in one launch: the first `cblk` blocks sum the long rows' chunks into partials (they
// are dispatched first, so the hub rows' T ranges stream concurrently with the short rows
// instead of after them), the remaining blocks run the short-row walk.
template <int DOUT, bool kCompact>
__global__ void __launch_bounds__(256, DOUT <= 32 ? STRATA_RGMS_SUM_MINB : 4)  // wider rows: more registers
rgms_row_sum_kernel(const int32_t* __restrict__ dptr, const float* __restrict__ T, long long m,
                    float* __restrict__ Y, const uint32_t* __restrict__ dbits,
                    const int32_t* __restrict__ long_rows,
                    const int32_t* __restrict__ chunk_off, int nlong, int nchunks,
                    float* __restrict__ partial, int cblk, const int32_t* __restrict__ cptr,
                    const int32_t* __restrict__ rowlist, long long nlist) {
  if (static_cast<int>(blockIdx.x) < cblk)
    long_chunk_body<DOUT>(dptr, long_rows, chunk_off, nlong, nchunks, T, partial, blockIdx.x, cblk);
  else if constexpr (kCompact)
    row_sum_body<DOUT, true>(cptr, T, nlist, Y, dbits, rowlist, blockIdx.x - cblk, gridDim.x - cblk);
  else
    row_sum_body<DOUT, false>(dptr, T, m, Y, dbits, nullptr, blockIdx.x - cblk, gridDim.x - cblk);
}

// One warp per long row: Y[row] = sum of its chunks' partials (same fixed split as above).
template <int DOUT>
__global__ void __launch_bounds__(256)
rgms_long_finish_kernel(const int32_t* __restrict__ long_rows, const int32_t* __restrict__ chunk_off,
                        int nlong, const float* __restrict__ partial, float* __restrict__ Y) {
  using RS = RowSumShape<DOUT>;
  constexpr int kF4 = RS::kF4, kL = RS::kL, kF = RS::kF, kGrp = RS::kGrp;
  const int lane = threadIdx.x & 31, l = lane % kL, grp = lane / kL;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  for (int li = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); li < nlong; li += nwarps) {
    const int c0 = __ldg(chunk_off + li), c1 = __ldg(chunk_off + li + 1);
    float4 acc[kF];
#pragma unroll
    for (int g = 0; g < kF; ++g) acc[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c = c0 + grp; c < c1; c += kGrp) {
#pragma unroll
      for (int g = 0; g < kF; ++g)
        acc[g] = add4(acc[g], reinterpret_cast<const float4*>(partial + static_cast<long long>(c) * DOUT)[g * kL + l]);
    }
    const long long row = __ldg(long_rows + li);
#pragma unroll
    for (int g = 0; g < kF; ++g) {
      const float4 v = reduce_groups<kL>(acc[g]);
      if (grp == 0) st_stream4(reinterpret_cast<float4*>(Y + row * DOUT) + g * kL + l, v);
    }
  }
}

// Plan helpers for the long rows.
__global__ void long_flags_kernel(const int32_t* __restrict__ dptr, long long m,
                                  uint8_t* __restrict__ flag, int32_t* __restrict__ nch) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int deg = dptr[i + 1] - dptr[i];
    flag[i] = deg > kLong;
    nch[i] = deg > kLong ? (deg + kChunk - 1) / kChunk : 0;
  }
}

__global__ void gather_i32_kernel(const int32_t* __restrict__ idx, const int32_t* __restrict__ v,
                                  int n, int32_t* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = v[idx[i]];
}

template <int DIN, int DOUT>
void launch_rgms(const strata_rgms& h, const __nv_bfloat16* X, const __nv_bfloat16* W, float* Y,
                 float* T, float* partial, cudaStream_t s) {
  using SM = RgmsWsSmem<DIN, DOUT>;
  constexpr int smem = SM::kBytes;
  auto* k1 = rgms_edge_gemm_kernel<DIN, DOUT>;
  static PerDeviceOnce once;
  once([&] {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  // Resident CTAs per SM: shared memory (~227 KB usable) and TMEM (512 columns) bound it.  (The
  // occupancy API reports 2 at C4's 74 KB; a grid of 3 per SM measured 0.398 vs 0.537 ms.)
  const int per_sm = std::max(1, std::min({STRATA_RGMS_CTAS, (227 * 1024) / (smem + 2048),
                                           512 / SM::kTmemCols}));
  const long long grid = std::min<long long>(h.ntiles, static_cast<long long>(num_sms()) * per_sm);
  const CUtensorMap wmap = make_tensor_map_bf16_2d(W, h.R * DIN, DOUT, 8, DIN, CU_TENSOR_MAP_SWIZZLE_NONE);
  k1<<<static_cast<unsigned>(std::max<long long>(grid, 1)), kWsThreads, smem, s>>>(wmap, X, h.edges.p,
                                                                                   h.ntiles, T, Y);
  STRATA_CUDA_CHECK(cudaGetLastError());
  const long long lanes = (STRATA_RGMS_COMPACT ? h.nlist : h.m) * RowSumShape<DOUT>::kL;
  // Grid: up to 32 CTAs per SM (~1.6 warp-blocks of 32 rows per warp at C4) — CTAs retire and
  // are replaced as their rows finish, which balances the power-law row lengths better than a
  // resident-only persistent grid (measured, knob above).
  const long long blocks = std::min<long long>((lanes + 255) / 256,
                                               static_cast<long long>(num_sms()) * STRATA_RGMS_SUM_WAVE);
  const int wpb = 8;
  const int cblk = h.nlong > 0 ? (h.nchunks + wpb - 1) / wpb : 0;
  rgms_row_sum_kernel<DOUT, STRATA_RGMS_COMPACT != 0><<<static_cast<unsigned>(std::max<long long>(blocks, 1) + cblk), 256, 0, s>>>(
      h.dptr.p, T, h.m, Y, h.dbits.p, h.long_rows.p, h.chunk_off.p, h.nlong, h.nchunks,
      partial, cblk, h.cptr.p, h.rowlist.p, h.nlist);
  if (h.nlong > 0) {
    rgms_long_finish_kernel<DOUT><<<static_cast<unsigned>((h.nlong + wpb - 1) / wpb), 32 * wpb, 0, s>>>(
        h.long_rows.p, h.chunk_off.p, h.nlong, partial, Y);
  }
  STRATA_CUDA_CHECK(cudaGetLastError());
}

void require_sm100() {
  int dev = 0, major = 0;
  STRATA_CUDA_CHECK(cudaGetDevice(&dev));
  STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a");
}

void check_dims(int64_t d_in, int64_t d_out) {
  switch (d_in * 1000 + d_out) {
    case 16016: case 16032: case 32016: case 32032: case 32064: case 64032: case 64064:
    case 32128: case 64128: return;
    default:
      throw ApiError(STRATA_ERR_USAGE,
                     "rgms_bf16: (d_in, d_out) must be in {16,32,64} x {16,32,64,128}");
  }
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return STRATA_OK;
  } catch (const ApiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return STRATA_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" int strata_rgms_plan(const int32_t* rel_ptr, const int32_t* dst, const int32_t* src,
                                const float* A, int64_t R, int64_t m, int64_t n, int64_t nnz,
                                strata_rgms** out, void* stream) {
  return guarded([&] {
    if (!out) throw ApiError(STRATA_ERR_USAGE, "null output handle");
    *out = nullptr;
    if (R < 1) throw ApiError(STRATA_ERR_USAGE, "RGMS requires at least one relation");  // kernels.cpp:139
    if (nnz > INT32_MAX || m >= INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "nnz exceeds int32");
    require_sm100();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto h = std::make_unique<strata_rgms>();
    STRATA_CUDA_CHECK(cudaGetDevice(&h->device));
    h->R = R; h->m = m; h->n = n; h->nnz = nnz;
    h->dptr.alloc(m + 1);
    const long long RR = R;
    const long long max_tiles = (nnz + kEdges - 1) / kEdges + R;  // upper bound on tiles
    long long* ntiles = static_cast<long long*>(workspace_alloc(sizeof(long long) * (R + 1), s));
    long long* tile_start = static_cast<long long*>(workspace_alloc(sizeof(long long) * (R + 1), s));
    int32_t* tile_rel = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * max_tiles, s));
    rel_tiles_kernel<<<static_cast<unsigned>((R + 1 + 255) / 256), 256, 0, s>>>(rel_ptr, R, ntiles);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, ntiles, tile_start, R + 1, s);
    void* tmp = workspace_alloc(tb, s);
    cub::DeviceScan::ExclusiveSum(tmp, tb, ntiles, tile_start, R + 1, s);
    tile_rel_kernel<<<static_cast<unsigned>(R), 256, 0, s>>>(tile_start, R, tile_rel);
    long long hnt = 0;
    STRATA_CUDA_CHECK(cudaMemcpyAsync(&hnt, tile_start + R, sizeof(hnt), cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    h->ntiles = hnt;
    if (nnz > 0) {
      // Runs: heads -> inclusive scan -> run ids; a stable radix sort of the runs by
      // destination gives each run its T row (a row's runs keep relation order) and dptr.
      int32_t* head = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * nnz * 2, s));
      int32_t* incl = head + nnz;
      const unsigned g = static_cast<unsigned>(std::min<long long>((nnz + 255) / 256, num_sms() * 16LL));
      const unsigned ge = static_cast<unsigned>(std::min<long long>((h->ntiles * kEdges + 255) / 256, num_sms() * 16LL));
      run_heads_kernel<<<ge, 256, 0, s>>>(rel_ptr, tile_start, tile_rel, h->ntiles, dst, head);
      size_t ib = 0;
      cub::DeviceScan::InclusiveSum(nullptr, ib, head, incl, nnz, s);
      void* itmp = workspace_alloc(ib, s);
      cub::DeviceScan::InclusiveSum(itmp, ib, head, incl, nnz, s);
      int32_t hr = 0;
      STRATA_CUDA_CHECK(cudaMemcpyAsync(&hr, incl + nnz - 1, sizeof(hr), cudaMemcpyDeviceToHost, s));
      STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
      const long long nr = hr;
      h->nruns = nr;
      int32_t* ids = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * nr * 5, s));
      int32_t* order = ids + nr;
      int32_t* keys = ids + 2 * nr;
      int32_t* run_pos = ids + 3 * nr;
      int32_t* run_dst = ids + 4 * nr;
      const unsigned gn = static_cast<unsigned>(std::min<long long>((nr + 255) / 256, num_sms() * 16LL));
      run_dst_kernel<<<g, 256, 0, s>>>(head, incl, dst, nnz, run_dst);
      iota_kernel<<<gn, 256, 0, s>>>(ids, nr);
      int bits = 1;
      while (bits < 31 && (1LL << bits) <= m) ++bits;
      size_t sb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, sb, run_dst, keys, ids, order, nr, 0, bits, s);
      void* stmp = workspace_alloc(sb, s);
      cub::DeviceRadixSort::SortPairs(stmp, sb, run_dst, keys, ids, order, nr, 0, bits, s);
      invert_kernel<<<gn, 256, 0, s>>>(order, nr, run_pos);
      const unsigned gr = static_cast<unsigned>(std::min<long long>((m + 1 + 255) / 256, num_sms() * 16LL));
      row_ptr_kernel<<<gr, 256, 0, s>>>(keys, nr, m, h->dptr.p);
      // Direct rows (exactly one run): bitmask, then T rows compacted over the other runs.
      h->dbits.alloc(static_cast<size_t>((m + 31) / 32) + 1);
      direct_bits_kernel<<<gr, 256, 0, s>>>(h->dptr.p, m, h->dbits.p);
      int32_t* dflag = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * (nr + 1) * 2, s));
      int32_t* dbefore = dflag + nr + 1;
      direct_flags_kernel<<<gn, 256, 0, s>>>(keys, nr, h->dptr.p, dflag);
      size_t db = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, db, dflag, dbefore, nr + 1, s);
      void* dtmp = workspace_alloc(db, s);
      cub::DeviceScan::ExclusiveSum(dtmp, db, dflag, dbefore, nr + 1, s);
      direct_pos_kernel<<<gn, 256, 0, s>>>(keys, dflag, dbefore, nr, run_pos);
      compact_dptr_kernel<<<gr, 256, 0, s>>>(dbefore, m, h->dptr.p);
      int32_t hd = 0;
      STRATA_CUDA_CHECK(cudaMemcpyAsync(&hd, dbefore + nr, sizeof(hd), cudaMemcpyDeviceToHost, s));
      STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
      h->trows = nr - hd;
      STRATA_CUDA_CHECK(cudaFreeAsync(dtmp, s));
      STRATA_CUDA_CHECK(cudaFreeAsync(dflag, s));
      h->edges.alloc(static_cast<size_t>(h->ntiles) * kTileWords);
      tile_edges_kernel<<<ge, 256, 0, s>>>(rel_ptr, RR, tile_start, tile_rel, h->ntiles, src, head,
                                           incl, run_pos, A, h->edges.p);
      STRATA_CUDA_CHECK(cudaFreeAsync(stmp, s));
      STRATA_CUDA_CHECK(cudaFreeAsync(ids, s));
      STRATA_CUDA_CHECK(cudaFreeAsync(itmp, s));
      STRATA_CUDA_CHECK(cudaFreeAsync(head, s));
      // Pass 2's work list (one host sync sizes it).
      if (m > 0) {
        uint8_t* flag = static_cast<uint8_t*>(workspace_alloc(m, s));
        int32_t* sel = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * (m + 1), s));
        int32_t* cnt = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t), s));
        const unsigned gm = static_cast<unsigned>(std::min<long long>((m + 255) / 256, num_sms() * 16LL));
        nondirect_flags_kernel<<<gm, 256, 0, s>>>(h->dbits.p, m, flag);
        cub::CountingInputIterator<int32_t> it(0);
        size_t fb = 0;
        cub::DeviceSelect::Flagged(nullptr, fb, it, flag, sel, cnt, m, s);
        void* ftmp = workspace_alloc(fb, s);
        cub::DeviceSelect::Flagged(ftmp, fb, it, flag, sel, cnt, m, s);
        int32_t hn = 0;
        STRATA_CUDA_CHECK(cudaMemcpyAsync(&hn, cnt, sizeof(hn), cudaMemcpyDeviceToHost, s));
        STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
        h->nlist = hn;
        h->rowlist.alloc(std::max<int32_t>(hn, 1));
        h->cptr.alloc(hn + 1);
        if (hn > 0)
          STRATA_CUDA_CHECK(cudaMemcpyAsync(h->rowlist.p, sel, sizeof(int32_t) * hn, cudaMemcpyDeviceToDevice, s));
        list_ptr_kernel<<<static_cast<unsigned>(std::min<long long>((hn + 256) / 256, num_sms() * 16LL)), 256, 0, s>>>(
            sel, h->dptr.p, hn, m, h->cptr.p);
        STRATA_CUDA_CHECK(cudaGetLastError());
        STRATA_CUDA_CHECK(cudaFreeAsync(ftmp, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(cnt, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(sel, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(flag, s));
      }
      // Long rows (> kLong edges) and their chunk offsets; one host sync sizes the partials.
      if (m > 0) {
        uint8_t* flag = static_cast<uint8_t*>(workspace_alloc(m, s));
        int32_t* nch = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * (m + 1), s));
        int32_t* sel = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * (m + 1), s));
        int32_t* cnt = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * 2, s));
        const unsigned gm = static_cast<unsigned>(std::min<long long>((m + 255) / 256, num_sms() * 16LL));
        long_flags_kernel<<<gm, 256, 0, s>>>(h->dptr.p, m, flag, nch);
        cub::CountingInputIterator<int32_t> it(0);
        size_t fb = 0, rb = 0;
        cub::DeviceSelect::Flagged(nullptr, fb, it, flag, sel, cnt, m, s);
        cub::DeviceReduce::Sum(nullptr, rb, nch, cnt + 1, m, s);
        void* ftmp = workspace_alloc(std::max(fb, rb), s);
        cub::DeviceSelect::Flagged(ftmp, fb, it, flag, sel, cnt, m, s);
        cub::DeviceReduce::Sum(ftmp, rb, nch, cnt + 1, m, s);
        int32_t hc[2] = {0, 0};
        STRATA_CUDA_CHECK(cudaMemcpyAsync(hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
        STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
        h->nlong = hc[0];
        h->nchunks = hc[1];
        if (h->nlong > 0) {
          h->long_rows.alloc(h->nlong);
          h->chunk_off.alloc(h->nlong + 1);
          STRATA_CUDA_CHECK(cudaMemcpyAsync(h->long_rows.p, sel, sizeof(int32_t) * h->nlong,
                                            cudaMemcpyDeviceToDevice, s));
          // chunk counts of the long rows, then their exclusive scan (+ total at [nlong])
          int32_t* lc = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * (h->nlong + 1), s));
          gather_i32_kernel<<<static_cast<unsigned>((h->nlong + 255) / 256), 256, 0, s>>>(
              sel, nch, h->nlong, lc);
          STRATA_CUDA_CHECK(cudaMemsetAsync(lc + h->nlong, 0, sizeof(int32_t), s));
          size_t eb = 0;
          cub::DeviceScan::ExclusiveSum(nullptr, eb, lc, h->chunk_off.p, h->nlong + 1, s);
          void* etmp = workspace_alloc(eb, s);
          cub::DeviceScan::ExclusiveSum(etmp, eb, lc, h->chunk_off.p, h->nlong + 1, s);
          STRATA_CUDA_CHECK(cudaFreeAsync(etmp, s));
          STRATA_CUDA_CHECK(cudaFreeAsync(lc, s));
        }
        STRATA_CUDA_CHECK(cudaFreeAsync(ftmp, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(cnt, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(sel, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(nch, s));
        STRATA_CUDA_CHECK(cudaFreeAsync(flag, s));
      }
    } else if (m >= 0) {
      STRATA_CUDA_CHECK(cudaMemsetAsync(h->dptr.p, 0, sizeof(int32_t) * (m + 1), s));
    }
    if (!h->dbits.p) {  // no runs: no direct rows
      h->dbits.alloc(static_cast<size_t>((m + 31) / 32) + 1);
      STRATA_CUDA_CHECK(cudaMemsetAsync(h->dbits.p, 0, sizeof(uint32_t) * ((m + 31) / 32 + 1), s));
    }
    STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(tile_rel, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(tile_start, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(ntiles, s));
    STRATA_CUDA_CHECK(cudaGetLastError());
    *out = h.release();
  });
}

extern "C" int strata_rgms_run_bf16(const strata_rgms* h, const void* X_bf16, const void* W_bf16,
                                    float* Y, int64_t d_in, int64_t d_out, void* stream) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null rgms plan");
    check_dims(d_in, d_out);
    require_sm100();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (h->nnz == 0) {
      if (h->m > 0) STRATA_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(float) * h->m * d_out, s));
      return;
    }
    const size_t need = static_cast<size_t>(std::max<int64_t>(h->trows, 1)) * d_out;
    const size_t pneed = static_cast<size_t>(h->nchunks) * d_out;
    // Per-run scratch from the stream-ordered pool (cached there), so a plan may be run on
    // several streams at once: message rows T, then the long rows' chunk partials.
    float* T = static_cast<float*>(workspace_alloc(sizeof(float) * (need + pneed), s));
    float* partial = T + need;
    const auto* X = static_cast<const __nv_bfloat16*>(X_bf16);
    const auto* W = static_cast<const __nv_bfloat16*>(W_bf16);
#define STRATA_RGMS_CASE(I, O) \
  case I * 1000 + O: launch_rgms<I, O>(*h, X, W, Y, T, partial, s); break;
    switch (d_in * 1000 + d_out) {
      STRATA_RGMS_CASE(16, 16) STRATA_RGMS_CASE(16, 32) STRATA_RGMS_CASE(32, 16)
      STRATA_RGMS_CASE(32, 32) STRATA_RGMS_CASE(32, 64) STRATA_RGMS_CASE(64, 32)
      STRATA_RGMS_CASE(64, 64) STRATA_RGMS_CASE(32, 128) STRATA_RGMS_CASE(64, 128)
    }
#undef STRATA_RGMS_CASE
    STRATA_CUDA_CHECK(cudaFreeAsync(T, s));
  });
}

extern "C" int strata_rgms_info(const strata_rgms* h, int64_t* tiles_bound, int64_t* t_bytes_per_dout) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null rgms plan");
    if (tiles_bound) *tiles_bound = h->ntiles;
    if (t_bytes_per_dout) *t_bytes_per_dout = h->trows * 4;  // T rows (direct rows excluded)
  });
}

extern "C" int strata_rgms_destroy(strata_rgms* h) {
  return guarded([&] {
    if (h) {
      DeviceGuard g(h->device);  // free on the plan's device, then restore the caller's
      delete h;
    }
  });
}

extern "C" int strata_rgms_bf16(const int32_t* rel_ptr, const int32_t* dst, const int32_t* src,
                                const float* A, int64_t R, int64_t m, int64_t n, int64_t nnz,
                                const void* X_bf16, const void* W_bf16, float* Y, int64_t d_in,
                                int64_t d_out, void* stream) {
  if (R >= 1) {  // dimension errors before any device work, like the reference's binding checks
    const int rc = guarded([&] { check_dims(d_in, d_out); });
    if (rc != STRATA_OK) return rc;
  }
  strata_rgms* h = nullptr;
  int rc = strata_rgms_plan(rel_ptr, dst, src, A, R, m, n, nnz, &h, stream);
  if (rc != STRATA_OK) return rc;
  rc = strata_rgms_run_bf16(h, X_bf16, W_bf16, Y, d_in, d_out, stream);
  if (rc == STRATA_OK) {  // the plan's buffers are freed synchronously: finish its work first
    rc = guarded([&] { STRATA_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
  }
  strata_rgms_destroy(h);
  return rc;
}
