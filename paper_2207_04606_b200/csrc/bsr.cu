// bsr.cu — device csr_to_bsr and the tcgen05 (UMMA) BSR SpMM.
//
// csr_to_bsr (storage.cpp:138-188): per block row the sorted unique block columns, then every
// CSR entry scattered into its b x b block (row-major inside the block).  Device version:
// block-column keys -> cub segmented sort per block row (a block row's entries are one
// contiguous CSR range) -> per-block-row unique count -> scan -> JO_indices -> scatter with a
// binary search of the block column, exactly like the reference's lower_bound.
//
// BSR SpMM (bsr_rule, transform.cpp:466-483; lowered nest in SURVEY Appendix B):
//   Y[(io*b+ii)*d + f] = sum_jo sum_ji A_bsr[jo][ii][ji] * X[(JO_idx[jo]*b + ji)*d + f]
// One CTA per block row.  Per block the tensor core computes the transposed product
//   D[f][ii] += sum_ji X[jb*b + ji][f] * A_blk[ii][ji]
// i.e. M = d (feature tile of 64 or 128), N = b = 32, K = b = 32 (two K=16 bf16 steps), with the
// X tile as the MN-major A operand (X rows are feature-contiguous, so no transpose is needed)
// and the block as the K-major B operand.  Accumulation over the block row stays in TMEM
// (f32).  A TMA producer thread streams blocks (bulk copy of a pre-arranged bf16 block) and
// X tiles (TMA tensor tiles) through a 6-stage full/empty mbarrier ring to a single MMA-issuer
// thread; tcgen05.commit recycles stages.  Epilogue: tcgen05.ld -> registers -> Y.
#include <cub/cub.cuh>
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <memory>
#include <cuda_bf16.h>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

using namespace strata_b200;


// DBSR (storage.cpp:336-370): the BSR of the same matrix plus its stored block rows.
struct strata_dbsr {
  strata_bsr* bsr = nullptr;
  int64_t nstored = 0;
  DevBuf<int32_t> stored;  // IO_indices [nstored]
  DevBuf<int32_t> jptr;    // JO_indptr [nstored + 1] over stored rows
  ~strata_dbsr() { delete bsr; }
};

namespace {

__global__ void block_keys_kernel(const int32_t* __restrict__ indices, long long nnz, int b,
                                  int32_t* __restrict__ keys) {
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
       q += static_cast<long long>(gridDim.x) * blockDim.x)
    keys[q] = indices[q] / b;
}

__global__ void seg_bounds_kernel(const int32_t* __restrict__ indptr, long long rows, int b,
                                  long long mb, int32_t* __restrict__ beg, int32_t* __restrict__ end) {
  const long long br = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (br >= mb) return;
  beg[br] = indptr[min64(br * b, rows)];
  end[br] = indptr[min64((br + 1) * b, rows)];
}

// Unique block columns of each block row (keys sorted within the row's segment).
template <bool kWrite>
__global__ void __launch_bounds__(256)
bsr_unique_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ beg,
                  const int32_t* __restrict__ end, long long* __restrict__ cnt,
                  const long long* __restrict__ off, int32_t* __restrict__ jo_indices) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long running;
  const long long br = blockIdx.x;
  const long long q0 = beg[br], q1 = end[br];
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  for (long long base = q0; base < q1; base += 256) {
    const long long q = base + threadIdx.x;
    const int is_new = q < q1 && (q == q0 || keys[q] != keys[q - 1]);
    int rank, total;
    Scan(tmp).ExclusiveSum(is_new, rank, total);
    if (kWrite && is_new) jo_indices[off[br] + running + rank] = keys[q];
    __syncthreads();
    if (threadIdx.x == 0) running += total;
    __syncthreads();
  }
  if (!kWrite && threadIdx.x == 0) cnt[br] = running;
}

// One warp per CSR row: place each entry in its block (storage.cpp:175-183).
__global__ void bsr_scatter_kernel(const int32_t* __restrict__ indptr,
                                   const int32_t* __restrict__ indices,
                                   const float* __restrict__ values, long long rows, int b,
                                   const int32_t* __restrict__ jo_indptr,
                                   const int32_t* __restrict__ jo_indices, float* __restrict__ bv,
                                   __nv_bfloat16* __restrict__ bvh) {
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  const long long br = i / b;
  const int lo0 = jo_indptr[br], hi0 = jo_indptr[br + 1];
  for (long long q = indptr[i] + lane; q < indptr[i + 1]; q += 32) {
    const int32_t j = indices[q];
    const int32_t bc = j / b;
    int lo = lo0, hi = hi0;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (jo_indices[mid] < bc) lo = mid + 1; else hi = mid;
    }
    const long long pos = static_cast<long long>(lo) * b * b + (i % b) * b + (j % b);
    bv[pos] = values[q];
    bvh[pos] = __float2bfloat16_rn(values[q]);  // tensor-core operand copy, same layout
  }
}

// ---- tensor-core SpMM ---------------------------------------------------------------------
#ifdef STRATA_BSR_TRACE  // development: per-CTA %globaltimer stamps (tools/ab_rgcn.py prints them)
__device__ unsigned long long g_bsr_trace[1024][8];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define BSR_TRACE(k) \
  do { if ((threadIdx.x & 31) == 0 && blockIdx.x < 1024) g_bsr_trace[blockIdx.x][k] = gtimer(); } while (0)
#else
#define BSR_TRACE(k) do {} while (0)
#endif
constexpr int kB = 32;        // block size served by the tensor-core path
// smem ring depth: 8 stages (48 KB at d = 64: 4 CTAs per SM for the multi-head grid; a
// 16-deep ring measured no faster on C3), bounded by ~200 KB of stages.
template <int D>
constexpr int bsr_stages() {
  constexpr int stage = 32 * 32 * 2 + 32 * D * 2;
  return (200 * 1024) / stage < 8 ? (200 * 1024) / stage : 8;
}
constexpr int kThreads = 128;
#ifndef STRATA_BSR_PDL  // A/B knob: programmatic dependent launch of the BSR SpMM
#define STRATA_BSR_PDL 1
#endif
constexpr int kMaxPre = 256;  // block-column indices of a block row preloaded into smem

// Warp-specialised, mbarrier-pipelined block-row SpMM:
//   warp 0 / lane 0  TMA producer: per block, one 2 KB bulk copy of the pre-arranged bf16 block
//                    (K-major B operand) + d/64 TMA tiles {64 features x 32 rows} of X with
//                    the 128-byte swizzle (MN-major SW128 A operand); completion is
//                    counted in bytes on full[s]; the slot is reused once empty[s] fires.
//   warp 1 / lane 0  MMA issuer: waits full[s], issues tcgen05.mma (M = feature tile, N = 32
//                    block rows, K = 2 x 16), tcgen05.commit -> empty[s]; final commit -> done.
//   all 4 warps      epilogue: tcgen05.ld of the TMEM accumulator -> Y rows.
template <int D>  // feature count, 64 or a multiple of 128 (<= 512)
__global__ void __launch_bounds__(kThreads, 1)
bsr_spmm_tc_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap xmap,
                   const int32_t* __restrict__ jo_indptr, const int32_t* __restrict__ jo_indices,
                   const int32_t* __restrict__ rowmap, long long nblocks, long long x_rows,
                   long long y_rows, float* __restrict__ Y) {
  constexpr int kM = D == 64 ? 64 : 128;         // UMMA M (feature tile)
  constexpr int kTiles = D / kM;                  // feature tiles
  constexpr int kCols = kTiles * kB < 32 ? 32 : kTiles * kB;  // TMEM columns (pow2 >= 32)
  constexpr int kAB = kB * kB * 2;                // block bytes (B operand)
  constexpr int kXB = kB * D * 2;                 // X tile bytes (A operand)
  constexpr int kStageB = kAB + kXB;
  constexpr int kStages = bsr_stages<D>();
  constexpr uint32_t kIdesc = tc::make_idesc_bf16(kM, kB, /*A MN-major*/ true, /*B K-major*/ false);
  static_assert(D == 64 || (D % 128 == 0 && D <= 512), "unsupported feature size");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SWIZZLE_128B atoms need 1024-byte alignment: round the dynamic base up (1 KB is reserved).
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t tmem_slot;
  __shared__ int32_t s_cols[kMaxPre];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // CTA = (stored block row, head); DBSR maps stored row -> block row (IO_indices).
  const long long sr = blockIdx.x, head = blockIdx.y;
  BSR_TRACE(0);
  // Prologue that touches no input (overlaps the previous kernel under PDL).
  if (warp == 0) tc::tmem_alloc<kCols>(&tmem_slot);
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    tc::mbar_fence_init();
  }
  if (tid == 64) {
    tc::prefetch_tensormap(&amap);
    tc::prefetch_tensormap(&xmap);
  }
  tc::pdl_wait();
  const long long br = rowmap ? rowmap[sr] : sr;
  const int q0 = jo_indptr[sr], nblk = jo_indptr[sr + 1] - q0;
  for (int j = tid; j < nblk && j < kMaxPre; j += kThreads) s_cols[j] = jo_indices[q0 + j];
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  tc::pdl_launch();
  const uint32_t tmem = tmem_slot;
  BSR_TRACE(1);

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kStages;
        if (j >= kStages) tc::mbar_wait(&empty[s], ((j / kStages) - 1) & 1);
        uint8_t* sa = smem + s * kStageB;
        tc::mbar_arrive_expect_tx(&full[s], kStageB);
        // block (head, q0 + j): rows of the [heads * nblocks * 32][32] value view, SW64
        tc::tma_load_2d(sa, &amap, 0, static_cast<int>((head * nblocks + q0 + j) * kB), &full[s]);
        const int col = j < kMaxPre ? s_cols[j] : jo_indices[q0 + j];
#pragma unroll
        for (int fa = 0; fa < D / 64; ++fa)  // one {64 features x 32 rows} box per 128-B atom
          tc::tma_load_2d(sa + kAB + fa * 4096, &xmap, fa * 64,
                          static_cast<int>(head * x_rows + col * kB), &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      for (int j = 0; j < nblk; ++j) {
        const int s = j % kStages;
        tc::mbar_wait(&full[s], (j / kStages) & 1);
        if (j == 0) BSR_TRACE(2);
        if (j == nblk - 1) BSR_TRACE(3);
        tc::fence_after_sync();
        const uint32_t sa = tc::smem_u32(smem + s * kStageB);
        const uint32_t sx = sa + kAB;
#pragma unroll
        for (int t = 0; t < kTiles; ++t) {
#pragma unroll
          for (int kk = 0; kk < kB / 16; ++kk) {
            // A = X tile, MN-major SWIZZLE_128B: 64-feature atoms 4 KB apart (LBO), 8-row K
            // groups 1 KB apart (SBO); K step kk starts 16 rows = 2 KB later.
            const uint64_t adesc = tc::make_desc_sw128(sx + t * (kM / 64) * 4096 + kk * 2048, 4096, 1024);
            // B = block, K-major SWIZZLE_64B (rows ii of 64 B, 8-row groups 512 B apart);
            // K step kk = 16 elements = 32 B inside the swizzled row.
            const uint64_t bdesc = tc::make_desc_sw64(sa + kk * 32, 0, 512);
            tc::mma_bf16(tmem + t * kB, adesc, bdesc, kIdesc, j > 0 || kk > 0);
          }
        }
        tc::mma_commit(&empty[s]);
      }
      if (nblk > 0) tc::mma_commit(&done);
    }
    __syncwarp();
  }

  float* yrow = Y + (head * y_rows + br * kB) * D;
  if (nblk > 0) {
    tc::mbar_wait(&done, 0);
    if (tid == 0) BSR_TRACE(4);
    tc::fence_after_sync();
#pragma unroll
    for (int t = 0; t < kTiles; ++t) {
      uint32_t r[32];
      tc::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + t * kB, r);
      tc::tmem_ld_wait();
      // M = 128: TMEM lane = feature row.  M = 64: rows 16w..16w+15 live in lanes 32w..32w+15.
      const int f = kM == 128 ? t * 128 + warp * 32 + lane : warp * 16 + lane;
      if (kM == 128 || lane < 16) {
#pragma unroll
        for (int ii = 0; ii < kB; ++ii) yrow[ii * D + f] = __uint_as_float(r[ii]);
      }
    }
  } else {
    for (int e = tid; e < kB * D; e += kThreads) yrow[e] = 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();
  BSR_TRACE(5);
  if (warp == 0) tc::tmem_dealloc<kCols>(tmem);
}

// X viewed as [heads * x_rows][D] bf16, box {64 features, 32 rows}, 128-byte swizzle: one box
// = one 4 KB column of MN-major SW128 atoms of the A operand.  Block values viewed as
// [heads * nblocks * 32][32] bf16 (row-major blocks), box {32, 32}, 64-byte swizzle: one box =
// the K-major SW64 B operand.
template <int D>
void launch_bsr(const strata_bsr& h, const __nv_bfloat16* vals, long long heads,
                const __nv_bfloat16* X, float* Y, cudaStream_t s, const int32_t* jo_indptr,
                const int32_t* rowmap, long long nrows) {
  constexpr int smem = bsr_stages<D>() * (kB * kB * 2 + kB * D * 2) + 1024;
  static PerDeviceOnce once;
  once([&] {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(bsr_spmm_tc_kernel<D>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  const long long x_rows = h.nb * kB, y_rows = h.mb * kB;
  const CUtensorMap xmap = make_tensor_map_bf16_2d(X, heads * x_rows, D, 64, kB, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap amap = make_tensor_map_bf16_2d(vals, heads * std::max<long long>(h.nblocks, 1) * kB,
                                                   kB, kB, kB, CU_TENSOR_MAP_SWIZZLE_64B);
  // Programmatic dependent launch: this grid's prologue may overlap the tail of the previous
  // kernel on the stream (the kernel waits on griddepcontrol before reading any input).
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nrows), static_cast<unsigned>(heads));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = STRATA_BSR_PDL;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  STRATA_CUDA_CHECK(cudaLaunchKernelEx(&cfg, bsr_spmm_tc_kernel<D>, amap, xmap, jo_indptr,
                                       static_cast<const int32_t*>(h.indices.p), rowmap,
                                       static_cast<long long>(h.nblocks), x_rows, y_rows, Y));
}

// rows of a stored-row view: stored[i] = block rows with >= 1 block, jptr = compressed indptr
__global__ void dbsr_rows_kernel(const int32_t* __restrict__ bp, long long mb,
                                 const long long* __restrict__ pos, int32_t* __restrict__ stored,
                                 int32_t* __restrict__ jptr) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < mb && bp[r + 1] > bp[r]) {
    stored[pos[r]] = static_cast<int32_t>(r);
    jptr[pos[r] + 1] = bp[r + 1];
  }
  if (r == 0) jptr[0] = 0;
}

__global__ void nonempty_kernel(const int32_t* __restrict__ bp, long long mb, long long* __restrict__ f) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < mb) f[r] = bp[r + 1] > bp[r] ? 1 : 0;
  if (r == mb) f[r] = 0;
}

void require_device_bsr() {
  int dev = 0, major = 0;
  STRATA_CUDA_CHECK(cudaGetDevice(&dev));
  STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a");
}

template <class F>
int guard_bsr(F&& f) {
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

extern "C" {

#ifdef STRATA_BSR_TRACE
int strata_debug_bsr_trace(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_bsr_trace, sizeof(g_bsr_trace)) == cudaSuccess ? 0 : 1;
}
#endif

int strata_bsr_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                        int64_t rows, int64_t cols, int64_t nnz, int64_t b, void* stream,
                        strata_bsr** out) {
  return guard_bsr([&] {
    if (b < 1) throw ApiError(STRATA_ERR_USAGE, "block size must be >= 1");  // storage.cpp:139
    if (!out) throw ApiError(STRATA_ERR_USAGE, "null output handle");
    if (nnz > INT32_MAX || rows >= INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "CSR exceeds int32");
    require_device_bsr();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto* h = new strata_bsr();
    try {
      STRATA_CUDA_CHECK(cudaGetDevice(&h->device));
      h->rows = rows; h->cols = cols; h->nnz = nnz; h->b = b;
      h->mb = (rows + b - 1) / b;
      h->nb = (cols + b - 1) / b;
      h->indptr.alloc(h->mb + 1);
      DevBuf<int32_t> keys(std::max<int64_t>(nnz, 1)), sorted(std::max<int64_t>(nnz, 1));
      DevBuf<int32_t> beg(std::max<int64_t>(h->mb, 1)), end(std::max<int64_t>(h->mb, 1));
      DevBuf<long long> cnt(h->mb + 1), off(h->mb + 1);
      STRATA_CUDA_CHECK(cudaMemsetAsync(cnt.p, 0, cnt.n * sizeof(long long), s));
      if (h->mb > 0) {
        seg_bounds_kernel<<<static_cast<unsigned>((h->mb + 255) / 256), 256, 0, s>>>(
            indptr, rows, static_cast<int>(b), h->mb, beg.p, end.p);
        if (nnz > 0) {
          block_keys_kernel<<<static_cast<unsigned>(std::min<int64_t>((nnz + 255) / 256, 8192)), 256, 0, s>>>(
              indices, nnz, static_cast<int>(b), keys.p);
          size_t tb = 0;
          cub::DeviceSegmentedSort::SortKeys(nullptr, tb, keys.p, sorted.p, nnz, h->mb, beg.p, end.p, s);
          DevBuf<unsigned char> tmp(tb);
          cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, keys.p, sorted.p, nnz, h->mb, beg.p, end.p, s);
          bsr_unique_kernel<false><<<static_cast<unsigned>(h->mb), 256, 0, s>>>(
              sorted.p, beg.p, end.p, cnt.p, nullptr, nullptr);
        }
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.p, off.p, h->mb + 1, s);
        DevBuf<unsigned char> tmp(tb);
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.p, off.p, h->mb + 1, s);
        STRATA_CUDA_CHECK(cudaGetLastError());
      }
      long long total = 0;
      if (h->mb > 0)
        STRATA_CUDA_CHECK(cudaMemcpyAsync(&total, off.p + h->mb, sizeof(long long),
                                          cudaMemcpyDeviceToHost, s));
      STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
      if (total * b * b > INT32_MAX * 16ll) throw ApiError(STRATA_ERR_CAPACITY, "BSR too large");
      h->nblocks = total;
      h->pad_slots = total * b * b - nnz;  // storage.cpp:186
      // JO_indptr as int32 (reference IntArray)
      std::vector<long long> hoff(h->mb + 1);
      if (h->mb > 0)
        STRATA_CUDA_CHECK(cudaMemcpy(hoff.data(), off.p, (h->mb + 1) * sizeof(long long),
                                     cudaMemcpyDeviceToHost));
      std::vector<int32_t> hptr(h->mb + 1, 0);
      for (int64_t i = 0; i <= h->mb; ++i) hptr[i] = static_cast<int32_t>(hoff[i]);
      STRATA_CUDA_CHECK(cudaMemcpy(h->indptr.p, hptr.data(), hptr.size() * sizeof(int32_t),
                                   cudaMemcpyHostToDevice));
      h->indices.alloc(total);
      h->values.alloc(total * b * b);
      h->vals_bf.alloc(total * b * b);
      if (total > 0) {
        STRATA_CUDA_CHECK(cudaMemsetAsync(h->values.p, 0, total * b * b * sizeof(float), s));
        STRATA_CUDA_CHECK(cudaMemsetAsync(h->vals_bf.p, 0, total * b * b * sizeof(__nv_bfloat16), s));
        bsr_unique_kernel<true><<<static_cast<unsigned>(h->mb), 256, 0, s>>>(
            sorted.p, beg.p, end.p, nullptr, off.p, h->indices.p);
        bsr_scatter_kernel<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, s>>>(
            indptr, indices, values, rows, static_cast<int>(b), h->indptr.p, h->indices.p,
            h->values.p, h->vals_bf.p);
        STRATA_CUDA_CHECK(cudaGetLastError());
      }
      STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int strata_bsr_info(const strata_bsr* h, int64_t* mb, int64_t* nb, int64_t* b, int64_t* nblocks,
                    int64_t* pad_slots) {
  return guard_bsr([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null bsr handle");
    if (mb) *mb = h->mb;
    if (nb) *nb = h->nb;
    if (b) *b = h->b;
    if (nblocks) *nblocks = h->nblocks;
    if (pad_slots) *pad_slots = h->pad_slots;
  });
}

int strata_bsr_read(const strata_bsr* h, int32_t* jo_indptr, int32_t* jo_indices, float* values) {
  return guard_bsr([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null bsr handle");
    if (jo_indptr)
      STRATA_CUDA_CHECK(cudaMemcpy(jo_indptr, h->indptr.p, (h->mb + 1) * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost));
    if (jo_indices && h->nblocks)
      STRATA_CUDA_CHECK(cudaMemcpy(jo_indices, h->indices.p, h->nblocks * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost));
    if (values && h->nblocks)
      STRATA_CUDA_CHECK(cudaMemcpy(values, h->values.p, h->nblocks * h->b * h->b * sizeof(float),
                                   cudaMemcpyDeviceToHost));
  });
}

int strata_bsr_destroy(strata_bsr* h) {
  delete h;
  return STRATA_OK;
}

int strata_bsr_spmm_bf16_batched(const strata_bsr* h, const void* values_bf16, const void* X_bf16,
                                 float* Y, int64_t heads, int64_t d, void* stream) {
  return guard_bsr([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null bsr handle");
    if (h->b != kB) throw ApiError(STRATA_ERR_USAGE, "bsr_spmm_bf16: tensor-core path needs b == 32");
    if (heads < 1 || heads > 65535) throw ApiError(STRATA_ERR_USAGE, "bsr_spmm_bf16: heads must be in [1, 65535]");
    if (d != 64 && d != 128 && d != 256 && d != 512)
      throw ApiError(STRATA_ERR_USAGE, "bsr_spmm_bf16: d must be 64, 128, 256 or 512");
    if (!values_bf16 && heads > 1)
      throw ApiError(STRATA_ERR_USAGE, "bsr_spmm_bf16: per-head values are required when heads > 1");
    if (h->mb == 0) return;
    require_device_bsr();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const auto* X = static_cast<const __nv_bfloat16*>(X_bf16);
    const auto* V = values_bf16 ? static_cast<const __nv_bfloat16*>(values_bf16) : h->vals_bf.p;
    if (h->nblocks == 0) {  // no stored block: Y = 0 (interp.cpp:584-587)
      STRATA_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(float) * heads * h->mb * kB * d, s));
      return;
    }
    switch (d) {
      case 64: launch_bsr<64>(*h, V, heads, X, Y, s, h->indptr.p, nullptr, h->mb); break;
      case 128: launch_bsr<128>(*h, V, heads, X, Y, s, h->indptr.p, nullptr, h->mb); break;
      case 256: launch_bsr<256>(*h, V, heads, X, Y, s, h->indptr.p, nullptr, h->mb); break;
      case 512: launch_bsr<512>(*h, V, heads, X, Y, s, h->indptr.p, nullptr, h->mb); break;
    }
  });
}

int strata_bsr_spmm_bf16(const strata_bsr* h, const void* X_bf16, float* Y, int64_t d,
                         void* stream) {
  return strata_bsr_spmm_bf16_batched(h, nullptr, X_bf16, Y, 1, d, stream);
}

int strata_dbsr_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                         int64_t rows, int64_t cols, int64_t nnz, int64_t b, void* stream,
                         strata_dbsr** out) {
  return guard_bsr([&] {
    if (!out) throw ApiError(STRATA_ERR_USAGE, "null output handle");
    *out = nullptr;
    strata_bsr* bsr = nullptr;
    const int rc = strata_bsr_from_csr(indptr, indices, values, rows, cols, nnz, b, stream, &bsr);
    if (rc != STRATA_OK) throw ApiError(rc, strata_last_error());
    auto h = std::make_unique<strata_dbsr>();
    h->bsr = bsr;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const long long mb = bsr->mb;
    DevBuf<long long> flag(mb + 1), pos(mb + 1);
    const unsigned g = static_cast<unsigned>((mb + 1 + 255) / 256);
    nonempty_kernel<<<g, 256, 0, s>>>(bsr->indptr.p, mb, flag.p);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, flag.p, pos.p, mb + 1, s);
    DevBuf<unsigned char> tmp(tb);
    cub::DeviceScan::ExclusiveSum(tmp.p, tb, flag.p, pos.p, mb + 1, s);
    long long ns = 0;
    STRATA_CUDA_CHECK(cudaMemcpyAsync(&ns, pos.p + mb, sizeof(ns), cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    h->nstored = ns;
    h->stored.alloc(std::max<long long>(ns, 1));
    h->jptr.alloc(ns + 1);
    dbsr_rows_kernel<<<g, 256, 0, s>>>(bsr->indptr.p, mb, pos.p, h->stored.p, h->jptr.p);
    STRATA_CUDA_CHECK(cudaGetLastError());
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    *out = h.release();
  });
}

int strata_dbsr_info(const strata_dbsr* h, int64_t* mb, int64_t* nb, int64_t* b, int64_t* nstored,
                     int64_t* nblocks, int64_t* pad_slots) {
  return guard_bsr([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null dbsr handle");
    if (nstored) *nstored = h->nstored;
    const int rc = strata_bsr_info(h->bsr, mb, nb, b, nblocks, pad_slots);
    if (rc != STRATA_OK) throw ApiError(rc, strata_last_error());
  });
}

int strata_dbsr_read(const strata_dbsr* h, int32_t* io_indices, int32_t* jo_indptr,
                     int32_t* jo_indices, float* values) {
  return guard_bsr([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null dbsr handle");
    if (io_indices && h->nstored)
      STRATA_CUDA_CHECK(cudaMemcpy(io_indices, h->stored.p, h->nstored * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost));
    if (jo_indptr)
      STRATA_CUDA_CHECK(cudaMemcpy(jo_indptr, h->jptr.p, (h->nstored + 1) * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost));
    const int rc = strata_bsr_read(h->bsr, nullptr, jo_indices, values);  // same block order
    if (rc != STRATA_OK) throw ApiError(rc, strata_last_error());
  });
}

int strata_dbsr_destroy(strata_dbsr* h) {
  delete h;
  return STRATA_OK;
}

int strata_dbsr_spmm_bf16(const strata_dbsr* h, const void* X_bf16, float* Y, int64_t d,
                          void* stream) {
  return guard_bsr([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null dbsr handle");
    const strata_bsr* b = h->bsr;
    if (b->b != kB) throw ApiError(STRATA_ERR_USAGE, "bsr_spmm_bf16: tensor-core path needs b == 32");
    if (d != 64 && d != 128 && d != 256 && d != 512)
      throw ApiError(STRATA_ERR_USAGE, "bsr_spmm_bf16: d must be 64, 128, 256 or 512");
    if (b->mb == 0) return;
    require_device_bsr();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Block rows that DBSR does not store are zero (interp.cpp:584-587).
    if (h->nstored < b->mb) STRATA_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(float) * b->mb * kB * d, s));
    if (h->nstored == 0) return;
    const auto* X = static_cast<const __nv_bfloat16*>(X_bf16);
    switch (d) {
      case 64: launch_bsr<64>(*b, b->vals_bf.p, 1, X, Y, s, h->jptr.p, h->stored.p, h->nstored); break;
      case 128: launch_bsr<128>(*b, b->vals_bf.p, 1, X, Y, s, h->jptr.p, h->stored.p, h->nstored); break;
      case 256: launch_bsr<256>(*b, b->vals_bf.p, 1, X, Y, s, h->jptr.p, h->stored.p, h->nstored); break;
      case 512: launch_bsr<512>(*b, b->vals_bf.p, 1, X, Y, s, h->jptr.p, h->stored.p, h->nstored); break;
    }
  });
}

}  // extern "C"
