// srbcrs.cu — SR-BCRS(t, g) on the device: csr_to_srbcrs (storage.cpp:372-440) and its SpMM
// on tcgen05 tensor cores (SparseTIR's pruned-weight format).
//
// Format (reference): tile rows of t CSR rows; per tile row the distinct columns of its
// non-zeros, sorted, cut into groups of g (the last group padded with the last column);
// G_indptr[mb+1] (groups per tile row, prefix), JT_indices[groups*g], values
// [groups*g][t] (slot-major: for each column slot the t rows' values, zero where absent).
// Device build: per-tile-row segmented sort of the column indices -> unique count -> groups ->
// scan -> JT fill (pads = last column) -> one warp per CSR row scatters its values by binary
// search over the tile row's unique columns, exactly like the reference's lower_bound.
//
// SpMM (t = 8, g = 32): one CTA per tile row; per group the tensor core computes
//   D[f][e] += sum_slot X[JT[slot]][f] * A[e][slot]   M = d tile (64 / 128), N = 8 (16 when
// M = 128: zero-padded), K = 32.  The 32 gathered X rows arrive by TMA tile::gather4 (4 rows per
// op) into the MN-major SW128 A operand; the group's 32 x 8 bf16 values are already the MN-major
// SWIZZLE_NONE B operand ([slot][e], 16-byte rows) and arrive by one bulk copy.  Producer /
// MMA-issuer / epilogue hand-offs through a full/empty mbarrier ring, accumulator in TMEM.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <vector>
#include <cuda_bf16.h>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

using namespace strata_b200;

struct strata_srbcrs {
  int device = 0;
  int64_t rows = 0, cols = 0, nnz = 0, t = 1, g = 1, mb = 0, groups = 0, pad_slots = 0;
  DevBuf<int32_t> gptr;            // G_indptr [mb + 1]
  DevBuf<int32_t> jt;              // JT_indices [groups * g]
  DevBuf<float> values;            // [groups * g * t] f32 (readback)
  DevBuf<__nv_bfloat16> vals_bf;   // tensor-core operand, same layout
};

namespace {

__global__ void tile_bounds_kernel(const int32_t* __restrict__ indptr, long long rows, int t,
                                   long long mb, int32_t* __restrict__ beg, int32_t* __restrict__ end) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= mb) return;
  beg[r] = indptr[min64(r * t, rows)];
  end[r] = indptr[min64((r + 1) * t, rows)];
}

// Unique sorted columns of each tile row: count (pass 1) or write them (pass 2) and pad the
// last group with the last column (storage.cpp:411-420).
template <bool kWrite>
__global__ void __launch_bounds__(256)
srbcrs_unique_kernel(const int32_t* __restrict__ keys, const int32_t* __restrict__ beg,
                     const int32_t* __restrict__ end, int g, long long* __restrict__ ucnt,
                     const long long* __restrict__ goff, int32_t* __restrict__ jt) {
  using Scan = cub::BlockScan<int, 256>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ long long running;
  __shared__ int32_t last;
  const long long r = blockIdx.x;
  const long long q0 = beg[r], q1 = end[r];
  if (threadIdx.x == 0) running = 0;
  __syncthreads();
  for (long long base = q0; base < q1; base += 256) {
    const long long q = base + threadIdx.x;
    const int is_new = q < q1 && (q == q0 || keys[q] != keys[q - 1]);
    int rank, total;
    Scan(tmp).ExclusiveSum(is_new, rank, total);
    if (kWrite && is_new) jt[goff[r] * g + running + rank] = keys[q];
    __syncthreads();
    if (threadIdx.x == 0) running += total;
    __syncthreads();
  }
  if (!kWrite) {
    if (threadIdx.x == 0) ucnt[r] = running;
    return;
  }
  if (threadIdx.x == 0) last = q1 > q0 ? keys[q1 - 1] : 0;
  __syncthreads();
  const long long slots = (goff[r + 1] - goff[r]) * g;
  for (long long k = running + threadIdx.x; k < slots; k += blockDim.x) jt[goff[r] * g + k] = last;
}

__global__ void groups_kernel(const long long* __restrict__ ucnt, long long mb, int g,
                              long long* __restrict__ ng) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < mb) ng[r] = (ucnt[r] + g - 1) / g;
  if (r == mb) ng[r] = 0;
}

__global__ void to_i32_kernel(const long long* __restrict__ a, long long n, int32_t* __restrict__ b) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) b[i] = static_cast<int32_t>(a[i]);
}

// One warp per CSR row: value (i, col) -> slot of col among the tile row's unique columns.
__global__ void srbcrs_scatter_kernel(const int32_t* __restrict__ indptr,
                                      const int32_t* __restrict__ indices,
                                      const float* __restrict__ values, long long rows, int t, int g,
                                      const long long* __restrict__ goff,
                                      const long long* __restrict__ ucnt,
                                      const int32_t* __restrict__ jt, float* __restrict__ v,
                                      __nv_bfloat16* __restrict__ vh) {
  const long long i = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (i >= rows) return;
  const long long r = i / t;
  const long long base = goff[r] * g;
  const int u = static_cast<int>(ucnt[r]);
  for (long long q = indptr[i] + lane; q < indptr[i + 1]; q += 32) {
    const int32_t col = indices[q];
    int lo = 0, hi = u;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (jt[base + mid] < col) lo = mid + 1; else hi = mid;
    }
    const long long flat = (base + lo) * t + (i % t);
    v[flat] = values[q];
    vh[flat] = __float2bfloat16_rn(values[q]);
  }
}

// ---- tensor-core SpMM (t = 8, g = 32) ---------------------------------------------------------
constexpr int kT = 8, kG = 32, kThreads = 128, kStages = 6;

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
srbcrs_spmm_tc_kernel(const __grid_constant__ CUtensorMap xmap, const int32_t* __restrict__ gptr,
                      const int32_t* __restrict__ jt, const __nv_bfloat16* __restrict__ vals,
                      long long rows, float* __restrict__ Y) {
  constexpr int kM = D == 64 ? 64 : 128;   // UMMA M (feature tile)
  constexpr int kN = kM == 64 ? 8 : 16;     // UMMA N: t = 8, zero-padded to 16 when M = 128
  constexpr int kTiles = D / kM;
  constexpr int kCols = kTiles * kN <= 32 ? 32 : 64;
  constexpr int kXB = kG * D * 2;           // gathered X rows (A operand), SW128 atoms
  constexpr int kVB = kG * kT * 2;          // one group's values (B operand), 512 B
  constexpr int kBB = kG * kN * 2;          // B operand incl. zero padding
  constexpr int kStageB = kXB + kBB;
  constexpr uint32_t kIdesc = tc::make_idesc_bf16(kM, kN, /*A MN-major*/ true, /*B MN-major*/ true);
  static_assert(D == 64 || (D % 128 == 0 && D <= 512), "unsupported feature size");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t tmem_slot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long r = blockIdx.x;
  const int q0 = gptr[r], ng = gptr[r + 1] - q0;
  if (warp == 0) tc::tmem_alloc<kCols>(&tmem_slot);
  if (tid == 32) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    tc::mbar_fence_init();
  }
  if (kN > kT)  // zero padding columns of every stage's B operand (written once)
    for (int s = 0; s < kStages; ++s)
      for (int i = tid; i < (kBB - kVB) / 16; i += kThreads)
        reinterpret_cast<int4*>(smem + s * kStageB + kXB + kVB)[i] = make_int4(0, 0, 0, 0);
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    // producer (whole warp): lane 0 arms the stage, lanes issue the row gathers
    if (lane == 0) tc::prefetch_tensormap(&xmap);
    for (int j = 0; j < ng; ++j) {
      const int s = j % kStages;
      if (j >= kStages) tc::mbar_wait(&empty[s], ((j / kStages) - 1) & 1);
      uint8_t* sx = smem + s * kStageB;
      if (lane == 0) {
        tc::mbar_arrive_expect_tx(&full[s], kXB + kVB);
        tc::bulk_copy_g2s(sx + kXB, vals + static_cast<long long>(q0 + j) * kG * kT, kVB, &full[s]);
      }
      __syncwarp();
      // 32 rows x (D / 64) atoms, 4 rows per gather4: lane l -> (atom l / 8, rows 4 (l % 8) ..)
      for (int op = lane; op < (kG / 4) * (D / 64); op += 32) {
        const int fa = op / (kG / 4), q = op % (kG / 4);
        const int4 rr = *reinterpret_cast<const int4*>(jt + static_cast<long long>(q0 + j) * kG + 4 * q);
        tc::tma_gather4(sx + fa * (kG * 128) + q * 4 * 128, &xmap, fa * 64, rr.x, rr.y, rr.z, rr.w,
                        &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      for (int j = 0; j < ng; ++j) {
        const int s = j % kStages;
        tc::mbar_wait(&full[s], (j / kStages) & 1);
        tc::fence_after_sync();
        const uint32_t sx = tc::smem_u32(smem + s * kStageB);
        const uint32_t sv = sx + kXB;
#pragma unroll
        for (int tt = 0; tt < kTiles; ++tt) {
#pragma unroll
          for (int kk = 0; kk < kG / 16; ++kk) {
            // A: X rows, MN-major SW128 (64-feature atoms of 32 rows = 4 KB, 8-row groups 1 KB);
            // B: values [slot][e], MN-major SWIZZLE_NONE (LBO 128 B, SBO 512 B to the padding).
            const uint64_t adesc = tc::make_desc_sw128(sx + tt * (kM / 64) * (kG * 128) + kk * 2048, kG * 128, 1024);
            const uint64_t bdesc = tc::make_desc(sv + kk * 256, 128, kVB);
            tc::mma_bf16(tmem + tt * kN, adesc, bdesc, kIdesc, j > 0 || kk > 0);
          }
        }
        tc::mma_commit(&empty[s]);
      }
      if (ng > 0) tc::mma_commit(&done);
    }
    __syncwarp();
  }

  // epilogue: D[f][e] -> Y[r * t + e][f]
  const long long row0 = r * kT;
  if (ng > 0) {
    tc::mbar_wait(&done, 0);
    tc::fence_after_sync();
#pragma unroll
    for (int tt = 0; tt < kTiles; ++tt) {
      uint32_t v[8];
      tc::tmem_ld_32x32b_x8(tmem + (static_cast<uint32_t>(warp * 32) << 16) + tt * kN, v);
      tc::tmem_ld_wait();
      const int f = kM == 128 ? tt * 128 + warp * 32 + lane : warp * 16 + lane;
      if (kM == 128 || lane < 16) {
#pragma unroll
        for (int e = 0; e < kT; ++e) Y[(row0 + e) * D + f] = __uint_as_float(v[e]);
      }
    }
  } else {
    for (int i = tid; i < kT * D; i += kThreads) Y[row0 * D + i] = 0.f;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kCols>(tmem);
}

template <int D>
void launch_srbcrs(const strata_srbcrs& h, const __nv_bfloat16* X, float* Y, cudaStream_t s) {
  constexpr int kM = D == 64 ? 64 : 128;
  constexpr int kN = kM == 64 ? 8 : 16;
  constexpr int smem = kStages * (kG * D * 2 + kG * kN * 2) + 1024;
  static PerDeviceOnce once;
  once([&] {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(srbcrs_spmm_tc_kernel<D>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  const CUtensorMap xmap = make_tensor_map_bf16_2d(X, h.cols, D, 64, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  srbcrs_spmm_tc_kernel<D><<<static_cast<unsigned>(h.mb), kThreads, smem, s>>>(
      xmap, h.gptr.p, h.jt.p, h.vals_bf.p, h.rows, Y);
  STRATA_CUDA_CHECK(cudaGetLastError());
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

void require_sm100_srbcrs() {
  int dev = 0, major = 0;
  STRATA_CUDA_CHECK(cudaGetDevice(&dev));
  STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a");
}

}  // namespace

extern "C" {

int strata_srbcrs_from_csr(const int32_t* indptr, const int32_t* indices, const float* values,
                           int64_t rows, int64_t cols, int64_t nnz, int64_t t, int64_t g,
                           void* stream, strata_srbcrs** out) {
  return guarded([&] {
    if (!out) throw ApiError(STRATA_ERR_USAGE, "null output handle");
    *out = nullptr;
    if (t < 1 || g < 1) throw ApiError(STRATA_ERR_USAGE, "SR-BCRS requires t >= 1 and g >= 1");  // storage.cpp:374
    if (nnz > INT32_MAX || rows >= INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "CSR exceeds int32");
    require_sm100_srbcrs();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto h = std::make_unique<strata_srbcrs>();
    STRATA_CUDA_CHECK(cudaGetDevice(&h->device));
    h->rows = rows; h->cols = cols; h->nnz = nnz; h->t = t; h->g = g;
    h->mb = (rows + t - 1) / t;
    const long long mb = h->mb;
    h->gptr.alloc(mb + 1);
    DevBuf<int32_t> sorted(std::max<int64_t>(nnz, 1));
    DevBuf<int32_t> beg(std::max<long long>(mb, 1)), end(std::max<long long>(mb, 1));
    DevBuf<long long> ucnt(mb + 1), ng(mb + 1), goff(mb + 1);
    STRATA_CUDA_CHECK(cudaMemsetAsync(ucnt.p, 0, ucnt.n * sizeof(long long), s));
    const unsigned gm = static_cast<unsigned>((mb + 1 + 255) / 256);
    if (mb > 0) {
      tile_bounds_kernel<<<gm, 256, 0, s>>>(indptr, rows, static_cast<int>(t), mb, beg.p, end.p);
      if (nnz > 0) {
        size_t tb = 0;
        cub::DeviceSegmentedSort::SortKeys(nullptr, tb, indices, sorted.p, nnz, mb, beg.p, end.p, s);
        DevBuf<unsigned char> tmp(tb);
        cub::DeviceSegmentedSort::SortKeys(tmp.p, tb, indices, sorted.p, nnz, mb, beg.p, end.p, s);
        srbcrs_unique_kernel<false><<<static_cast<unsigned>(mb), 256, 0, s>>>(
            sorted.p, beg.p, end.p, static_cast<int>(g), ucnt.p, nullptr, nullptr);
      }
    }
    groups_kernel<<<gm, 256, 0, s>>>(ucnt.p, mb, static_cast<int>(g), ng.p);
    size_t sb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, sb, ng.p, goff.p, mb + 1, s);
    DevBuf<unsigned char> stmp(sb);
    cub::DeviceScan::ExclusiveSum(stmp.p, sb, ng.p, goff.p, mb + 1, s);
    to_i32_kernel<<<gm, 256, 0, s>>>(goff.p, mb + 1, h->gptr.p);
    long long total = 0;
    STRATA_CUDA_CHECK(cudaMemcpyAsync(&total, goff.p + mb, sizeof(total), cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    if (total * g * t > INT32_MAX * 16ll) throw ApiError(STRATA_ERR_CAPACITY, "SR-BCRS too large");
    h->groups = total;
    h->pad_slots = total * g * t - nnz;  // storage.cpp:438
    h->jt.alloc(std::max<long long>(total * g, 1));
    h->values.alloc(std::max<long long>(total * g * t, 1));
    h->vals_bf.alloc(std::max<long long>(total * g * t, 1));
    if (total > 0) {
      STRATA_CUDA_CHECK(cudaMemsetAsync(h->values.p, 0, total * g * t * sizeof(float), s));
      STRATA_CUDA_CHECK(cudaMemsetAsync(h->vals_bf.p, 0, total * g * t * sizeof(__nv_bfloat16), s));
      srbcrs_unique_kernel<true><<<static_cast<unsigned>(mb), 256, 0, s>>>(
          sorted.p, beg.p, end.p, static_cast<int>(g), nullptr, goff.p, h->jt.p);
      srbcrs_scatter_kernel<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, s>>>(
          indptr, indices, values, rows, static_cast<int>(t), static_cast<int>(g), goff.p, ucnt.p,
          h->jt.p, h->values.p, h->vals_bf.p);
    }
    STRATA_CUDA_CHECK(cudaGetLastError());
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));  // temporaries are freed on return
    *out = h.release();
  });
}

int strata_srbcrs_info(const strata_srbcrs* h, int64_t* mb, int64_t* t, int64_t* g,
                       int64_t* groups, int64_t* pad_slots) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null srbcrs handle");
    if (mb) *mb = h->mb;
    if (t) *t = h->t;
    if (g) *g = h->g;
    if (groups) *groups = h->groups;
    if (pad_slots) *pad_slots = h->pad_slots;
  });
}

int strata_srbcrs_read(const strata_srbcrs* h, int32_t* g_indptr, int32_t* jt_indices, float* values) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null srbcrs handle");
    if (g_indptr)
      STRATA_CUDA_CHECK(cudaMemcpy(g_indptr, h->gptr.p, (h->mb + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost));
    if (jt_indices && h->groups)
      STRATA_CUDA_CHECK(cudaMemcpy(jt_indices, h->jt.p, h->groups * h->g * sizeof(int32_t),
                                   cudaMemcpyDeviceToHost));
    if (values && h->groups)
      STRATA_CUDA_CHECK(cudaMemcpy(values, h->values.p, h->groups * h->g * h->t * sizeof(float),
                                   cudaMemcpyDeviceToHost));
  });
}

int strata_srbcrs_destroy(strata_srbcrs* h) {
  delete h;
  return STRATA_OK;
}

int strata_srbcrs_spmm_bf16(const strata_srbcrs* h, const void* X_bf16, float* Y, int64_t d,
                            void* stream) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null srbcrs handle");
    if (h->t != kT || h->g != kG)
      throw ApiError(STRATA_ERR_USAGE, "srbcrs_spmm_bf16: tensor-core path needs t == 8 and g == 32");
    if (d != 64 && d != 128 && d != 256 && d != 512)
      throw ApiError(STRATA_ERR_USAGE, "srbcrs_spmm_bf16: d must be 64, 128, 256 or 512");
    if (h->mb == 0) return;
    require_sm100_srbcrs();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const auto* X = static_cast<const __nv_bfloat16*>(X_bf16);
    switch (d) {
      case 64: launch_srbcrs<64>(*h, X, Y, s); break;
      case 128: launch_srbcrs<128>(*h, X, Y, s); break;
      case 256: launch_srbcrs<256>(*h, X, Y, s); break;
      case 512: launch_srbcrs<512>(*h, X, Y, s); break;
    }
  });
}

}  // extern "C"
