// rgms.cu — RGMS / RGCN aggregation on tcgen05 tensor cores: per-relation gather -> GEMM ->
// scatter.
//
// Reference op (kernels.cpp:138-167, driver.cpp:241-314):
//   Y[i, l] = sum_r sum_j A[r, i, j] * sum_k X[j, k] * W[r, k, l]
// over the RelSparse layout (kernels.cpp:19-62): relation-major edges, rows ascending inside a
// relation.  Flattened here to rel_ptr[R+1] / dst / src / A.
//
// Work unit: a tile of 128 edges of one relation r (tiles never straddle relations).
//   gather   X[src[e]] rows (d_in bf16) into a K-major smem tile       (cp.async, 16 B chunks)
//   stage    W_r [d_in][d_out] as the MN-major B operand                (cp.async)
//   MMA      D[e][l] = sum_k X[src e][k] * W_r[k][l]   M = 128 edges, N = d_out, K = d_in,
//            f32 accumulators in TMEM (d_in / 16 tcgen05.mma steps, one issuing thread)
//   scatter  thread e: tcgen05.ld its row, scale by A[e], red.global.add.v4.f32 into Y[dst e]
// Persistent CTAs (TMEM allocated once) walk tiles t = blockIdx.x, +gridDim.x, ... through a
// two-stage smem ring: the next tile's index loads and row gathers are in flight while the
// current tile's MMA and scatter run.  A precomputed tile -> relation map replaces any search.
// The atomic scatter makes the summation order run-dependent; with the reference's integer
// operands every partial sum is exact in f32, so results are still bitwise equal to it.
#include <cub/cub.cuh>

#include <algorithm>
#include <cuda_bf16.h>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

using namespace strata_b200;

namespace {

constexpr int kEdges = 128;  // UMMA M
constexpr int kThreads = 128;
constexpr int kCtasPerSm = 4;

__global__ void rel_tiles_kernel(const int32_t* __restrict__ rel_ptr, long long R,
                                 long long* __restrict__ ntiles) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < R) ntiles[r] = (rel_ptr[r + 1] - rel_ptr[r] + kEdges - 1) / kEdges;
  if (r == R) ntiles[R] = 0;
}

// tile_rel[t] = relation of tile t; key[t] = first destination row of tile t (one CTA per
// relation).  Unused tail entries of key (t >= tile_start[R]) are set to INT32_MAX.
__global__ void tile_rel_kernel(const int32_t* __restrict__ rel_ptr,
                                const long long* __restrict__ tile_start, long long R,
                                const int32_t* __restrict__ dst, long long max_tiles,
                                int32_t* __restrict__ tile_rel, int32_t* __restrict__ key,
                                int32_t* __restrict__ ids) {
  const long long r = blockIdx.x;
  if (r < R) {
    for (long long t = tile_start[r] + threadIdx.x; t < tile_start[r + 1]; t += blockDim.x) {
      tile_rel[t] = static_cast<int32_t>(r);
      key[t] = dst[rel_ptr[r] + (t - tile_start[r]) * kEdges];
      ids[t] = static_cast<int32_t>(t);
    }
  } else {  // block R: the padding tail
    for (long long t = tile_start[R] + threadIdx.x; t < max_tiles; t += blockDim.x) {
      key[t] = INT32_MAX;
      ids[t] = static_cast<int32_t>(t);
    }
  }
}

template <int DIN, int DOUT>
struct RgmsSmem {
  static constexpr int kABytes = kEdges * DIN * 2;
  static constexpr int kWBytes = DIN * DOUT * 2;
  static constexpr int kStage = kABytes + kWBytes;
  static constexpr int kBytes = 2 * kStage;
};

template <int DIN, int DOUT>
__global__ void __launch_bounds__(kThreads)
rgms_tc_kernel(const int32_t* __restrict__ rel_ptr, const long long* __restrict__ tile_start,
               const int32_t* __restrict__ tile_rel, const int32_t* __restrict__ order, long long R,
               const int32_t* __restrict__ dst, const int32_t* __restrict__ src,
               const float* __restrict__ A, const __nv_bfloat16* __restrict__ X,
               const __nv_bfloat16* __restrict__ W, float* __restrict__ Y) {
  using SM = RgmsSmem<DIN, DOUT>;
  constexpr int kCols = DOUT <= 32 ? 32 : (DOUT <= 64 ? 64 : (DOUT <= 128 ? 128 : 256));
  constexpr int kSboA = (DIN / 8) * 128;  // K-major A: 8-edge group stride
  constexpr int kSboW = (DIN / 8) * 128;  // MN-major B: 8-column group stride
  constexpr uint32_t kIdesc = tc::make_idesc_bf16(kEdges, DOUT, /*A K-major*/ false, /*B MN-major*/ true);
  static_assert(DIN % 16 == 0 && DIN <= 64 && DOUT % 16 == 0 && DOUT <= 256, "unsupported dims");

  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  __shared__ long long s_e0[2];
  __shared__ int s_ne[2];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long ntiles = tile_start[R];
  if (static_cast<long long>(blockIdx.x) >= ntiles) return;

  if (warp == 0) tc::tmem_alloc<kCols>(&tmem_slot);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_fence_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;

  // Issue the gathers of the p-th tile of the schedule into stage s (no wait).  Tiles run in
  // order of their first destination row, so the CTAs in flight scatter into a narrow window
  // of Y that stays in L2 (atomics into L2-missing rows were the bottleneck: 3.6 ms -> see
  // DESIGN.md §4.5).
  auto load_tile = [&](long long p, int s) {
    const long long t = order[p];
    const long long r = tile_rel[t];
    const long long e0 = rel_ptr[r] + (t - tile_start[r]) * kEdges;
    const int ne = static_cast<int>(min64(kEdges, rel_ptr[r + 1] - e0));
    if (tid == 0) {
      s_e0[s] = e0;
      s_ne[s] = ne;
    }
    uint8_t* sA = smem + s * SM::kStage;
    uint8_t* sW = sA + SM::kABytes;
    constexpr int kPer = kEdges * (DIN / 8) / kThreads;  // chunks of the A tile per thread
    long long jj[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {  // all index loads first, then the dependent copies
      const int e = (tid + q * kThreads) / (DIN / 8);
      jj[q] = e < ne ? __ldg(src + e0 + e) : 0;
    }
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int c = tid + q * kThreads;
      const int e = c / (DIN / 8), kc = c % (DIN / 8);
#ifndef STRATA_RGMS_KO_GATHER
      tc::cp_async16(sA + (e >> 3) * kSboA + kc * 128 + (e & 7) * 16, X + jj[q] * DIN + kc * 8);
#endif
    }
    const __nv_bfloat16* Wr = W + r * DIN * DOUT;
    for (int c = tid; c < DIN * (DOUT / 8); c += kThreads) {
      const int k = c / (DOUT / 8), lc = c % (DOUT / 8);
      tc::cp_async16(sW + lc * kSboW + (k >> 3) * 128 + (k & 7) * 16, Wr + k * DOUT + lc * 8);
    }
  };

  long long t = blockIdx.x;
  load_tile(t, 0);
  tc::cp_async_commit();
  for (int it = 0; t < ntiles; ++it, t += gridDim.x) {
    const int s = it & 1;
    const long long tn = t + gridDim.x;
    if (tn < ntiles) load_tile(tn, s ^ 1);
    tc::cp_async_commit();
    tc::cp_async_wait<1>();  // this tile's group has landed (the next tile's may still fly)
    tc::fence_proxy_async();
    __syncthreads();
    const long long e0 = s_e0[s];
    const int ne = s_ne[s];
#ifndef STRATA_RGMS_KO_MMA
    if (tid == 0) {
      tc::fence_after_sync();
      const uint32_t a0 = tc::smem_u32(smem + s * SM::kStage);
      const uint32_t w0 = a0 + SM::kABytes;
#pragma unroll
      for (int kk = 0; kk < DIN / 16; ++kk)
        tc::mma_bf16(tmem, tc::make_desc(a0 + kk * 256, 128, kSboA),
                     tc::make_desc(w0 + kk * 256, 128, kSboW), kIdesc, kk > 0);
      tc::mma_commit(&mbar);
    }
#endif
    // Epilogue operands, fetched while the MMA runs.
    const int e = warp * 32 + lane;
    const bool valid = e < ne;
    const float a = valid ? __ldg(A + e0 + e) : 0.f;
    const long long drow = valid ? __ldg(dst + e0 + e) : 0;
#ifndef STRATA_RGMS_KO_MMA
    tc::mbar_wait(&mbar, it & 1);
#endif
    tc::fence_after_sync();
    float* y = Y + drow * DOUT;
#pragma unroll
    for (int c0 = 0; c0 < DOUT; c0 += 32) {
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
      tc::tmem_ld_wait();
      if (valid) {
        const int n = DOUT - c0 < 32 ? DOUT - c0 : 32;
#pragma unroll
        for (int q = 0; q < 32; q += 4)
          if (q < n) {
#ifndef STRATA_RGMS_KO_RED
            tc::red_add_v4(y + c0 + q, a * __uint_as_float(v[q]), a * __uint_as_float(v[q + 1]),
                           a * __uint_as_float(v[q + 2]), a * __uint_as_float(v[q + 3]));
#else
            reinterpret_cast<float4*>(y + c0 + q)[0] = make_float4(a * __uint_as_float(v[q]), 0.f, 0.f, 0.f);
#endif
          }
      }
    }
    tc::fence_before_sync();
    __syncthreads();  // TMEM drained and stage s free before the next MMA / reload
  }
  if (warp == 0) tc::tmem_dealloc<kCols>(tmem);
}

template <int DIN, int DOUT>
void launch_rgms(const int32_t* rel_ptr, const long long* tile_start, const int32_t* tile_rel,
                 const int32_t* order, long long R, long long max_tiles, const int32_t* dst, const int32_t* src,
                 const float* A, const __nv_bfloat16* X, const __nv_bfloat16* W, float* Y,
                 cudaStream_t s) {
  constexpr int smem = RgmsSmem<DIN, DOUT>::kBytes;
  STRATA_CUDA_CHECK(cudaFuncSetAttribute(rgms_tc_kernel<DIN, DOUT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const long long grid = std::min<long long>(max_tiles, static_cast<long long>(num_sms()) * kCtasPerSm);
  rgms_tc_kernel<DIN, DOUT><<<static_cast<unsigned>(grid), kThreads, smem, s>>>(
      rel_ptr, tile_start, tile_rel, order, R, dst, src, A, X, W, Y);
  STRATA_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

extern "C" int strata_rgms_bf16(const int32_t* rel_ptr, const int32_t* dst, const int32_t* src,
                                const float* A, int64_t R, int64_t m, int64_t n, int64_t nnz,
                                const void* X_bf16, const void* W_bf16, float* Y, int64_t d_in,
                                int64_t d_out, void* stream) {
  try {
    (void)n;
    if (R < 1) throw ApiError(STRATA_ERR_USAGE, "RGMS requires at least one relation");  // kernels.cpp:139
    if (nnz > INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "nnz exceeds int32");
    int dev = 0, major = 0;
    STRATA_CUDA_CHECK(cudaGetDevice(&dev));
    STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a");
    const int dims = static_cast<int>(d_in * 1000 + d_out);
    switch (dims) {
      case 16016: case 16032: case 32016: case 32032: case 32064: case 64032: case 64064:
      case 32128: case 64128: break;
      default:
        throw ApiError(STRATA_ERR_USAGE,
                       "rgms_bf16: (d_in, d_out) must be in {16,32,64} x {16,32,64,128}");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (m > 0) STRATA_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(float) * m * d_out, s));
    if (nnz == 0) return STRATA_OK;
    const long long max_tiles = (nnz + kEdges - 1) / kEdges + R;  // upper bound on tiles
    long long *ntiles = nullptr, *tile_start = nullptr;
    int32_t* tile_rel = nullptr;
    ntiles = static_cast<long long*>(workspace_alloc(sizeof(long long) * (R + 1), s));
    tile_start = static_cast<long long*>(workspace_alloc(sizeof(long long) * (R + 1), s));
    tile_rel = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * max_tiles, s));
    rel_tiles_kernel<<<static_cast<unsigned>((R + 1 + 255) / 256), 256, 0, s>>>(rel_ptr, R, ntiles);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, ntiles, tile_start, R + 1, s);
    void* tmp = nullptr;
    tmp = workspace_alloc(tb, s);
    cub::DeviceScan::ExclusiveSum(tmp, tb, ntiles, tile_start, R + 1, s);
    int32_t* key = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * max_tiles * 2, s));
    int32_t* ids = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * max_tiles * 2, s));
    tile_rel_kernel<<<static_cast<unsigned>(R + 1), 256, 0, s>>>(rel_ptr, tile_start, R, dst,
                                                                 max_tiles, tile_rel, key, ids);
    size_t sb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, sb, key, key + max_tiles, ids, ids + max_tiles,
                                    max_tiles, 0, 32, s);
    void* stmp = workspace_alloc(sb, s);
    cub::DeviceRadixSort::SortPairs(stmp, sb, key, key + max_tiles, ids, ids + max_tiles,
                                    max_tiles, 0, 32, s);
    const int32_t* order = ids + max_tiles;
    STRATA_CUDA_CHECK(cudaGetLastError());
    const auto* X = static_cast<const __nv_bfloat16*>(X_bf16);
    const auto* W = static_cast<const __nv_bfloat16*>(W_bf16);
#define STRATA_RGMS_CASE(I, O)                                                                \
  case I * 1000 + O:                                                                          \
    launch_rgms<I, O>(rel_ptr, tile_start, tile_rel, order, R, max_tiles, dst, src, A, X, W, Y, s); \
    break;
    switch (dims) {
      STRATA_RGMS_CASE(16, 16) STRATA_RGMS_CASE(16, 32) STRATA_RGMS_CASE(32, 16)
      STRATA_RGMS_CASE(32, 32) STRATA_RGMS_CASE(32, 64) STRATA_RGMS_CASE(64, 32)
      STRATA_RGMS_CASE(64, 64) STRATA_RGMS_CASE(32, 128) STRATA_RGMS_CASE(64, 128)
    }
#undef STRATA_RGMS_CASE
    STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(stmp, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(key, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(ids, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(tile_rel, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(ntiles, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(tile_start, s));
    return STRATA_OK;
  } catch (const ApiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return STRATA_ERR_INTERNAL;
  }
}
