// rgms.cu — RGMS / RGCN aggregation on tcgen05 tensor cores: per-relation gather -> GEMM ->
// scatter.
//
// Reference op (kernels.cpp:138-167, driver.cpp:241-314):
//   Y[i, l] = sum_r sum_j A[r, i, j] * sum_k X[j, k] * W[r, k, l]
// over the RelSparse layout (kernels.cpp:19-62): relation-major edges, rows ascending inside a
// relation.  Flattened here to rel_ptr[R+1] / dst / src / A.
//
// Kernel: one CTA per tile of 128 edges of one relation r.
//   gather   X[src[e]] rows (d_in bf16) into a K-major smem tile       (cp.async, 16 B chunks)
//   stage    W_r [d_in][d_out] as the MN-major B operand                (cp.async)
//   MMA      D[e][l] = sum_k X[src e][k] * W_r[k][l]   M = 128 edges, N = d_out, K = d_in,
//            f32 accumulators in TMEM (d_in / 16 tcgen05.mma steps, one issuing thread)
//   scatter  thread e: tcgen05.ld its row, scale by A[e], red.global.add.v4.f32 into Y[dst e]
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

__global__ void rel_tiles_kernel(const int32_t* __restrict__ rel_ptr, long long R,
                                 long long* __restrict__ ntiles) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r < R) ntiles[r] = (rel_ptr[r + 1] - rel_ptr[r] + kEdges - 1) / kEdges;
  if (r == R) ntiles[R] = 0;
}

template <int DIN, int DOUT>
__global__ void __launch_bounds__(kThreads)
rgms_tc_kernel(const int32_t* __restrict__ rel_ptr, const long long* __restrict__ tile_start,
               long long R, const int32_t* __restrict__ dst, const int32_t* __restrict__ src,
               const float* __restrict__ A, const __nv_bfloat16* __restrict__ X,
               const __nv_bfloat16* __restrict__ W, float* __restrict__ Y) {
  constexpr int kCols = DOUT < 32 ? 32 : (DOUT <= 32 ? 32 : (DOUT <= 64 ? 64 : (DOUT <= 128 ? 128 : 256)));
  constexpr int kSboA = (DIN / 8) * 128;   // K-major A: 8-edge group stride
  constexpr int kSboW = (DIN / 8) * 128;   // MN-major B: 8-column group stride
  constexpr int kABytes = kEdges * DIN * 2;
  constexpr uint32_t kIdesc = tc::make_idesc_bf16(kEdges, DOUT, /*A K-major*/ false, /*B MN-major*/ true);
  static_assert(DIN % 16 == 0 && DIN <= 64 && DOUT % 16 == 0 && DOUT <= 256, "unsupported dims");

  __shared__ __align__(128) uint8_t sA[kABytes];
  __shared__ __align__(128) uint8_t sW[DIN * DOUT * 2];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_slot;
  __shared__ long long s_rel;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const long long t = blockIdx.x;
  if (tid == 0) {  // relation of this tile: last r with tile_start[r] <= t
    long long lo = 0, hi = R;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (tile_start[mid] <= t) lo = mid; else hi = mid - 1;
    }
    s_rel = (t < tile_start[R]) ? lo : -1;
  }
  __syncthreads();
  const long long r = s_rel;
  if (r < 0) return;
  const long long e0 = rel_ptr[r] + (t - tile_start[r]) * kEdges;
  const int ne = static_cast<int>(min64(kEdges, rel_ptr[r + 1] - e0));

  if (warp == 0) tc::tmem_alloc<kCols>(&tmem_slot);
  if (tid == 0) {
    tc::mbar_init(&mbar, 1);
    tc::mbar_fence_init();
  }
  // Gather the 128 source rows (K-major) and W_r (MN-major).
  for (int c = tid; c < kEdges * (DIN / 8); c += kThreads) {
    const int e = c / (DIN / 8), kc = c % (DIN / 8);
    const long long j = e < ne ? src[e0 + e] : 0;
    tc::cp_async16(sA + (e >> 3) * kSboA + kc * 128 + (e & 7) * 16, X + j * DIN + kc * 8);
  }
  const __nv_bfloat16* Wr = W + r * DIN * DOUT;
  for (int c = tid; c < DIN * (DOUT / 8); c += kThreads) {
    const int k = c / (DOUT / 8), lc = c % (DOUT / 8);
    tc::cp_async16(sW + lc * kSboW + (k >> 3) * 128 + (k & 7) * 16, Wr + k * DOUT + lc * 8);
  }
  tc::cp_async_commit();
  tc::cp_async_wait<0>();
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {
    const uint32_t a0 = tc::smem_u32(sA), w0 = tc::smem_u32(sW);
#pragma unroll
    for (int kk = 0; kk < DIN / 16; ++kk)
      tc::mma_bf16(tmem, tc::make_desc(a0 + kk * 256, 128, kSboA),
                   tc::make_desc(w0 + kk * 256, 128, kSboW), kIdesc, kk > 0);
    tc::mma_commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();

  const int e = warp * 32 + lane;
  const bool valid = e < ne;
  const float a = valid ? A[e0 + e] : 0.f;
  float* y = valid ? Y + static_cast<long long>(dst[e0 + e]) * DOUT : nullptr;
#pragma unroll
  for (int c0 = 0; c0 < DOUT; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    if (valid) {
      const int n = DOUT - c0 < 32 ? DOUT - c0 : 32;
#pragma unroll
      for (int q = 0; q < 32; q += 4)
        if (q < n)
          tc::red_add_v4(y + c0 + q, a * __uint_as_float(v[q]), a * __uint_as_float(v[q + 1]),
                         a * __uint_as_float(v[q + 2]), a * __uint_as_float(v[q + 3]));
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<kCols>(tmem);
}

template <int DIN, int DOUT>
void launch_rgms(const int32_t* rel_ptr, const long long* tile_start, long long R, long long grid,
                 const int32_t* dst, const int32_t* src, const float* A, const __nv_bfloat16* X,
                 const __nv_bfloat16* W, float* Y, cudaStream_t s) {
  rgms_tc_kernel<DIN, DOUT><<<static_cast<unsigned>(grid), kThreads, 0, s>>>(
      rel_ptr, tile_start, R, dst, src, A, X, W, Y);
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
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (m > 0) STRATA_CUDA_CHECK(cudaMemsetAsync(Y, 0, sizeof(float) * m * d_out, s));
    if (nnz == 0) return STRATA_OK;
    long long *ntiles = nullptr, *tile_start = nullptr;
    STRATA_CUDA_CHECK(cudaMallocAsync(&ntiles, sizeof(long long) * (R + 1), s));
    STRATA_CUDA_CHECK(cudaMallocAsync(&tile_start, sizeof(long long) * (R + 1), s));
    rel_tiles_kernel<<<static_cast<unsigned>((R + 1 + 255) / 256), 256, 0, s>>>(rel_ptr, R, ntiles);
    size_t tb = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, ntiles, tile_start, R + 1, s);
    void* tmp = nullptr;
    STRATA_CUDA_CHECK(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), s));
    cub::DeviceScan::ExclusiveSum(tmp, tb, ntiles, tile_start, R + 1, s);
    const long long grid = (nnz + kEdges - 1) / kEdges + R;  // upper bound on tiles
    const auto* X = static_cast<const __nv_bfloat16*>(X_bf16);
    const auto* W = static_cast<const __nv_bfloat16*>(W_bf16);
    const int key = static_cast<int>(d_in * 1000 + d_out);
    switch (key) {
      case 16016: launch_rgms<16, 16>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 16032: launch_rgms<16, 32>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 32016: launch_rgms<32, 16>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 32032: launch_rgms<32, 32>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 32064: launch_rgms<32, 64>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 64032: launch_rgms<64, 32>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 64064: launch_rgms<64, 64>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 32128: launch_rgms<32, 128>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      case 64128: launch_rgms<64, 128>(rel_ptr, tile_start, R, grid, dst, src, A, X, W, Y, s); break;
      default:
        throw ApiError(STRATA_ERR_USAGE,
                       "rgms_bf16: (d_in, d_out) must be in {16,32,64} x {16,32,64,128}");
    }
    STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
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
