// csr_ops.cu — CSR SDDMM (the reference's fused nest) and the row-split CSR SpMM baseline.
//
// SDDMM (kernels.cpp:110-136, fused by sparse_fuse at :135; stage-III nest in SURVEY
// Appendix B):  B[ij] = sum_k A[ij] * X[i*d + k] * Y[k*n + J[ij]]   with Y stored [d][n].
//
// Design:
//  * Y's [d][n] layout makes the per-non-zero operand a strided column; it is transposed once
//    per call into a row-major Yt[n][d] workspace (d*n*8 bytes of traffic, tiny next to the
//    nnz*d gathers) so every gather is one coalesced 128-bit access per lane;
//  * work is split by non-zeros, not rows (power-law rows range over 4+ orders of magnitude):
//    each virtual warp (L = d/4 lanes) takes a fixed 256-non-zero chunk, stages its column
//    indices and A values in shared memory (cp.async; read back as broadcasts, no per-non-zero
//    shuffles), finds its first row with one binary search on indptr (the reference does one
//    per non-zero, lower.cpp:375-402) and walks rows forward holding the X row fragment in
//    registers; groups of L non-zeros without a row boundary skip the per-non-zero row test;
//  * per group of L non-zeros each lane forms partial dot products over its 4 features, then
//    a butterfly reduce-scatter (L-1 shuffles for L results, PAPER.md:442's two-stage
//    reduction) leaves non-zero t's full dot product in lane t, which scales by A and stores
//    B coalesced.
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

namespace strata_b200 {

namespace {

constexpr int kBlock = 256;
constexpr int kNnzPerChunk = 256;
// SDDMM non-zeros per virtual warp: 256, halved for 4-lane VWs so the staged indices / values of
// a CTA's 64 VWs stay at 64 KB of shared memory.
__host__ __device__ constexpr int sddmm_chunk(int L) { return L >= 8 ? kNnzPerChunk : kNnzPerChunk / 2; }
constexpr long long kCsrLong = 2048;  // row-split CSR SpMM: longer rows are chunked
constexpr long long kCsrChunk = 256;  // non-zeros per chunk of a long row
constexpr long long kCsrGroup = 64;   // chunk partials summed per level-1 group

// nonfinite != nullptr: set to 1 when any element is inf / NaN (for the SDDMM's integer-pipe
// conversion twins; zeroed by the caller).
template <class TO>
__global__ void transpose_kernel(const float* __restrict__ in, TO* __restrict__ out,
                                 long long rows, long long cols, int* __restrict__ nonfinite = nullptr) {
  // in[rows][cols] -> out[cols][rows]
  __shared__ float tile[32][33];
  const long long c0 = static_cast<long long>(blockIdx.x) * 32, r0 = static_cast<long long>(blockIdx.y) * 32;
  bool bad = false;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) {
      const float v = __ldcs(in + r * cols + c);
      tile[i][threadIdx.x] = v;
      bad |= (__float_as_uint(v) & 0x7f800000u) == 0x7f800000u;
    }
  }
  if (nonfinite && __any_sync(0xffffffffu, bad) && threadIdx.x == 0) *nonfinite = 1;
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const long long c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = static_cast<TO>(tile[threadIdx.x][i]);
  }
}

template <int L, class T>
__device__ __forceinline__ T reduce_scatter(T (&v)[L], int lane, unsigned mask) {
#pragma unroll
  for (int w = L / 2; w >= 1; w >>= 1) {
    const bool hi = (lane & w) != 0;
#pragma unroll
    for (int i = 0; i < w; ++i) {
      const T send = hi ? v[i] : v[i + w];
      const T keep = hi ? v[i + w] : v[i];
      v[i] = keep + __shfl_xor_sync(mask, send, w, L);
    }
  }
  return v[0];
}

#ifndef STRATA_SDDMM_F64  // A/B knob: 1 = f64 dot products (default), 0 = f32
#define STRATA_SDDMM_F64 1
#endif
// A/B knobs: float4s per lane (VEC) for d = 32 / 64 / 128; lanes per non-zero L = d / (4 VEC).
// C2 graph (114.6M nnz), VEC = 2 everywhere (256-bit gathers, U = 4 in flight, 2 CTAs/SM):
//   d = 32: 4 lanes 1.89 -> 1.71 ms; d = 64: 8 lanes 4.12 -> 3.21 ms (at U = 8 it needed 170
//   registers, 1 CTA/SM: 7.93 ms); d = 128: 16 lanes 17.20 -> 7.30 ms.  VEC = 4 spills.
#ifndef STRATA_SDDMM_ICVT  // A/B knob: gathered Yt values converted on the integer pipes, with an
#define STRATA_SDDMM_ICVT 0  // F2F twin for inf / NaN (C2 d = 64: 3.255 vs 3.224 ms — off)
#endif
#ifndef STRATA_SDDMM_VEC32
#define STRATA_SDDMM_VEC32 2
#endif
#ifndef STRATA_SDDMM_VEC64
#define STRATA_SDDMM_VEC64 2
#endif
#ifndef STRATA_SDDMM_VEC128
#define STRATA_SDDMM_VEC128 2
#endif

// Dot-product numerics.  The reference accumulates sum_k A*X*Y in f64 and rounds each partial
// to f32 (interp.cpp:88-94); the parity bar is |x - y| <= 1e-5 max(|x|, |y|, 1) against its F64
// pipeline (driver.cpp:124-144).  An f32 dot of 64 N(0,1) terms misses that bar on cancelling
// rows (measured 0.73-1.12e-5), so each lane forms its 4-feature partial with exact f64
// products (f32 x f32 fits in 53 bits) and the butterfly reduces f64: one rounding, at B.
// The X row fragment is converted once per row; Y values once per gathered element.
template <bool kF64>
struct DotT { using T = float; using XV = float4; };
template <>
struct DotT<true> { using T = double; using XV = double4; };

// The row's X fragment in the dot's precision: converted once per row, not per non-zero.
// kUp: scaled by 2^896 to pair with the integer-pipe conversion of the gathered Yt values
// (cvt_down, common.cuh) — the products x * y are unchanged.
template <bool kF64, bool kUp = false>
__device__ __forceinline__ typename DotT<kF64>::XV xfrag(const float4& x) {
  if constexpr (kF64) {
    constexpr double sc = kUp ? 0x1p896 : 1.0;
    return make_double4(static_cast<double>(x.x) * sc, static_cast<double>(x.y) * sc,
                        static_cast<double>(x.z) * sc, static_cast<double>(x.w) * sc);
  } else {
    return x;
  }
}

template <bool kUp>
__device__ __forceinline__ double ycvt(float y) {
  if constexpr (kUp) return cvt_down(y);
  else return static_cast<double>(y);
}

template <bool kF64, bool kUp = false>
__device__ __forceinline__ typename DotT<kF64>::T dot4(const typename DotT<kF64>::XV& x, const float4& y) {
  if constexpr (kF64) {
    double s = x.x * ycvt<kUp>(y.x);
    s = fma(x.y, ycvt<kUp>(y.y), s);
    s = fma(x.z, ycvt<kUp>(y.z), s);
    return fma(x.w, ycvt<kUp>(y.w), s);
  } else {
    return x.x * y.x + x.y * y.y + x.z * y.z + x.w * y.w;
  }
}

// VEC float4 per lane (VEC = 2: 8 consecutive features, one 256-bit gather per Yt row slice,
// half the lanes per non-zero and half the reduce-scatter shuffles).
template <int VEC>
struct YSlice {
  float4 v[VEC];
};

#ifndef STRATA_SDDMM_U2  // gathers in flight per lane for the 256-bit variant (A/B knob)
#define STRATA_SDDMM_U2 4
#endif

#ifndef STRATA_SDDMM_MINB  // CTAs/SM the 256-bit variants are register-budgeted for (A/B knob)
#define STRATA_SDDMM_MINB 2
#endif

// kCvt: 0 = F2F conversions of the gathered Yt values; 1 = integer-pipe conversions (exits when
// Yt holds an inf / NaN, *yflag != 0); 2 = F2F, exits when Yt is all finite (the twin of 1).
template <int L, int VEC = 1, bool kF64 = STRATA_SDDMM_F64, int kCvt = 0>
__global__ void __launch_bounds__(kBlock, VEC > 1 ? STRATA_SDDMM_MINB : 1)
sddmm_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
             const float* __restrict__ A, const float* __restrict__ X,
             const float* __restrict__ Yt, float* __restrict__ B, long long rows, long long nnz,
             long long d, const int* __restrict__ yflag) {
  if constexpr (kCvt != 0) {
    const bool nonfinite = *yflag != 0;
    if (nonfinite == (kCvt == 1)) return;
  }
  constexpr bool kUp = kF64 && kCvt == 1;
  using T = typename DotT<kF64>::T;
  using YV = YSlice<VEC>;
  constexpr int U = VEC > 1 ? STRATA_SDDMM_U2 : 8;  // (VEC = 2, U = 8 needed 170 registers: 1 CTA/SM)
  const int wl = threadIdx.x & 31;
  const int lane = threadIdx.x & (L - 1);
  const int vbase = wl & ~(L - 1);
  const unsigned vmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << vbase);
  const long long vw = (static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x) / L;
  constexpr int kChunk = sddmm_chunk(L);
  const long long e0 = vw * kChunk;
  if (e0 >= nnz) return;
  const int ne = static_cast<int>(min64(kChunk, nnz - e0));

  // Stage the chunk's column indices and A values in this VW's shared-memory slice (one
  // memory round trip; read back as broadcasts, no per-non-zero shuffles).
  extern __shared__ int4 sddmm_smem[];
  int32_t* sJ = reinterpret_cast<int32_t*>(sddmm_smem) + (threadIdx.x / L) * (2 * kChunk);
  float* sA = reinterpret_cast<float*>(sJ + kChunk);
  if (ne == kChunk) {
    for (int q = lane; q < kChunk / 4; q += L) {
      ::strata_b200::tc::cp_async16(sJ + 4 * q, indices + e0 + 4 * q);
      ::strata_b200::tc::cp_async16(sA + 4 * q, A + e0 + 4 * q);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  } else {
    for (int q = lane; q < ne; q += L) {
      sJ[q] = ld_stream(indices + e0 + q);
      sA[q] = ld_stream(A + e0 + q);
    }
  }

  // Row of e0: last row r with indptr[r] <= e0 (the reference's LocateSegment, once per chunk),
  // then rows advance with the chunk; the VW keeps the current X row fragment in registers.
  long long lo = 0, hi = rows;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) >> 1;
    if (__ldg(indptr + mid) <= e0) lo = mid; else hi = mid - 1;
  }
  int row = static_cast<int>(lo);
  long long row_end = __ldg(indptr + row + 1);
  typename DotT<kF64>::XV x[VEC];
  auto load_x = [&]() {
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      x[i] = xfrag<kF64, kUp>(ld_gather4(reinterpret_cast<const float4*>(X + static_cast<long long>(row) * d) +
                                    lane * VEC + i));
  };
  load_x();
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncwarp(vmask);

  const float4* Y4 = reinterpret_cast<const float4*>(Yt) + lane * VEC;
  const int d4 = static_cast<int>(d / 4);
  auto gather_y = [&](int col) -> YV {
    YV y;
    // the staged variants run only for d == 4 * L * VEC: a compile-time row stride, one wide
    // multiply-add per gathered row address (col >= 0)
    const float4* p;
    asm("mad.wide.u32 %0, %1, %2, %3;"
        : "=l"(p)
        : "r"(static_cast<uint32_t>(col)), "r"(static_cast<uint32_t>(L * VEC * 16)), "l"(Y4));
    (void)d4;
    if constexpr (VEC % 2 == 0) {  // Yt is the call's own 256-byte aligned workspace
#pragma unroll
      for (int i = 0; i < VEC; i += 2)
        asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(y.v[i].x), "=f"(y.v[i].y), "=f"(y.v[i].z), "=f"(y.v[i].w),
                       "=f"(y.v[i + 1].x), "=f"(y.v[i + 1].y), "=f"(y.v[i + 1].z), "=f"(y.v[i + 1].w)
                     : "l"(p + i));
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) y.v[i] = ld_gather4(p + i);
    }
    return y;
  };
  for (int g = 0; g < ne; g += L) {
    const int n = min(L, ne - g);
    const bool one_row = e0 + g + n <= row_end;  // VW-uniform: no row boundary in this group
    T part[L];
#pragma unroll
    for (int u0 = 0; u0 < L; u0 += U) {
      YV yv[U];
#pragma unroll
      for (int u = 0; u < U; u += 4) {
        const int4 c = *reinterpret_cast<const int4*>(sJ + g + u0 + u);  // broadcast LDS.128
        const int cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (u0 + u + v < n) yv[u + v] = gather_y(cc[v]);
          else
#pragma unroll
            for (int i = 0; i < VEC; ++i) yv[u + v].v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      auto dot = [&](const YV& y) -> T {
        T r = dot4<kF64, kUp>(x[0], y.v[0]);
#pragma unroll
        for (int i = 1; i < VEC; ++i) r += dot4<kF64, kUp>(x[i], y.v[i]);
        return r;
      };
      if (one_row) {
#pragma unroll
        for (int u = 0; u < U; ++u) part[u0 + u] = dot(yv[u]);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (u0 + u < n) {
            const long long e = e0 + g + u0 + u;
            if (e >= row_end) {  // next non-empty row containing e
              do { ++row; row_end = __ldg(indptr + row + 1); } while (e >= row_end);
              load_x();
            }
          }
          part[u0 + u] = dot(yv[u]);
        }
      }
    }
    const T dsum = reduce_scatter<L, T>(part, lane, vmask);
    if (lane < n) st_stream(B + e0 + g + lane, static_cast<float>(static_cast<T>(sA[g + lane]) * dsum));
  }
}

// Fallback for feature sizes the vectorised kernel does not cover: one thread per non-zero.
__global__ void sddmm_scalar_kernel(const int32_t* __restrict__ indptr,
                                    const int32_t* __restrict__ indices,
                                    const float* __restrict__ A, const float* __restrict__ X,
                                    const float* __restrict__ Yt, float* __restrict__ B,
                                    long long rows, long long nnz, long long d) {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long lo = 0, hi = rows;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) >> 1;
      if (indptr[mid] <= e) lo = mid; else hi = mid - 1;
    }
    const float* x = X + lo * d;
    const float* y = Yt + static_cast<long long>(indices[e]) * d;
    double s = 0.0;  // exact f32 products, f64 sum (see DotT)
    for (long long k = 0; k < d; ++k) s = fma(static_cast<double>(x[k]), static_cast<double>(y[k]), s);
    B[e] = static_cast<float>(static_cast<double>(A[e]) * s);
  }
}

// f64 accumulator of a float4 fragment: the CSR SpMM uses the hyb kernel's numerics (every
// product a * x exact in f64 and added in f64, one rounding at the store).
struct D4 {
  double x, y, z, w;
};
__device__ __forceinline__ void fma_d4(D4& a, float v, const float4& x) {
  const double vd = static_cast<double>(v);
  a.x = fma(vd, static_cast<double>(x.x), a.x);
  a.y = fma(vd, static_cast<double>(x.y), a.y);
  a.z = fma(vd, static_cast<double>(x.z), a.z);
  a.w = fma(vd, static_cast<double>(x.w), a.w);
}
__device__ __forceinline__ float4 round4(const D4& a) {
  return make_float4(static_cast<float>(a.x), static_cast<float>(a.y), static_cast<float>(a.z),
                     static_cast<float>(a.w));
}
__device__ __forceinline__ void add_d4(D4& a, const double4& b) {
  a.x += b.x; a.y += b.y; a.z += b.z; a.w += b.w;
}

// Row-split CSR SpMM: one virtual warp per row (the "csr" format of the reference pipeline).
template <int L>
__global__ void __launch_bounds__(kBlock)
spmm_csr_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                const float* __restrict__ A, const float* __restrict__ X, float* __restrict__ Y,
                long long rows, long long d) {
  constexpr int U = 8;
  const int wl = threadIdx.x & 31;
  const int lane = threadIdx.x & (L - 1);
  const int vbase = wl & ~(L - 1);
  const unsigned vmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << vbase);
  const long long r = (static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x) / L;
  if (r >= rows) return;
  const long long q0 = __ldg(indptr + r), q1 = __ldg(indptr + r + 1);
  if (q1 - q0 > kCsrLong) return;  // long row: spmm_csr_chunk_kernel + the two merge levels
  D4 acc{0.0, 0.0, 0.0, 0.0};
  for (long long g = q0; g < q1; g += L) {
    const long long q = g + lane;
    const int32_t col = q < q1 ? ld_stream(indices + q) : 0;
    const float val = q < q1 ? ld_stream(A + q) : 0.f;
    const int n = static_cast<int>(min64(L, q1 - g));
    for (int u0 = 0; u0 < n; u0 += U) {
      float4 xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int32_t cu = __shfl_sync(vmask, col, (u0 + u) & (L - 1), L);
        if (u0 + u < n) xv[u] = ld_gather4(reinterpret_cast<const float4*>(X + static_cast<long long>(cu) * d) + lane);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float vu = __shfl_sync(vmask, val, (u0 + u) & (L - 1), L);
        if (u0 + u < n) fma_d4(acc, vu, xv[u]);
      }
    }
  }
  st_stream4(reinterpret_cast<float4*>(Y + r * d) + lane, round4(acc));
}

// ---- long rows of the row-split CSR SpMM --------------------------------------------------
// A power-law hub row (C5: 1.8 M non-zeros) would serialise one virtual warp for milliseconds.
// Rows longer than kCsrLong are cut into kCsrChunk-non-zero chunks (one VW each, f32 partial
// in non-zero order); level 1 sums up to kCsrGroup consecutive chunk partials of a row, level
// 2 sums a row's level-1 partials — fixed shapes and orders, so the result is deterministic.
// All counts stay on the device (grid-stride over an upper bound): no host synchronisation.
struct CsrLongPlan {
  long long* coff;   // [rows + 1] exclusive scan of chunks per row (0 for short rows)
  long long* goff;   // [rows + 1] exclusive scan of level-1 groups per row
};

__global__ void csr_long_counts_kernel(const int32_t* __restrict__ indptr, long long rows,
                                       long long* __restrict__ nch, long long* __restrict__ ngr) {
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r <= rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long len = r < rows ? indptr[r + 1] - indptr[r] : 0;
    const long long c = len > kCsrLong ? (len + kCsrChunk - 1) / kCsrChunk : 0;
    nch[r] = c;
    ngr[r] = (c + kCsrGroup - 1) / kCsrGroup;
  }
}

// owner of item c: last r with off[r] <= c (off non-decreasing, off[rows] = total)
__device__ __forceinline__ long long owner_row(const long long* __restrict__ off, long long rows,
                                               long long c) {
  long long lo = 0, hi = rows;
  while (hi - lo > 1) {
    const long long mid = (lo + hi) >> 1;
    if (off[mid] <= c) lo = mid; else hi = mid;
  }
  return lo;
}

template <int L>
__global__ void __launch_bounds__(kBlock)
spmm_csr_chunk_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                      const float* __restrict__ A, const float* __restrict__ X,
                      const long long* __restrict__ coff, long long rows, double* __restrict__ part) {
  constexpr int U = 8, D = 4 * L;
  const int lane = threadIdx.x & (L - 1);
  const long long nvw = static_cast<long long>(gridDim.x) * kBlock / L;
  const long long total = coff[rows];
  for (long long c = (static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x) / L; c < total;
       c += nvw) {
    const long long r = owner_row(coff, rows, c);
    const long long q0 = indptr[r] + (c - coff[r]) * kCsrChunk;
    const long long q1 = min64(q0 + kCsrChunk, static_cast<long long>(indptr[r + 1]));
    D4 acc{0.0, 0.0, 0.0, 0.0};
    for (long long g = q0; g < q1; g += U) {
      float4 xv[U];
      float vv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (g + u < q1) {
          const int32_t cu = __ldg(indices + g + u);
          vv[u] = __ldg(A + g + u);
          xv[u] = ld_gather4(reinterpret_cast<const float4*>(X + static_cast<long long>(cu) * D) + lane);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (g + u < q1) fma_d4(acc, vv[u], xv[u]);
    }
    reinterpret_cast<double4*>(part + c * D)[lane] = make_double4(acc.x, acc.y, acc.z, acc.w);
  }
}

// level 1: group g of a row sums chunk partials [first, first + kCsrGroup) of that row, in order
template <int L>
__global__ void __launch_bounds__(kBlock)
spmm_csr_group_kernel(const long long* __restrict__ coff, const long long* __restrict__ goff,
                      long long rows, const double* __restrict__ part, double* __restrict__ l1) {
  constexpr int D = 4 * L;
  const int lane = threadIdx.x & (L - 1);
  const long long nvw = static_cast<long long>(gridDim.x) * kBlock / L;
  const long long total = goff[rows];
  for (long long g = (static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x) / L; g < total;
       g += nvw) {
    const long long r = owner_row(goff, rows, g);
    const long long c0 = coff[r] + (g - goff[r]) * kCsrGroup;
    const long long c1 = min64(c0 + kCsrGroup, coff[r + 1]);
    D4 acc{0.0, 0.0, 0.0, 0.0};
    for (long long c = c0; c < c1; ++c) add_d4(acc, reinterpret_cast<const double4*>(part + c * D)[lane]);
    reinterpret_cast<double4*>(l1 + g * D)[lane] = make_double4(acc.x, acc.y, acc.z, acc.w);
  }
}

// level 2: one VW per long row, its level-1 partials in order -> Y row
template <int L>
__global__ void __launch_bounds__(kBlock)
spmm_csr_rowsum_kernel(const long long* __restrict__ goff, long long rows,
                       const double* __restrict__ l1, float* __restrict__ Y) {
  constexpr int D = 4 * L;
  const int lane = threadIdx.x & (L - 1);
  const long long nvw = static_cast<long long>(gridDim.x) * kBlock / L;
  for (long long r = (static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x) / L; r < rows;
       r += nvw) {
    const long long g0 = goff[r], g1 = goff[r + 1];
    if (g1 == g0) continue;
    D4 acc{0.0, 0.0, 0.0, 0.0};
    for (long long g = g0; g < g1; ++g) add_d4(acc, reinterpret_cast<const double4*>(l1 + g * D)[lane]);
    st_stream4(reinterpret_cast<float4*>(Y + r * D) + lane, round4(acc));
  }
}

__global__ void spmm_csr_scalar_kernel(const int32_t* __restrict__ indptr,
                                       const int32_t* __restrict__ indices,
                                       const float* __restrict__ A, const float* __restrict__ X,
                                       float* __restrict__ Y, long long rows, long long d) {
  const long long r = blockIdx.x;
  if (r >= rows) return;
  for (long long f = threadIdx.x; f < d; f += blockDim.x) {
    double acc = 0.0;  // exact products, f64 sum, one rounding
    for (long long q = indptr[r]; q < indptr[r + 1]; ++q)
      acc = fma(static_cast<double>(A[q]), static_cast<double>(X[static_cast<long long>(indices[q]) * d + f]), acc);
    Y[r * d + f] = static_cast<float>(acc);
  }
}

}  // namespace

void sddmm_csr_launch(const int32_t* indptr, const int32_t* indices, const float* A,
                      const float* X, const float* Y, float* B, int64_t rows, int64_t cols,
                      int64_t nnz, int64_t d, cudaStream_t s) {
  if (d <= 0) throw ApiError(STRATA_ERR_USAGE, "sddmm: d must be >= 1");
  if (nnz == 0) return;
  // Y[d][n] -> Yt[n][d] once per call (f32; the vectorised kernels gather 128- / 256-bit slices),
  // noting whether Y holds an inf / NaN (selects the integer-pipe or the F2F twin below)
  float* Yt = static_cast<float*>(workspace_alloc(sizeof(float) * cols * d + 256, s));
  int* yflag = reinterpret_cast<int*>(Yt + cols * d);
  if (STRATA_SDDMM_ICVT) STRATA_CUDA_CHECK(cudaMemsetAsync(yflag, 0, sizeof(int), s));
  {
    dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((d + 31) / 32));
    transpose_kernel<float><<<grid, dim3(32, 8), 0, s>>>(Y, Yt, d, cols, STRATA_SDDMM_ICVT ? yflag : nullptr);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }
  const bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0;
  auto blocks_for = [&](int L) {
    const long long chunks = (nnz + sddmm_chunk(L) - 1) / sddmm_chunk(L);
    return static_cast<unsigned>((chunks * L + kBlock - 1) / kBlock);
  };
  // per virtual warp: column indices + A values of one chunk (2 KB; 1 KB for 4-lane VWs)
  auto smem_for = [&](int L) { return (kBlock / L) * 2 * sddmm_chunk(L) * 4; };
  const bool staged = aligned && reinterpret_cast<uintptr_t>(indices) % 16 == 0 &&
                      reinterpret_cast<uintptr_t>(A) % 16 == 0;
  // Lanes per non-zero: each lane owns 4 * VEC consecutive features (256-bit gathers for VEC >= 2)
  // so a non-zero's dot is reduced across L = d / (4 VEC) lanes; fewer lanes, fewer reduce steps.
  constexpr int v32 = STRATA_SDDMM_VEC32, v64 = STRATA_SDDMM_VEC64, v128 = STRATA_SDDMM_VEC128;
  constexpr bool kF = STRATA_SDDMM_F64 != 0;
  // (kCvt 1 + 2: the integer-pipe kernel and its F2F twin, one of which exits at once)
  constexpr int c1 = (kF && STRATA_SDDMM_ICVT) ? 1 : 0, c2 = c1 ? 2 : 0;
  static PerDeviceOnce once;  // VWs of <= 8 lanes stage 64 KB per CTA
  auto attr = [&](auto kern, int L) {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_for(L)));
  };
  once([&] {
    attr(sddmm_kernel<32 / (4 * v32), v32, kF, c1>, 32 / (4 * v32));
    attr(sddmm_kernel<32 / (4 * v32), v32, kF, c2>, 32 / (4 * v32));
    attr(sddmm_kernel<64 / (4 * v64), v64, kF, c1>, 64 / (4 * v64));
    attr(sddmm_kernel<64 / (4 * v64), v64, kF, c2>, 64 / (4 * v64));
    attr(sddmm_kernel<128 / (4 * v128), v128, kF, c1>, 128 / (4 * v128));
    attr(sddmm_kernel<128 / (4 * v128), v128, kF, c2>, 128 / (4 * v128));
  });
  auto run = [&](auto k1, auto k2, int L) {
    k1<<<blocks_for(L), kBlock, smem_for(L), s>>>(indptr, indices, A, X, Yt, B, rows, nnz, d, yflag);
    if (c2) k2<<<blocks_for(L), kBlock, smem_for(L), s>>>(indptr, indices, A, X, Yt, B, rows, nnz, d, yflag);
  };
  if (staged && d == 32)
    run(sddmm_kernel<32 / (4 * v32), v32, kF, c1>, sddmm_kernel<32 / (4 * v32), v32, kF, c2>, 32 / (4 * v32));
  else if (staged && d == 64)
    run(sddmm_kernel<64 / (4 * v64), v64, kF, c1>, sddmm_kernel<64 / (4 * v64), v64, kF, c2>, 64 / (4 * v64));
  else if (staged && d == 128)
    run(sddmm_kernel<128 / (4 * v128), v128, kF, c1>, sddmm_kernel<128 / (4 * v128), v128, kF, c2>, 128 / (4 * v128));
  else {
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((nnz + 255) / 256, 148 * 32));
    sddmm_scalar_kernel<<<blocks, 256, 0, s>>>(indptr, indices, A, X, Yt, B, rows, nnz, d);
  }
  STRATA_CUDA_CHECK(cudaGetLastError());
  STRATA_CUDA_CHECK(cudaFreeAsync(Yt, s));
}

void spmm_csr_launch(const int32_t* indptr, const int32_t* indices, const float* A,
                     const float* X, float* Y, int64_t rows, int64_t d, cudaStream_t s) {
  if (d <= 0) throw ApiError(STRATA_ERR_USAGE, "spmm: d must be >= 1");
  if (rows == 0) return;
  const bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(Y) % 16 == 0;
  auto blocks_for = [&](int L) { return static_cast<unsigned>((rows * L + kBlock - 1) / kBlock); };
  const int L = !aligned ? 0 : (d == 32 ? 8 : (d == 64 ? 16 : (d == 128 ? 32 : 0)));
  if (L == 0) {
    spmm_csr_scalar_kernel<<<static_cast<unsigned>(rows), 128, 0, s>>>(indptr, indices, A, X, Y, rows, d);
    STRATA_CUDA_CHECK(cudaGetLastError());
    return;
  }
  if (L == 8) spmm_csr_kernel<8><<<blocks_for(8), kBlock, 0, s>>>(indptr, indices, A, X, Y, rows, d);
  else if (L == 16) spmm_csr_kernel<16><<<blocks_for(16), kBlock, 0, s>>>(indptr, indices, A, X, Y, rows, d);
  else spmm_csr_kernel<32><<<blocks_for(32), kBlock, 0, s>>>(indptr, indices, A, X, Y, rows, d);
  // Long rows: per-row chunk and group counts, their scans, one host read of the totals (the
  // only synchronisation of this call; skipped work when no row is long), then three passes.
  long long* nch = static_cast<long long*>(workspace_alloc(sizeof(long long) * (rows + 1) * 4, s));
  long long *ngr = nch + (rows + 1), *coff = ngr + (rows + 1), *goff = coff + (rows + 1);
  const unsigned gr = static_cast<unsigned>(std::min<long long>((rows + 256) / 256, 148LL * 16));
  csr_long_counts_kernel<<<gr, 256, 0, s>>>(indptr, rows, nch, ngr);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, nch, coff, rows + 1, s);
  void* tmp = workspace_alloc(tb, s);
  cub::DeviceScan::ExclusiveSum(tmp, tb, nch, coff, rows + 1, s);
  cub::DeviceScan::ExclusiveSum(tmp, tb, ngr, goff, rows + 1, s);
  long long tot[2] = {0, 0};
  STRATA_CUDA_CHECK(cudaMemcpyAsync(&tot[0], coff + rows, sizeof(long long), cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaMemcpyAsync(&tot[1], goff + rows, sizeof(long long), cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  const long long max_chunks = tot[0], max_groups = tot[1];
  if (max_chunks == 0) {
    STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
    STRATA_CUDA_CHECK(cudaFreeAsync(nch, s));
    return;
  }
  double* part = static_cast<double*>(workspace_alloc(sizeof(double) * (max_chunks + max_groups) * d, s));
  double* l1 = part + max_chunks * d;
  const unsigned gc = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((max_chunks * L + kBlock - 1) / kBlock, 148LL * 64)));
  const unsigned gg = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((max_groups * L + kBlock - 1) / kBlock, 148LL * 64)));
  const unsigned grr = static_cast<unsigned>(std::min<long long>((rows * L + kBlock - 1) / kBlock, 148LL * 64));
  if (L == 8) {
    spmm_csr_chunk_kernel<8><<<gc, kBlock, 0, s>>>(indptr, indices, A, X, coff, rows, part);
    spmm_csr_group_kernel<8><<<gg, kBlock, 0, s>>>(coff, goff, rows, part, l1);
    spmm_csr_rowsum_kernel<8><<<grr, kBlock, 0, s>>>(goff, rows, l1, Y);
  } else if (L == 16) {
    spmm_csr_chunk_kernel<16><<<gc, kBlock, 0, s>>>(indptr, indices, A, X, coff, rows, part);
    spmm_csr_group_kernel<16><<<gg, kBlock, 0, s>>>(coff, goff, rows, part, l1);
    spmm_csr_rowsum_kernel<16><<<grr, kBlock, 0, s>>>(goff, rows, l1, Y);
  } else {
    spmm_csr_chunk_kernel<32><<<gc, kBlock, 0, s>>>(indptr, indices, A, X, coff, rows, part);
    spmm_csr_group_kernel<32><<<gg, kBlock, 0, s>>>(coff, goff, rows, part, l1);
    spmm_csr_rowsum_kernel<32><<<grr, kBlock, 0, s>>>(goff, rows, l1, Y);
  }
  STRATA_CUDA_CHECK(cudaGetLastError());
  STRATA_CUDA_CHECK(cudaFreeAsync(part, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(nch, s));
}

}  // namespace strata_b200

// ---- csr_to_ell (storage.cpp:190-227) ---------------------------------------------------
namespace strata_b200 {
namespace {

__global__ void ell_capacity_kernel(const int32_t* __restrict__ indptr, long long rows,
                                    long long w, unsigned long long* __restrict__ first_bad) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < rows;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    if (indptr[i + 1] - indptr[i] > w) atomicMin(first_bad, static_cast<unsigned long long>(i));
}

__global__ void ell_fill_kernel(const int32_t* __restrict__ indptr,
                                const int32_t* __restrict__ indices,
                                const float* __restrict__ values, long long rows, long long w,
                                int32_t* __restrict__ J, float* __restrict__ V) {
  const long long total = rows * w;
  for (long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long i = t / w, s = t - i * w;
    const long long q0 = indptr[i], l = indptr[i + 1] - q0;
    if (s < l) {
      J[t] = indices[q0 + s];
      V[t] = values[q0 + s];
    } else {  // pad with the row's last real column (0 for an empty row), value 0
      J[t] = l > 0 ? indices[q0 + l - 1] : 0;
      V[t] = 0.f;
    }
  }
}

}  // namespace

void ell_from_csr_launch(const int32_t* indptr, const int32_t* indices, const float* values,
                         int64_t rows, int64_t cols, int64_t w, int32_t* J, float* V,
                         cudaStream_t s) {
  if (w < 1) throw ApiError(STRATA_ERR_USAGE, "ELL width must be >= 1");
  if (w > cols) throw ApiError(STRATA_ERR_USAGE, "ELL width exceeds column count");
  if (rows == 0) return;
  unsigned long long* bad = nullptr;
  bad = static_cast<unsigned long long*>(workspace_alloc(sizeof(unsigned long long), s));
  STRATA_CUDA_CHECK(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s));
  ell_capacity_kernel<<<static_cast<unsigned>(std::min<long long>((rows + 255) / 256, 4096)), 256, 0, s>>>(
      indptr, rows, w, bad);
  unsigned long long hbad = 0;
  STRATA_CUDA_CHECK(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(bad, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  if (hbad != ~0ull) {
    int32_t ip[2];
    STRATA_CUDA_CHECK(cudaMemcpy(ip, indptr + hbad, sizeof(ip), cudaMemcpyDeviceToHost));
    throw ApiError(STRATA_ERR_CAPACITY, "row " + std::to_string(hbad) + " has " +
                                            std::to_string(ip[1] - ip[0]) +
                                            " non-zeros, exceeds ELL width " + std::to_string(w));
  }
  const long long total = rows * w;
  ell_fill_kernel<<<static_cast<unsigned>(std::min<long long>((total + 255) / 256, 148 * 64)), 256, 0, s>>>(
      indptr, indices, values, rows, w, J, V);
  STRATA_CUDA_CHECK(cudaGetLastError());
}

}  // namespace strata_b200
