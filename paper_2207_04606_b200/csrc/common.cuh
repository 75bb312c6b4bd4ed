// common.cuh — small device helpers shared by the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace strata_b200 {

__host__ __device__ __forceinline__ long long min64(long long a, long long b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ long long max64(long long a, long long b) { return a > b ? a : b; }

// Streaming (evict-first) loads for data touched exactly once: index / value arrays.
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) { return __ldcs(p); }
__device__ __forceinline__ float ld_stream(const float* p) { return __ldcs(p); }

// Gathered dense-operand rows: read-only path, L1-allocating (a row gathered by one slot is
// often re-gathered by the pad slots and duplicate columns of the same segment).
__device__ __forceinline__ float4 ld_gather4(const float4* p) { return __ldg(p); }
__device__ __forceinline__ float ld_gather(const float* p) { return __ldg(p); }

// Output rows are written once: streaming store, do not keep in L2.
__device__ __forceinline__ void st_stream4(float4* p, float4 v) { __stcs(p, v); }
__device__ __forceinline__ void st_stream(float* p, float v) { __stcs(p, v); }

__device__ __forceinline__ void fma4(float4& acc, float a, const float4& x) {
  acc.x = fmaf(a, x.x, acc.x);
  acc.y = fmaf(a, x.y, acc.y);
  acc.z = fmaf(a, x.z, acc.z);
  acc.w = fmaf(a, x.w, acc.w);
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

// f32 -> f64 of a FINITE x on the integer pipes, scaled by 2^-896: the f32 bit fields re-based
// in place (sign | e32 | m[22:3] into the high word, m[2:0] into the low word), so every normal
// f32 lands on a normal double, a subnormal on the equal double subnormal, +-0 on +-0.  With
// the other factor scaled by 2^896 (exact: |a| < 2^128), fma(a * 2^896, cvt_down(x), s) ==
// fma(double(a), double(x), s) bit for bit.  It replaces one F2F per gathered element — the
// XU pipe's rate bounds the L2-resident gathers (C2 SpMM: ncu XU 74 % of peak) — by three
// integer ops.  inf / NaN map to finite values, so kernels using it run only when the gathered
// operand was scanned finite; otherwise their F2F twin runs.
__device__ __forceinline__ double cvt_down(float x) {
  const uint32_t u = __float_as_uint(x);
  const uint32_t hi = static_cast<uint32_t>(static_cast<int32_t>(u) >> 3) & 0x8FFFFFFFu;
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(u << 29));
}

}  // namespace strata_b200
