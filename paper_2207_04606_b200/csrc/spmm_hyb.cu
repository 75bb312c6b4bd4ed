// spmm_hyb.cu — hyb SpMM on sm_100a CUDA cores (HBM-bound gather kernel).
//
// Computes the reference's decomposed SpMM (kernels.cpp:85-108 through decompose_format,
// transform.cpp:215-388; stage-III nest in SURVEY Appendix B):
//   for each part (p, b) in rule order, for each ELL row r, slot s < 2^b, k < d:
//     Y[I[r]*d + k] += A[r*2^b + s] * X[J[r*2^b + s]*d + k]
//
// Design:
//  * one launch covers every part of a column partition ("horizontal fusion");
//  * work unit = chunk of ~256 consecutive ELL slots (whole rows) per *virtual warp* (VW) of
//    L = min(32, d/4) lanes; lane l owns float4 column groups l, l+L, ... of the feature row,
//    so every gathered X row is one fully coalesced 128-bit access per lane;
//  * index/value tiles are loaded L slots at a time (coalesced, streaming), pad slots are
//    detected with the reference's own rule (a slot repeating the previous column of the same
//    segment, storage.cpp:484/528) and skipped, and up to U real-slot gathers are issued before
//    any is consumed (U x 16 B in flight per lane) to hide HBM latency;
//  * each output row is produced by exactly one VW with a plain streaming store, except the
//    rows that decompose_hyb split into several bucket-k segments (storage.cpp:301-309) and
//    whose segment run crosses a chunk boundary: those chunks write their partial row to a
//    carry buffer and spmm_fixup_kernel sums the carries of each run in chunk order with a
//    fixed-shape tree.  No atomics, so the result is bitwise reproducible run to run.
//  * c > 1: partitions are launched in order and accumulate (Y zeroed first), which keeps
//    the reference's per-row accumulation order across partitions (ascending columns).
#include <algorithm>
#include <string>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

#define tc_cp_async16 ::strata_b200::tc::cp_async16

namespace strata_b200 {

namespace {

#ifndef STRATA_SPMM_XG  // A/B knob: lane-offset gather base + one wide multiply-add per row address
#define STRATA_SPMM_XG 1
#endif

constexpr int kMaxParts = 32;
constexpr int kBlock = 256;
constexpr int kPiece = 256;  // ELL slots staged in shared memory per virtual warp at a time
constexpr int kMaxYDests = STRATA_MAX_Y_DESTS;

struct SpmmPartDev {
  long long slot_off, row_off, nrows, chunk_begin, nchunks, carry_off;
  int b, rpc_log2, may_split, pad_;
};

// Output row destinations: every finished Y row is stored to each of the n buffers (the
// caller's Y, plus — for the fused multi-GPU all-gather — peers' Y replicas mapped over NVLink).
struct YDests {
  float* p[kMaxYDests];
  int n;
};

struct SpmmArgs {
  const int32_t* I;
  const int32_t* J;
  const float* V;
  const float* X;
  YDests Y;
  double* carry;
  double* yacc;  // c > 1 only: f64 accumulator [rows][d]; else nullptr
  long long d;
  long long total_chunks;
  int nparts;
  int w256;  // X 32-byte aligned: 256-bit slice loads for VEC >= 2
  const int* xflag;  // kCvt != 0 variants: 1 when X holds an inf / NaN (x_nonfinite_kernel)
  SpmmPartDev parts[kMaxParts];
};

template <int VEC, bool kScalar>
struct Frag {
  float4 v[VEC];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
};

// Gather one X row fragment owned by this lane.
template <int L, int VEC, bool kScalar>
__device__ __forceinline__ void gather(Frag<VEC, kScalar>& f, const float* __restrict__ X,
                                       long long col, long long d, int lane, long long feat0,
                                       bool w256) {
  if constexpr (kScalar) {
    const long long fi = feat0 + lane;
    f.v[0].x = fi < d ? ld_gather(X + col * d + fi) : 0.f;
  } else {
    // Vector variants are launched only for d == 4 * L * VEC, so the row stride is a
    // compile-time constant.  A lane owns VEC consecutive float4 of the row (feature
    // 4*VEC*lane ..): with VEC = 2 one 256-bit load (sm_100 LDG.256), with VEC = 4 two.
    // X is the lane-offset base (X + 4 * VEC * lane floats, hoisted out of the loop): one
    // 32 x 32 -> 64-bit multiply-add per gathered row instead of a shift / merge / LEA chain.
    (void)d;
#if STRATA_SPMM_XG
    (void)lane;
    const float4* xp;
    asm("mad.wide.u32 %0, %1, %2, %3;"
        : "=l"(xp)
        : "r"(static_cast<uint32_t>(col)), "r"(static_cast<uint32_t>(L * VEC * 16)), "l"(X));
#else
    const float4* xp = reinterpret_cast<const float4*>(X) +
                       (static_cast<unsigned long long>(static_cast<uint32_t>(col)) * (L * VEC)) + lane * VEC;
#endif
    // L < 32 VEC variants (d = 64) are launched only on 32-byte aligned X; d = 256 / 512 check
    if (VEC % 2 == 0 && (L < 32 || w256)) {  // warp-uniform
#pragma unroll
      for (int i = 0; i + 1 < VEC; i += 2)
        asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                     : "=f"(f.v[i].x), "=f"(f.v[i].y), "=f"(f.v[i].z), "=f"(f.v[i].w),
                       "=f"(f.v[i + 1].x), "=f"(f.v[i + 1].y), "=f"(f.v[i + 1].z), "=f"(f.v[i + 1].w)
                     : "l"(xp + i));
    } else {
#pragma unroll
      for (int i = 0; i < VEC; ++i) f.v[i] = ld_gather4(xp + i);
    }
  }
}

// Two-level accumulation.  Each batch of <= U gathered slots of one output row is summed with
// f32 FMAs into a partial, which is then folded into an f64 accumulator; the f64 sum is rounded
// to f32 once, at the store.  The f32 rounding error is therefore that of an <= U-term sum per
// batch instead of growing with the row (the reference's sequential f32 accumulation drifts by
// ~2e-5 from its own F64 pipeline on long rows, golden.npz), and only one F32->F64 conversion
// per lane-feature per batch is paid.  Integer operands stay exact (all partial sums < 2^24).
template <int VEC, bool kScalar>
struct Acc {
  double v[kScalar ? 1 : 4 * VEC];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int i = 0; i < (kScalar ? 1 : 4 * VEC); ++i) v[i] = 0.0;
  }
};

// Exact-product accumulation (STRATA_SPMM_F64 = 1, the default): every product a * x is formed
// and added in f64 (a product of two f32 is exact in f64), so the only f32 rounding is the final
// store.  The f32-batch form above rounds each product and each batch sum in f32; on long rows
// whose sum cancels towards 0 that alone exceeds the north_star's 1e-5 bar against the F64
// pipeline (sqrt(n) * 2^-24 * |a x|), so it is kept only as an A/B knob (STRATA_SPMM_F64=0).
#ifndef STRATA_SPMM_F64
#define STRATA_SPMM_F64 1
#endif

// Exact products with X converted on the integer pipes (cvt_down, common.cuh).
template <bool kUp, int VEC, bool kScalar>
__device__ __forceinline__ void fma_acc(Acc<VEC, kScalar>& acc, float a, const Frag<VEC, kScalar>& x) {
  if constexpr (kUp && !kScalar) {
    const double au = static_cast<double>(a) * 0x1p896;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      acc.v[4 * i + 0] = fma(au, cvt_down(x.v[i].x), acc.v[4 * i + 0]);
      acc.v[4 * i + 1] = fma(au, cvt_down(x.v[i].y), acc.v[4 * i + 1]);
      acc.v[4 * i + 2] = fma(au, cvt_down(x.v[i].z), acc.v[4 * i + 2]);
      acc.v[4 * i + 3] = fma(au, cvt_down(x.v[i].w), acc.v[4 * i + 3]);
    }
  } else {
    fma_acc(acc, a, x);
  }
}

template <int VEC, bool kScalar>
__device__ __forceinline__ void fma_acc(Acc<VEC, kScalar>& acc, float a, const Frag<VEC, kScalar>& x) {
  const double ad = static_cast<double>(a);
  if constexpr (kScalar) {
    acc.v[0] = fma(ad, static_cast<double>(x.v[0].x), acc.v[0]);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      acc.v[4 * i + 0] = fma(ad, static_cast<double>(x.v[i].x), acc.v[4 * i + 0]);
      acc.v[4 * i + 1] = fma(ad, static_cast<double>(x.v[i].y), acc.v[4 * i + 1]);
      acc.v[4 * i + 2] = fma(ad, static_cast<double>(x.v[i].z), acc.v[4 * i + 2]);
      acc.v[4 * i + 3] = fma(ad, static_cast<double>(x.v[i].w), acc.v[4 * i + 3]);
    }
  }
}

template <int VEC, bool kScalar>
__device__ __forceinline__ void add_acc(Acc<VEC, kScalar>& acc, const Acc<VEC, kScalar>& o) {
#pragma unroll
  for (int i = 0; i < (kScalar ? 1 : 4 * VEC); ++i) acc.v[i] += o.v[i];
}

template <int VEC, bool kScalar>
__device__ __forceinline__ void fma_part(Frag<VEC, kScalar>& part, float a,
                                         const Frag<VEC, kScalar>& x) {
  if constexpr (kScalar) {
    part.v[0].x = fmaf(a, x.v[0].x, part.v[0].x);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) fma4(part.v[i], a, x.v[i]);
  }
}

template <int VEC, bool kScalar>
__device__ __forceinline__ void add_part(Frag<VEC, kScalar>& part, const Frag<VEC, kScalar>& p1) {
  if constexpr (kScalar) {
    part.v[0].x += p1.v[0].x;
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) part.v[i] = add4(part.v[i], p1.v[i]);
  }
}

template <int VEC, bool kScalar>
__device__ __forceinline__ void absorb(Acc<VEC, kScalar>& acc, Frag<VEC, kScalar>& part) {
  if constexpr (kScalar) {
    acc.v[0] += static_cast<double>(part.v[0].x);
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      acc.v[4 * i + 0] += static_cast<double>(part.v[i].x);
      acc.v[4 * i + 1] += static_cast<double>(part.v[i].y);
      acc.v[4 * i + 2] += static_cast<double>(part.v[i].z);
      acc.v[4 * i + 3] += static_cast<double>(part.v[i].w);
    }
  }
  part.zero();
}

// Store one output row fragment of Y (f32): the single rounding of the whole sum.
template <int L, int VEC, bool kScalar>
__device__ __forceinline__ void put_row(float* __restrict__ row, const Acc<VEC, kScalar>& acc,
                                        long long d, int lane, long long feat0) {
  if constexpr (kScalar) {
    const long long fi = feat0 + lane;
    if (fi < d) row[fi] = static_cast<float>(acc.v[0]);
  } else {
    float4* rp = reinterpret_cast<float4*>(row) + lane * VEC;
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      st_stream4(rp + i, make_float4(static_cast<float>(acc.v[4 * i]), static_cast<float>(acc.v[4 * i + 1]),
                                         static_cast<float>(acc.v[4 * i + 2]), static_cast<float>(acc.v[4 * i + 3])));
  }
}

// Store (carry buffer) or add (c > 1 f64 accumulator) an f64 row fragment.
template <int L, int VEC, bool kScalar, bool kAdd>
__device__ __forceinline__ void put_f64(double* __restrict__ row, const Acc<VEC, kScalar>& acc,
                                        long long d, int lane, long long feat0) {
  if constexpr (kScalar) {
    const long long fi = feat0 + lane;
    if (fi < d) row[fi] = kAdd ? row[fi] + acc.v[0] : acc.v[0];
  } else {
    double2* rp = reinterpret_cast<double2*>(row) + 2 * lane * VEC;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      double2 a0 = make_double2(acc.v[4 * i], acc.v[4 * i + 1]);
      double2 a1 = make_double2(acc.v[4 * i + 2], acc.v[4 * i + 3]);
      if constexpr (kAdd) {
        const double2 o0 = rp[2 * i], o1 = rp[2 * i + 1];
        a0.x += o0.x; a0.y += o0.y; a1.x += o1.x; a1.y += o1.y;
      }
      rp[2 * i] = a0;
      rp[2 * i + 1] = a1;
    }
  }
}

#ifndef STRATA_SPMM_VEC64  // A/B knob: d = 64 as 8 lanes x 256-bit slices (2) or 16 x 128-bit (1)
#define STRATA_SPMM_VEC64 2    // (C2: 3.30 -> 2.91 ms)
#endif
#ifndef STRATA_SPMM_VEC128  // A/B knob: d = 128 as 16 lanes x 256-bit slices (2) or 32 x 128-bit (1)
#define STRATA_SPMM_VEC128 1   // (C5: 5.05 -> 5.54 ms with 2: the DRAM-bound case keeps 32 lanes)
#endif
#ifndef STRATA_SPMM_ICVT  // A/B knob: d = 64 gathers converted on the integer pipes (C2 2.91 -> 2.59 ms)
#define STRATA_SPMM_ICVT 1
#endif
#ifndef STRATA_SPMM_MINB_V2  // CTAs/SM the 256-bit d = 64 variant is register-budgeted for
#define STRATA_SPMM_MINB_V2 2
#endif
#ifndef STRATA_SPMM_MINB16  // CTAs/SM the d=64 variant is register-budgeted for (A/B knob)
#define STRATA_SPMM_MINB16 2
#endif
#ifndef STRATA_SPMM_MINB32  // CTAs/SM the d=128 variant is register-budgeted for (A/B knob)
#define STRATA_SPMM_MINB32 3
#endif

// Main kernel.  Per virtual warp (VW): one chunk of whole ELL rows, processed in pieces of
// <= 256 slots:
//   1. stage: the piece's J / V tiles and the output rows of its ELL rows are copied to the
//      VW's shared-memory buffer with one burst of cp.async per lane (one memory round trip);
//   2. compact (in place): pad slots — a repeat of the previous column inside a row, the
//      reference's own rule (storage.cpp:528) — are dropped with a VW-wide scan, and the first
//      slot of every ELL row is flagged in bit 31 of its column;
//   3. consume: batches of 8 real slots are read with broadcast 128-bit shared loads (no
//      shuffles), their X rows gathered UG at a time (128-bit per lane), and accumulated.
// kCvt: 0 = F2F conversions; 1 = integer-pipe conversions (cvt_down), exits when the call's X
// holds an inf / NaN (*a.xflag != 0); 2 = F2F, exits when X is all finite (the twin of 1).
template <int L, int VEC, bool kScalar, bool kMulti, int kCvt = 0>
// (the multi-destination instantiation keeps the 3-CTA budget only for one destination's worth
// of registers: it gets the 2-CTA budget, so its replica stores do not spill)
__global__ void __launch_bounds__(kBlock, (VEC > 1 && L == 32) ? 1 : (VEC > 1 ? STRATA_SPMM_MINB_V2 : ((L == 32 && !kScalar && !kMulti) ? STRATA_SPMM_MINB32 : (L == 16 && !kScalar ? STRATA_SPMM_MINB16 : 2))))
spmm_hyb_kernel(const __grid_constant__ SpmmArgs a) {
  if constexpr (kCvt != 0) {
    const bool nonfinite = *a.xflag != 0;
    if (nonfinite == (kCvt == 1)) return;
  }
  constexpr bool kUp = kCvt == 1;
  constexpr int kT = 8;  // real slots per consume batch / slots per lane per compaction round
#ifndef STRATA_SPMM_UG  // gathers in flight per lane for the float4 variants (A/B knob)
#define STRATA_SPMM_UG 8
#endif
#ifndef STRATA_SPMM_UG2  // ... for the 256-bit (VEC = 2) variants: the L2-resident (integer-pipe
#define STRATA_SPMM_UG2 2  // conversion, kCvt != 0) kernels (C2: UG = 1 / 2 / 4 / 8 -> 2.48 /
#endif                     // 2.45 / 2.51 / 3.75 ms) and the DRAM-bound F2F one (C5-shape d = 64:
#ifndef STRATA_SPMM_UG2_DRAM  // UG 2 -> 4: 4.07 -> 3.73 ms GNN layer 128 -> 64)
#define STRATA_SPMM_UG2_DRAM 4
#endif
  constexpr int UG = kScalar ? 8
                             : (VEC == 1 ? STRATA_SPMM_UG
                                         : (VEC == 2 ? (kCvt != 0 ? STRATA_SPMM_UG2 : STRATA_SPMM_UG2_DRAM) : 2));
  constexpr int kRound = kT * L;  // slots examined per compaction round
  constexpr int32_t kRowFlag = static_cast<int32_t>(0x80000000u);
  const int lane = threadIdx.x & (L - 1);
  const long long vw = (static_cast<long long>(blockIdx.x) * kBlock + threadIdx.x) / L;
  if (vw >= a.total_chunks) return;
  const long long feat0 = kScalar ? static_cast<long long>(blockIdx.y) * 32 : 0;
  const float* __restrict__ Xg = (kScalar || !STRATA_SPMM_XG) ? a.X : a.X + 4 * VEC * lane;  // gather base

  int pi = 0;
  while (pi + 1 < a.nparts && vw >= a.parts[pi + 1].chunk_begin) ++pi;
  const SpmmPartDev& P = a.parts[pi];
  const int b = P.b;
  // Part-local row / slot indices are 32-bit (the planner guarantees < 2^31 slots per part).
  const int wmask = (1 << b) - 1;
  const int c = static_cast<int>(vw - P.chunk_begin);
  const int r0 = c << P.rpc_log2;
  const int r1 = static_cast<int>(min64(static_cast<long long>(r0) + (1ll << P.rpc_log2), P.nrows));
  const int32_t* __restrict__ Ip = a.I + P.row_off;
  const int32_t* __restrict__ Jp = a.J + P.slot_off;  // slot_off is a multiple of 8 (16 B)
  const float* __restrict__ Vp = a.V + P.slot_off;
  const long long d = a.d;
  const bool split = P.may_split != 0;
  bool head_cont = false, tail_cont = false;
  if (split) {
    head_cont = c > 0 && __ldg(Ip + r0 - 1) == __ldg(Ip + r0);
    tail_cont = c + 1 < P.nchunks && __ldg(Ip + r1 - 1) == __ldg(Ip + r1);
  }

  Acc<VEC, kScalar> acc;    // f64 running sum of the current output row (group)
  Frag<VEC, kScalar> part;  // f32 partial of the current batch
  acc.zero();
  part.zero();
  bool started = false;
  int32_t cur_dest = -1;
  bool first_group = true;

  auto flush = [&](bool is_final) {
#if !STRATA_SPMM_F64
    absorb(acc, part);
#endif
    if (split && first_group && head_cont) {
      put_f64<L, VEC, kScalar, false>(a.carry + ((P.carry_off + c) * 2 + 0) * d, acc, d, lane, feat0);
    } else if (split && is_final && tail_cont) {
      put_f64<L, VEC, kScalar, false>(a.carry + ((P.carry_off + c) * 2 + 1) * d, acc, d, lane, feat0);
    } else {
      const long long dest = cur_dest;
      if (a.yacc) {  // c > 1: partitions accumulate in f64, rounded once at the end
        put_f64<L, VEC, kScalar, true>(a.yacc + dest * d, acc, d, lane, feat0);
      } else {
        put_row<L, VEC, kScalar>(a.Y.p[0] + dest * d, acc, d, lane, feat0);
        if constexpr (kMulti)  // replicas of the fused all-gather (separate instantiation:
          for (int i = 1; i < a.Y.n; ++i)  // the single-output kernels keep their registers)
            put_row<L, VEC, kScalar>(a.Y.p[i] + dest * d, acc, d, lane, feat0);
      }
    }
    acc.zero();
    first_group = false;
  };

  // A new ELL row starts with output row `dest`: close the previous group if the destination
  // changes (split runs keep accumulating across their segments).
  auto row_start = [&](int32_t dest) {
    if (started && (!split || dest != cur_dest)) flush(false);
    cur_dest = dest;
    started = true;
  };

  // This VW's staging buffer: J, V and the output rows of one piece (3 KB).
  extern __shared__ int4 spmm_smem[];
  int32_t* sJ = reinterpret_cast<int32_t*>(spmm_smem) + (threadIdx.x / L) * (3 * kPiece);
  float* sV = reinterpret_cast<float*>(sJ + kPiece);
  int32_t* sD = sJ + 2 * kPiece;
  const unsigned vmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << ((threadIdx.x & 31) & ~(L - 1)));

  const int s_end = r1 << b;
  int32_t carry_col = -1;  // column of the slot before the current compaction round
  int row = r0 - 1;        // ELL row of the latest row start consumed
  for (int pbase = r0 << b; pbase < s_end; pbase += kPiece) {
    const int np = min(kPiece, s_end - pbase);
    const int nq = ((np + kT - 1) / kT) * (kT / 4);  // 16-byte chunks per array (whole tiles:
                                                     // parts are 8-slot aligned and padded)
    const int row_lo = pbase >> b;
    const int nrow = ((pbase + np - 1) >> b) - row_lo + 1;
    __syncwarp(vmask);  // previous piece fully consumed
    for (int q = lane; q < nq; q += L) {
      tc_cp_async16(sJ + 4 * q, Jp + pbase + 4 * q);
      tc_cp_async16(sV + 4 * q, Vp + pbase + 4 * q);
    }
    for (int q = lane; q < nrow; q += L) ::strata_b200::tc::cp_async4(sD + q, Ip + row_lo + q);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp(vmask);

    // Compaction, in place (an entry only ever moves to a lower index; every lane reads its
    // 8 slots before any lane writes).
    int nreal = 0;
    for (int rb = 0; rb < np; rb += kRound) {
      const int s0 = rb + lane * kT;
      int32_t cc[kT];
      float vv[kT];
      {
        const int4 c0 = reinterpret_cast<const int4*>(sJ + s0)[0];
        const int4 c1 = reinterpret_cast<const int4*>(sJ + s0)[1];
        const float4 v0 = reinterpret_cast<const float4*>(sV + s0)[0];
        const float4 v1 = reinterpret_cast<const float4*>(sV + s0)[1];
        cc[0] = c0.x; cc[1] = c0.y; cc[2] = c0.z; cc[3] = c0.w;
        cc[4] = c1.x; cc[5] = c1.y; cc[6] = c1.z; cc[7] = c1.w;
        vv[0] = v0.x; vv[1] = v0.y; vv[2] = v0.z; vv[3] = v0.w;
        vv[4] = v1.x; vv[5] = v1.y; vv[6] = v1.z; vv[7] = v1.w;
      }
      int32_t prev = __shfl_up_sync(vmask, cc[kT - 1], 1, L);
      if (lane == 0) prev = carry_col;
      unsigned real = 0, rstart = 0;
#pragma unroll
      for (int u = 0; u < kT; ++u) {
        const int g = pbase + s0 + u;
        const bool rs = (g & wmask) == 0;
        const bool in = s0 + u < np;
        if (in && (rs || cc[u] != (u ? cc[u - 1] : prev))) real |= 1u << u;
        if (rs) rstart |= 1u << u;
      }
      const int cnt = __popc(real);
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < L; o <<= 1) {
        const int t = __shfl_up_sync(vmask, incl, o, L);
        if (lane >= o) incl += t;
      }
      const int total = __shfl_sync(vmask, incl, L - 1, L);
      carry_col = __shfl_sync(vmask, cc[kT - 1], L - 1, L);
      int pos = nreal + incl - cnt;
      __syncwarp(vmask);
#pragma unroll
      for (int u = 0; u < kT; ++u)
        if (real & (1u << u)) {
          sJ[pos] = cc[u] | ((rstart >> u) & 1u ? kRowFlag : 0);
          sV[pos] = vv[u];
          ++pos;
        }
      nreal += total;
    }
    __syncwarp(vmask);

    // Consume the real slots, 8 per batch.
    for (int e0 = 0; e0 < nreal; e0 += kT) {
      int32_t col[kT];
      {
        const int4 c0 = reinterpret_cast<const int4*>(sJ + e0)[0];  // broadcast LDS.128
        const int4 c1 = reinterpret_cast<const int4*>(sJ + e0)[1];
        col[0] = c0.x; col[1] = c0.y; col[2] = c0.z; col[3] = c0.w;
        col[4] = c1.x; col[5] = c1.y; col[6] = c1.z; col[7] = c1.w;
      }
      const int n = min(kT, nreal - e0);
      unsigned starts = 0;  // row-start flags; the columns die once the gathers are issued
#pragma unroll
      for (int u = 0; u < kT; ++u) starts |= (col[u] < 0 ? 1u : 0u) << u;
#ifndef STRATA_SPMM_FAST32  // A/B knob: fast path for the d = 128 (L = 32) variant too
#define STRATA_SPMM_FAST32 0
#endif
      // (the L = 32 variant is register-budgeted at 80 for 3 CTAs/SM and DRAM-bound at C5: the
      // fast path's second chain spills there and costs 26 %, so it is L < 32 only)
      if ((L < 32 || STRATA_SPMM_FAST32) && n == kT && starts == 0) {
        // Full batch inside one output row (most batches once rows are longer than a batch):
        // no per-slot predication or row-start branches; two independent FMA chains (even /
        // odd slots) halve the dependent-FMA latency.  part is zero here (absorbed after
        // every batch), and the batch sum (even + odd) is folded into f64 as before.
#if STRATA_SPMM_F64
        Acc<VEC, kScalar> a1;  // odd slots; added to the running sum in a fixed order
        a1.zero();
#pragma unroll
        for (int ub = 0; ub < kT; ub += UG) {
          Frag<VEC, kScalar> xv[UG];
#pragma unroll
          for (int u = 0; u < UG; ++u)
            gather<L, VEC, kScalar>(xv[u], Xg, col[ub + u], d, lane, feat0, a.w256);
#pragma unroll
          for (int u = 0; u < UG; ++u) fma_acc<kUp>((ub + u) & 1 ? a1 : acc, sV[e0 + ub + u], xv[u]);
        }
        add_acc(acc, a1);
#else
        Frag<VEC, kScalar> p1;
        p1.zero();
#pragma unroll
        for (int ub = 0; ub < kT; ub += UG) {
          Frag<VEC, kScalar> xv[UG];
#pragma unroll
          for (int u = 0; u < UG; ++u)
            gather<L, VEC, kScalar>(xv[u], Xg, col[ub + u], d, lane, feat0, a.w256);
#pragma unroll
          for (int u = 0; u < UG; ++u) fma_part((ub + u) & 1 ? p1 : part, sV[e0 + ub + u], xv[u]);
        }
        add_part(part, p1);
        absorb(acc, part);
#endif
        continue;
      }
#pragma unroll
      for (int ub = 0; ub < kT; ub += UG) {
        Frag<VEC, kScalar> xv[UG];
#pragma unroll
        for (int u = 0; u < UG; ++u)
          if (ub + u < n) gather<L, VEC, kScalar>(xv[u], Xg, col[ub + u] & 0x7fffffff, d, lane, feat0, a.w256);
#pragma unroll
        for (int u = 0; u < UG; ++u) {
          const int uu = ub + u;
          if (uu < n) {
            if ((starts >> uu) & 1u) row_start(sD[++row - row_lo]);
#if STRATA_SPMM_F64
            fma_acc<kUp>(acc, sV[e0 + uu], xv[u]);  // broadcast LDS
#else
            fma_part(part, sV[e0 + uu], xv[u]);  // broadcast LDS
#endif
          }
        }
      }
#if !STRATA_SPMM_F64
      absorb(acc, part);
#endif
    }
  }
  if (started) flush(true);
}

// Fix-up of split runs that cross chunk boundaries: a deterministic two-level tree.
//   level 1 (spmm_fixup_tiles_kernel): one CTA per tile of <= kFixTile consecutive carries of
//     one run; G thread groups take contributions g, g+G, ... (8 loads in flight per thread),
//     then the groups are combined in group order.  Runs that fit one tile write Y directly.
//   level 2 (spmm_fixup_runs_kernel): one CTA per longer run sums its tile partials the same
//     way.  Fixed shapes and orders => bitwise reproducible; no atomics.
constexpr int kFixBlock = 128;

// Carries and level-2 partials are f64 (see Acc); only the final store rounds to f32.
// Output: a Y row (f32 store) when yout != nullptr; else an f64 row, stored (level-2 slot) or
// added (`accumulate`: the c > 1 f64 accumulator).
template <int V>  // V = 2: double2 lanes (d even); V = 1: scalar
__device__ __forceinline__ void fix_reduce(const double* __restrict__ src, long long first_row,
                                           int count, int first_slot, bool two_slot,
                                           const YDests* ydst, long long yrow, double* l2out,
                                           long long d, bool accumulate) {
  __shared__ double2 part[kFixBlock];
  const long long dv = d / V;
  const int rt = static_cast<int>(min64(dv, kFixBlock));  // threads per feature row
  const int G = kFixBlock / rt;
  const int g = threadIdx.x / rt;
  for (long long fb = 0; fb < dv; fb += rt) {
    const long long f = fb + threadIdx.x % rt;
    const bool active = g < G && f < dv;
    double2 acc = make_double2(0.0, 0.0);
    if (active) {
      for (int q0 = g; q0 < count; q0 += 8 * G) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int q = q0 + u * G;
          v[u] = make_double2(0.0, 0.0);
          if (q < count) {
            const long long r = two_slot ? (first_row + q) * 2 + (q == 0 ? first_slot : 0)
                                         : first_row + q;
            if constexpr (V == 2) v[u] = reinterpret_cast<const double2*>(src + r * d)[f];
            else v[u].x = src[r * d + f];
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc.x += v[u].x;
          acc.y += v[u].y;
        }
      }
    }
    part[threadIdx.x] = acc;
    __syncthreads();
    if (g == 0 && f < dv) {
      double2 tot = part[threadIdx.x];
      for (int gg = 1; gg < G; ++gg) {
        tot.x += part[gg * rt + threadIdx.x].x;
        tot.y += part[gg * rt + threadIdx.x].y;
      }
      if (ydst) {
        for (int i = 0; i < ydst->n; ++i) {
          float* yout = ydst->p[i] + yrow * d;
          if constexpr (V == 2)
            reinterpret_cast<float2*>(yout)[f] =
                make_float2(static_cast<float>(tot.x), static_cast<float>(tot.y));
          else
            yout[f] = static_cast<float>(tot.x);
        }
      } else {
        if constexpr (V == 2) {
          double2* o = reinterpret_cast<double2*>(l2out) + f;
          if (accumulate) {
            const double2 old = *o;
            tot.x += old.x;
            tot.y += old.y;
          }
          *o = tot;
        } else {
          l2out[f] = accumulate ? l2out[f] + tot.x : tot.x;
        }
      }
    }
    __syncthreads();
  }
}

// yacc != nullptr (c > 1): final rows are added to the f64 accumulator instead of stored to Y.
template <int V>
__global__ void __launch_bounds__(kFixBlock)
spmm_fixup_tiles_kernel(const FixTile* __restrict__ tiles, const double* __restrict__ carry,
                        double* __restrict__ l2, const __grid_constant__ YDests Y,
                        double* __restrict__ yacc, long long d) {
  const FixTile t = tiles[blockIdx.x];
  if (t.out >= 0 && yacc)
    fix_reduce<V>(carry, t.carry0, t.count, t.first_slot, true, nullptr, 0, yacc + t.out * d, d, true);
  else if (t.out >= 0)
    fix_reduce<V>(carry, t.carry0, t.count, t.first_slot, true, &Y, t.out, nullptr, d, false);
  else
    fix_reduce<V>(carry, t.carry0, t.count, t.first_slot, true, nullptr, 0, l2 + (-t.out - 1) * d,
                  d, false);
}

template <int V>
__global__ void __launch_bounds__(kFixBlock)
spmm_fixup_runs_kernel(const FixRun* __restrict__ runs, const double* __restrict__ l2,
                       const __grid_constant__ YDests Y, double* __restrict__ yacc, long long d) {
  const FixRun r = runs[blockIdx.x];
  if (yacc)
    fix_reduce<V>(l2, r.l2_first, r.ntiles, 0, false, nullptr, 0, yacc + r.row * d, d, true);
  else
    fix_reduce<V>(l2, r.l2_first, r.ntiles, 0, false, &Y, r.row, nullptr, d, false);
}

__global__ void f64_to_f32_kernel(const double* __restrict__ in, const __grid_constant__ YDests Y,
                                  long long n) {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < n;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const float v = static_cast<float>(in[e]);
    for (int i = 0; i < Y.n; ++i) Y.p[i][e] = v;
  }
}

__global__ void zero_rows_kernel(const int32_t* __restrict__ rows, long long n,
                                 const __grid_constant__ YDests Y, long long d) {
  const long long total = n * d;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / d, f = e - r * d;
    for (int i = 0; i < Y.n; ++i) Y.p[i][static_cast<long long>(rows[r]) * d + f] = 0.f;
  }
}

// Any inf / NaN among X's n floats -> *flag = 1 (flag zeroed by the caller).  256-bit loads of
// a 32-byte aligned X; one store per warp that saw one.
__global__ void __launch_bounds__(256) x_nonfinite_kernel(const float* __restrict__ X, long long n,
                                                          int* __restrict__ flag) {
  const long long n8 = n / 8;
  bool bad = false;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    uint32_t v[8];
    asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "l"(X + i * 8));
#pragma unroll
    for (int k = 0; k < 8; ++k) bad |= (v[k] & 0x7f800000u) == 0x7f800000u;
  }
  if (blockIdx.x == 0)
    for (long long i = n8 * 8 + threadIdx.x; i < n; i += blockDim.x)
      bad |= (__float_as_uint(X[i]) & 0x7f800000u) == 0x7f800000u;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *flag = 1;
}

template <int L, int VEC, bool kScalar, bool kMulti, int kCvt = 0>
void launch_variant_m(const SpmmArgs& args, long long total_chunks, long long d, cudaStream_t s) {
  const long long threads = total_chunks * L;
  const unsigned blocks = static_cast<unsigned>((threads + kBlock - 1) / kBlock);
  dim3 grid(blocks, kScalar ? static_cast<unsigned>((d + 31) / 32) : 1u);
  constexpr int smem = (kBlock / L) * 3 * kPiece * 4;  // 3 KB staging per virtual warp
  auto* kern = spmm_hyb_kernel<L, VEC, kScalar, kMulti, kCvt>;
  static PerDeviceOnce once;  // per instantiation and device
  once([&] {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
#ifdef STRATA_SPMM_CARVEOUT  // A/B knob: prefer the largest shared-memory carveout
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
#endif
  });
  kern<<<grid, kBlock, smem, s>>>(args);
}

template <int L, int VEC, bool kScalar>
void launch_variant(const SpmmArgs& args, long long total_chunks, long long d, cudaStream_t s) {
  if (args.Y.n > 1) launch_variant_m<L, VEC, kScalar, true>(args, total_chunks, d, s);
  else launch_variant_m<L, VEC, kScalar, false>(args, total_chunks, d, s);
}

}  // namespace

void spmm_hyb_launch(const strata_hyb_impl& h, const float* X, float* const* Ydst, int ndst,
                     int64_t d, cudaStream_t s) {
  if (d <= 0) throw ApiError(STRATA_ERR_USAGE, "spmm: d must be >= 1");
  if (ndst < 1 || ndst > kMaxYDests)
    throw ApiError(STRATA_ERR_USAGE, "spmm: 1 to " + std::to_string(kMaxYDests) + " output buffers");
  YDests Y{};
  Y.n = ndst;
  bool aligned = reinterpret_cast<uintptr_t>(X) % 16 == 0;
  for (int i = 0; i < ndst; ++i) {
    Y.p[i] = Ydst[i];
    aligned = aligned && reinterpret_cast<uintptr_t>(Ydst[i]) % 16 == 0;
  }
  // Variant: lanes per VW (L) and float4s per lane (VEC).
  int L = 32, VEC = 1;
  bool scalar = true;
  if (aligned) {
    // 256-bit slices for d = 64 only with 32-byte aligned X (d = 256 / 512 fall back to two
    // 128-bit loads per slice inside the kernel)
    const bool a32 = reinterpret_cast<uintptr_t>(X) % 32 == 0;
    if (d == 32) { L = 8; scalar = false; }
    else if (d == 64) {
      const int v = (STRATA_SPMM_VEC64 == 2 && a32) ? 2 : 1;
      L = 16 / v; VEC = v; scalar = false;
    } else if (d == 128) {
      const int v = (STRATA_SPMM_VEC128 == 2 && a32) ? 2 : 1;
      L = 32 / v; VEC = v; scalar = false;
    }
    else if (d == 256) { L = 32; VEC = 2; scalar = false; }
    else if (d == 512) { L = 32; VEC = 4; scalar = false; }
  }

  // Per-call scratch from the stream-ordered pool (cached there): split-row carries, level-2
  // partials and, for c > 1, the f64 [rows][d] accumulator the partitions add into (rounded to
  // Y once at the end).  Nothing mutable lives in the handle, so calls on different streams
  // do not share scratch.
  const size_t n_carry = static_cast<size_t>(h.total_chunks_carry) * 2 * d;
  const size_t n_l2 = static_cast<size_t>(h.l2_slots) * d;
  const size_t n_yacc = (h.c > 1 && h.rows > 0) ? static_cast<size_t>(h.rows) * d : 0;
  double* scratch = (n_carry + n_l2 + n_yacc) > 0
                        ? static_cast<double*>(workspace_alloc(sizeof(double) * (n_carry + n_l2 + n_yacc), s))
                        : nullptr;
  double* carry = scratch;
  double* carry_l2 = scratch ? scratch + n_carry : nullptr;
  double* yacc = n_yacc ? scratch + n_carry + n_l2 : nullptr;
  if (yacc) {
    STRATA_CUDA_CHECK(cudaMemsetAsync(yacc, 0, sizeof(double) * n_yacc, s));
  } else if (h.n_empty > 0) {
    const long long total = h.n_empty * d;
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 4096));
    zero_rows_kernel<<<blocks, 256, 0, s>>>(h.empty_rows.p, h.n_empty, Y, d);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }

  // d = 64 in 256-bit slices (L = 8, VEC = 2), one destination, X small enough to stay in L2
  // (the XU-bound case; a DRAM-bound gather gains nothing and the scan would cost X's bytes
  // again): scan X for inf / NaN once per call (~10 us at C2) so the integer-pipe conversion
  // variant can run.
  int* xflag = nullptr;
#if STRATA_SPMM_ICVT
  if (!scalar && L == 8 && VEC == 2 && ndst == 1 && h.cols > 0 &&
      static_cast<long long>(h.cols) * d * 4 <= l2_bytes()) {
    xflag = static_cast<int*>(workspace_alloc(sizeof(int), s));
    STRATA_CUDA_CHECK(cudaMemsetAsync(xflag, 0, sizeof(int), s));
    const long long n = h.cols * d;
    const unsigned blocks = static_cast<unsigned>(std::min<long long>((n / 8 + 255) / 256 + 1, num_sms() * 8ll));
    x_nonfinite_kernel<<<blocks, 256, 0, s>>>(X, n, xflag);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }
#endif

  // One launch (plus the fix-up pair) per column partition, partitions in order.
  size_t pi = 0, fr = 0;
  const bool vec2 = d % 2 == 0;
  while (pi < h.parts.size()) {
    const int part_id = h.parts[pi].partition;
    SpmmArgs args{};
    args.I = h.I.p; args.J = h.J.p; args.V = h.V.p; args.X = X; args.Y = Y;
    args.carry = carry; args.yacc = yacc; args.d = d;
    args.w256 = reinterpret_cast<uintptr_t>(X) % 32 == 0 ? 1 : 0;
    long long chunks = 0;
    int np = 0;
    for (; pi < h.parts.size() && h.parts[pi].partition == part_id; ++pi) {
      const HybPart& P = h.parts[pi];
      if (np >= kMaxParts) throw ApiError(STRATA_ERR_USAGE, "spmm: too many buckets per partition");
      SpmmPartDev& q = args.parts[np++];
      q.slot_off = P.slot_off; q.row_off = P.row_off; q.nrows = P.nrows;
      q.chunk_begin = chunks; q.nchunks = P.nchunks; q.carry_off = P.carry_off;
      q.b = P.bucket; q.rpc_log2 = P.rpc_log2; q.may_split = P.may_split;
      chunks += P.nchunks;
    }
    args.nparts = np;
    args.total_chunks = chunks;
    if (chunks > 0) {
      if (scalar) launch_variant<32, 1, true>(args, chunks, d, s);
      else if (L == 8 && VEC == 1) launch_variant<8, 1, false>(args, chunks, d, s);
#if STRATA_SPMM_VEC64 == 2
      else if (L == 8 && VEC == 2 && xflag) {  // integer-pipe conversions, F2F twin for inf / NaN
        args.xflag = xflag;
        launch_variant_m<8, 2, false, false, 1>(args, chunks, d, s);
        launch_variant_m<8, 2, false, false, 2>(args, chunks, d, s);
      }
      else if (L == 8 && VEC == 2) launch_variant<8, 2, false>(args, chunks, d, s);
#endif
      else if (L == 16 && VEC == 1) launch_variant<16, 1, false>(args, chunks, d, s);
#if STRATA_SPMM_VEC128 == 2
      else if (L == 16 && VEC == 2) launch_variant<16, 2, false>(args, chunks, d, s);
#endif
      else if (VEC == 1) launch_variant<32, 1, false>(args, chunks, d, s);
      else if (VEC == 2) launch_variant<32, 2, false>(args, chunks, d, s);
      else launch_variant<32, 4, false>(args, chunks, d, s);
      STRATA_CUDA_CHECK(cudaGetLastError());
    }
    while (fr < h.fix_ranges.size() && h.fix_ranges[fr].partition < part_id) ++fr;
    if (fr < h.fix_ranges.size() && h.fix_ranges[fr].partition == part_id) {
      const FixRange& R = h.fix_ranges[fr];
      const long long nt = R.tile_end - R.tile_begin, nr = R.run_end - R.run_begin;
      if (nt > 0) {
        if (vec2)
          spmm_fixup_tiles_kernel<2><<<static_cast<unsigned>(nt), kFixBlock, 0, s>>>(
              h.fix_tiles.p + R.tile_begin, carry, carry_l2, Y, yacc, d);
        else
          spmm_fixup_tiles_kernel<1><<<static_cast<unsigned>(nt), kFixBlock, 0, s>>>(
              h.fix_tiles.p + R.tile_begin, carry, carry_l2, Y, yacc, d);
        STRATA_CUDA_CHECK(cudaGetLastError());
      }
      if (nr > 0) {
        if (vec2)
          spmm_fixup_runs_kernel<2><<<static_cast<unsigned>(nr), kFixBlock, 0, s>>>(
              h.fix_runs.p + R.run_begin, carry_l2, Y, yacc, d);
        else
          spmm_fixup_runs_kernel<1><<<static_cast<unsigned>(nr), kFixBlock, 0, s>>>(
              h.fix_runs.p + R.run_begin, carry_l2, Y, yacc, d);
        STRATA_CUDA_CHECK(cudaGetLastError());
      }
    }
  }
  if (yacc) {
    const long long n = h.rows * d;
    f64_to_f32_kernel<<<static_cast<unsigned>(std::min<long long>((n + 255) / 256, 148 * 32)), 256, 0, s>>>(
        yacc, Y, n);
    STRATA_CUDA_CHECK(cudaGetLastError());
  }
  if (scratch) STRATA_CUDA_CHECK(cudaFreeAsync(scratch, s));
  if (xflag) STRATA_CUDA_CHECK(cudaFreeAsync(xflag, s));
}

}  // namespace strata_b200
