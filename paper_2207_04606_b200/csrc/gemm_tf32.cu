// gemm_tf32.cu — the dense transform of the GNN layer step (Z = Y · W, fp32 in and out) on the
// sm_100a tensor cores: tcgen05.mma kind::tf32 with the 3xTF32 split, so the result keeps fp32
// accuracy (the north_star's 1e-5 bar) while the MMAs run on the tensor pipe.
//
// Split: a = a_hi + a_lo with a_hi = a rounded to nearest tf32 (10 explicit mantissa bits) and
// a_lo = a - a_hi (exact in f32, |a_lo| <= half a tf32 ulp, so its own tf32 rounding costs at
// most 2^-22 of a); likewise w.  The dropped a_lo·w_lo term is 2^-22 of a product.
// Accumulation: the tensor core rounds its f32 accumulator towards zero once per MMA, so one
// 3·K/8-long chain per output would cost up to 3·K/8 ulps (measured 3-7e-5 on N(0,1)·30 data).
// Instead every 64-wide K chunk gets its own TMEM accumulator: the chunk's small products
// (a_lo·w_hi + a_hi·w_lo, 2^-11 of the magnitude) go in first, while that accumulator is still
// small, then its 8 big products a_hi·w_hi; the epilogue adds the chunk accumulators in f32
// with round-to-nearest — the error of an f32 SGEMM (measured at or below it), not worse.
// On integer operands below 2^22 the split is exact and every partial sum an exact integer, so
// integer data gives exact sums.
//
// Shape: Z[M][N] = Y[M][K] · W[K][N], row-major.  One CTA per SM (persistent), 128-row tiles:
//   warp 0 / lane 0   TMA producer: per tile, K/32 boxes {32 k, 128 rows} of Y (128-byte
//                     swizzle = the K-major SW128 A operand) into a ring of stages;
//   warps 6-9         split: a_hi in place, a_lo into the stage's second buffer (the same
//                     swizzled offsets — the split is elementwise), fence.proxy.async, arrive;
//   warp 1 / lane 0   MMA issuer: 3 x (K/8) tcgen05.mma M = 128, N = Nt, K = 8 per tile into
//                     one of two TMEM accumulator sets, commit -> stage free / set full;
//   warps 2-5         epilogue: tcgen05.ld (TMEM lane quarter = warp % 4) -> Z rows.
// W's N-tile [K][Nt] is split once per CTA into W_hi / W_lo and kept in shared memory as the
// K-major SW128 B operand for the whole kernel.  Y is read once, Z written once: HBM-bound
// (M·(K + N)·4 bytes) whenever K·N ≤ ~16 K (C5 128→128: 2.5 GB, 0.38 ms at the copy peak).
#include <algorithm>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

namespace strata_b200 {
namespace {

constexpr int kBM = 128;             // rows per tile (UMMA M, TMEM lanes)
constexpr int kKB = 32;              // k per stage (one 128-byte swizzle atom row of f32)
constexpr int kStageBytes = kBM * kKB * 4;  // 16 KB raw/hi + 16 KB lo per stage
constexpr int kThreads = 320;        // 10 warps
constexpr int kMaxStages = 6;
constexpr uint32_t kHiMask = 0xFFFFE000u;  // tf32: 10 explicit mantissa bits
constexpr int kChunkK = 64;                // K per big-product accumulator
#ifndef STRATA_GEMM_EPI32  // A/B knob: 32-column epilogue steps, both K chunks loaded per wait
#define STRATA_GEMM_EPI32 0
#endif
#ifndef STRATA_GEMM_ST256  // A/B knob: 256-bit epilogue stores (when Z is 32-byte aligned)
#define STRATA_GEMM_ST256 1
#endif
#ifndef STRATA_GEMM_MIN_STAGES  // A/B knob: pipeline stages the N tile must leave room for
#define STRATA_GEMM_MIN_STAGES 2    // (4 at C5 128->128 = two N tiles, Y read twice: 0.74 -> 1.07 ms)
#endif

// f32 -> (nearest tf32, exact f32 remainder).  Rounding half away from zero in magnitude; a
// carry into the exponent is still exact (the remainder absorbs it).
__device__ __forceinline__ uint32_t tf32_rn(uint32_t u) { return (u + 0x1000u) & kHiMask; }

__host__ __device__ constexpr uint32_t make_idesc_tf32(int M, int N) {
  return (1u << 4)                                // D format: f32
         | (2u << 7)                              // A format: tf32
         | (2u << 10)                             // B format: tf32
         | (static_cast<uint32_t>(N >> 3) << 17)  // N / 8 (A and B K-major)
         | (static_cast<uint32_t>(M >> 4) << 24); // M / 16
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}

// Byte offset of element (row, k) of a K-major SW128 operand whose K is cut into 32-element
// blocks of `rows` x 128 B: 8-row atoms of 1 KB, 16-byte chunk c of row r stored at c ^ (r % 8).
__device__ __forceinline__ uint32_t sw128_off(int row, int k, int rows) {
  const int kb = k >> 5, w = k & 31, r = row & 7;
  return static_cast<uint32_t>(kb * rows * 128 + (row >> 3) * 1024 + r * 128 +
                               (((w >> 2) ^ r) << 4) + (w & 3) * 4);
}

struct GemmArgs {
  const float* W;  // [K][N]
  float* Z;        // [M][N]
  long long M;
  int K, N, Nt, stages;
  int st256;  // Z 32-byte aligned: 256-bit epilogue stores
};

__global__ void __launch_bounds__(kThreads, 1)
gemm_tf32x3_kernel(const __grid_constant__ CUtensorMap ymap, const __grid_constant__ GemmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  __shared__ uint64_t full[kMaxStages], split[kMaxStages], empty[kMaxStages];
  __shared__ uint64_t acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_slot;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int K = a.K, N = a.N, Nt = a.Nt, S = a.stages;
  const int n0 = blockIdx.y * Nt;
  const int nt = min(Nt, N - n0);  // this CTA's N tile (multiple of 16)
  const int kblocks = K / kKB;
  const long long tiles = (a.M + kBM - 1) / kBM;
  const uint32_t wbytes = static_cast<uint32_t>(K) * Nt * 4;
  uint8_t* w_hi = smem;
  uint8_t* w_lo = smem + wbytes;
  uint8_t* stages = smem + 2 * wbytes;
  // TMEM: two accumulator sets (double buffer) of nchunk accumulators of Nt columns each (K
  // chunk c at column c*Nt).
  const int nchunk = (K + kChunkK - 1) / kChunkK;
  int tcols = 32;
  while (tcols < 2 * nchunk * Nt) tcols <<= 1;
  const uint32_t acc_stride = static_cast<uint32_t>(tcols / 2);  // accumulator set 1 offset
  if (warp == 1) {
    switch (tcols) {  // tcgen05.alloc takes an immediate column count
      case 32: tc::tmem_alloc<32>(&tmem_slot); break;
      case 64: tc::tmem_alloc<64>(&tmem_slot); break;
      case 128: tc::tmem_alloc<128>(&tmem_slot); break;
      case 256: tc::tmem_alloc<256>(&tmem_slot); break;
      default: tc::tmem_alloc<512>(&tmem_slot); break;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&split[s], 128);
      tc::mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 4);
    }
    tc::mbar_fence_init();
    tc::prefetch_tensormap(&ymap);
  }
  // W's N tile -> W_hi / W_lo, K-major SW128 (row = n, k contiguous); columns >= nt are zero.
  for (int e = tid; e < K * Nt; e += kThreads) {
    const int k = e / Nt, n = e - k * Nt;
    const float w = n < nt ? __ldg(a.W + static_cast<long long>(k) * N + n0 + n) : 0.f;
    const float hi = __uint_as_float(tf32_rn(__float_as_uint(w)));
    const uint32_t off = sw128_off(n, k, Nt);
    *reinterpret_cast<float*>(w_hi + off) = hi;
    *reinterpret_cast<float*>(w_lo + off) = w - hi;
  }
  tc::fence_proxy_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      long long g = 0;
      for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int j = 0; j < kblocks; ++j, ++g) {
          const int s = static_cast<int>(g % S);
          if (g >= S) tc::mbar_wait(&empty[s], static_cast<uint32_t>((g / S - 1) & 1));
          uint8_t* st = stages + s * (2 * kStageBytes);
          tc::mbar_arrive_expect_tx(&full[s], kStageBytes);
          tc::tma_load_2d(st, &ymap, j * kKB, static_cast<int>(t * kBM), &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      const uint32_t idesc = make_idesc_tf32(kBM, Nt);
      const uint32_t whi = tc::smem_u32(w_hi), wlo = tc::smem_u32(w_lo);
      long long g = 0, i = 0;
      for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
        const int acc = static_cast<int>(i & 1);
        if (i >= 2) tc::mbar_wait(&acc_empty[acc], static_cast<uint32_t>((i / 2 - 1) & 1));
        tc::fence_after_sync();
        const uint32_t d = tmem + acc * acc_stride;
        // Per 64-wide K chunk (<= 2 stages): its small products first, while the chunk's
        // accumulator is still small (truncation relative to that magnitude), then its 8 big
        // products — so each chain carries only kChunkK/8 truncations at full magnitude.
        for (int j0 = 0; j0 < kblocks; j0 += kChunkK / kKB) {
          const int nb = min(kChunkK / kKB, kblocks - j0);
          const uint32_t dch = d + static_cast<uint32_t>((j0 * kKB / kChunkK) * Nt);
          for (int pass = 0; pass < 2; ++pass) {
            for (int jj = 0; jj < nb; ++jj) {
              const int j = j0 + jj;
              const long long gj = g + jj;
              const int s = static_cast<int>(gj % S);
              if (pass == 0) {
                tc::mbar_wait(&split[s], static_cast<uint32_t>((gj / S) & 1));
                tc::fence_after_sync();
              }
              const uint32_t ahi = tc::smem_u32(stages + s * (2 * kStageBytes));
              const uint32_t alo = ahi + kStageBytes;
              const uint32_t wb = static_cast<uint32_t>(j) * Nt * 128;
#pragma unroll
              for (int ks = 0; ks < kKB / 8; ++ks) {  // K = 8 per MMA: +32 B in the swizzled row
                const uint64_t dah = tc::make_desc_sw128(ahi + ks * 32, 0, 1024);
                const uint64_t dwh = tc::make_desc_sw128(whi + wb + ks * 32, 0, 1024);
                if (pass == 0) {
                  const uint64_t dal = tc::make_desc_sw128(alo + ks * 32, 0, 1024);
                  const uint64_t dwl = tc::make_desc_sw128(wlo + wb + ks * 32, 0, 1024);
                  mma_tf32(dch, dal, dwh, idesc, jj > 0 || ks > 0);
                  mma_tf32(dch, dah, dwl, idesc, true);
                } else {
                  mma_tf32(dch, dah, dwh, idesc, true);
                }
              }
              if (pass == 1) tc::mma_commit(&empty[s]);
            }
          }
          g += nb;
        }
        tc::mma_commit(&acc_full[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 6) {  // split warps: a_hi in place, a_lo alongside
    const int st_id = tid - 192;
    long long g = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int j = 0; j < kblocks; ++j, ++g) {
        const int s = static_cast<int>(g % S);
        tc::mbar_wait(&full[s], static_cast<uint32_t>((g / S) & 1));
        uint8_t* hi = stages + s * (2 * kStageBytes);
        uint8_t* lo = hi + kStageBytes;
#pragma unroll
        for (int q = 0; q < kStageBytes / 16 / 128; ++q) {
          const int off = (q * 128 + st_id) * 16;
          uint4 v = *reinterpret_cast<const uint4*>(hi + off);
          const uint4 h = make_uint4(tf32_rn(v.x), tf32_rn(v.y), tf32_rn(v.z), tf32_rn(v.w));
          const float4 l = make_float4(__uint_as_float(v.x) - __uint_as_float(h.x),
                                       __uint_as_float(v.y) - __uint_as_float(h.y),
                                       __uint_as_float(v.z) - __uint_as_float(h.z),
                                       __uint_as_float(v.w) - __uint_as_float(h.w));
          *reinterpret_cast<uint4*>(hi + off) = h;
          *reinterpret_cast<float4*>(lo + off) = l;
        }
        tc::fence_proxy_async();
        tc::mbar_arrive(&split[s]);
      }
    }
  } else {  // warps 2-5: epilogue, TMEM lane quarter warp % 4
    const int quarter = warp & 3;
    long long i = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x, ++i) {
      const int acc = static_cast<int>(i & 1);
      tc::mbar_wait(&acc_full[acc], static_cast<uint32_t>((i / 2) & 1));
      tc::fence_after_sync();
      const long long row = t * kBM + quarter * 32 + lane;
      float* zr = a.Z + row * N + n0;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) + acc * acc_stride;
#if STRATA_GEMM_ST256 && STRATA_GEMM_EPI32
      // Two K chunks, 32 columns per step: both chunks' TMEM loads in flight, one wait, then
      // four 256-bit stores (same f32 sum order as the general path below).
      if (nchunk == 2 && nt % 32 == 0 && a.st256) {
        for (int c = 0; c < nt; c += 32) {
          uint32_t r0[32], r1[32];
          tc::tmem_ld_32x32b_x32(taddr + static_cast<uint32_t>(c), r0);
          tc::tmem_ld_32x32b_x32(taddr + static_cast<uint32_t>(Nt + c), r1);
          tc::tmem_ld_wait();
          float z[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) z[q] = __uint_as_float(r0[q]) + __uint_as_float(r1[q]);
          if (c + 32 >= nt) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&acc_empty[acc]);
          }
          if (row < a.M) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                           ::"l"(zr + c + 8 * q), "f"(z[8 * q]), "f"(z[8 * q + 1]), "f"(z[8 * q + 2]),
                             "f"(z[8 * q + 3]), "f"(z[8 * q + 4]), "f"(z[8 * q + 5]), "f"(z[8 * q + 6]),
                             "f"(z[8 * q + 7])
                           : "memory");
          }
        }
        continue;
      }
#endif
      for (int c = 0; c < nt; c += 16) {
        uint32_t r[16];
        float z[16];
        tc::tmem_ld_32x32b_x16(taddr + static_cast<uint32_t>(c), r);
        tc::tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 16; ++q) z[q] = __uint_as_float(r[q]);
        for (int ch = 1; ch < nchunk; ++ch) {  // + the other chunks in K order (f32, nearest)
          tc::tmem_ld_32x32b_x16(taddr + static_cast<uint32_t>(ch * Nt + c), r);
          tc::tmem_ld_wait();
#pragma unroll
          for (int q = 0; q < 16; ++q) z[q] += __uint_as_float(r[q]);
        }
        if (c + 16 >= nt) {  // accumulator set drained: release it before the stores
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&acc_empty[acc]);
        }
        if (row < a.M) {
#if STRATA_GEMM_ST256
          // 256-bit stores (sm_100 STG.256): each lane writes whole 32-byte sectors of its row
          // (the 16-byte form left every warp store 32 half-sectors: 0.74 -> 0.57 ms at C5)
          if (a.st256) {
#pragma unroll
          for (int q = 0; q < 2; ++q)
            asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
                         ::"l"(zr + c + 8 * q), "f"(z[8 * q]), "f"(z[8 * q + 1]), "f"(z[8 * q + 2]),
                           "f"(z[8 * q + 3]), "f"(z[8 * q + 4]), "f"(z[8 * q + 5]), "f"(z[8 * q + 6]),
                           "f"(z[8 * q + 7])
                         : "memory");
          } else
#endif
          {
          float4* zp = reinterpret_cast<float4*>(zr + c);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            st_stream4(zp + q, make_float4(z[4 * q], z[4 * q + 1], z[4 * q + 2], z[4 * q + 3]));
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    switch (tcols) {
      case 32: tc::tmem_dealloc<32>(tmem); break;
      case 64: tc::tmem_dealloc<64>(tmem); break;
      case 128: tc::tmem_dealloc<128>(tmem); break;
      case 256: tc::tmem_dealloc<256>(tmem); break;
      default: tc::tmem_dealloc<512>(tmem); break;
    }
  }
}

// Shapes the tensor-core kernel does not take (K % 32 != 0, N % 16 != 0, or a W tile that does
// not fit shared memory): one thread per output, exact f32 products summed in f64.
__global__ void gemm_f64acc_kernel(const float* __restrict__ Y, const float* __restrict__ W,
                                   float* __restrict__ Z, long long M, int K, int N) {
  const long long total = M * N;
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long m = e / N;
    const int n = static_cast<int>(e - m * N);
    double s = 0.0;
    for (int k = 0; k < K; ++k)
      s = fma(static_cast<double>(Y[m * K + k]), static_cast<double>(__ldg(W + static_cast<long long>(k) * N + n)), s);
    Z[e] = static_cast<float>(s);
  }
}

CUtensorMap make_tensor_map_f32_2d(const void* base, long long rows, long long cols, int box_cols,
                                   int box_rows) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    STRATA_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
      throw ApiError(STRATA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  CUtensorMap map;
  const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(cols) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estride[2] = {1, 1};
  const CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim,
                            gstride, box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ApiError(STRATA_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return map;
}

constexpr int kSmemLimit = 232448;  // 227 KB opt-in per block
constexpr int kSmemStatic = 1024;   // barriers + TMEM slot (+ alignment slack below)

}  // namespace

// N tile for the tensor-core path: both accumulator sets (K/64 * Nt columns each) fit the
// 512 TMEM columns, and W_hi + W_lo (8·K·Nt bytes) plus >= 2 stages fit shared memory.
int gemm_tf32_tile_n(int K, int N) {
  if (K < kKB || K % kKB != 0 || N < 16 || N % 16 != 0) return 0;
  const int nchunk = (K + kChunkK - 1) / kChunkK;
  const int budget = kSmemLimit - 1024 - kSmemStatic - STRATA_GEMM_MIN_STAGES * 2 * kStageBytes;
  int nt = std::min({256 / nchunk, budget / (8 * K)}) / 16 * 16;
  if (nt < 16) return 0;
  nt = std::min(nt, N);
  // balance the N tiles (each a multiple of 16)
  const int ntiles = (N + nt - 1) / nt;
  nt = ((N + ntiles - 1) / ntiles + 15) / 16 * 16;
  return nt;
}

void gemm_f32_launch(const float* Y, const float* W, float* Z, long long M, int K, int N,
                     cudaStream_t s) {
  if (M == 0 || N == 0) return;
  const int nt = gemm_tf32_tile_n(K, N);
  if (nt == 0) {
    const long long total = M * N;
    const unsigned grid = static_cast<unsigned>(std::min<long long>((total + 255) / 256, 148LL * 16));
    gemm_f64acc_kernel<<<grid, 256, 0, s>>>(Y, W, Z, M, K, N);
    STRATA_CUDA_CHECK(cudaGetLastError());
    return;
  }
  const int wbytes = 8 * K * nt;
  const int stages = std::min(kMaxStages, (kSmemLimit - 1024 - kSmemStatic - wbytes) / (2 * kStageBytes));
  const int smem = wbytes + stages * 2 * kStageBytes + 1024;
  static PerDeviceOnce once;
  once([&] {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(gemm_tf32x3_kernel,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit - kSmemStatic));
  });
  const CUtensorMap ymap = make_tensor_map_f32_2d(Y, M, K, kKB, kBM);
  GemmArgs a{W, Z, M, K, N, nt, stages, reinterpret_cast<uintptr_t>(Z) % 32 == 0 ? 1 : 0};
  const long long tiles = (M + kBM - 1) / kBM;
  const int ntiles = (N + nt - 1) / nt;
  const long long per_y = std::max<long long>(1, num_sms() / ntiles);
  dim3 grid(static_cast<unsigned>(std::min<long long>(tiles, per_y)), static_cast<unsigned>(ntiles));
  gemm_tf32x3_kernel<<<grid, kThreads, smem, s>>>(ymap, a);
  STRATA_CUDA_CHECK(cudaGetLastError());
}

}  // namespace strata_b200
