// bsr_sddmm.cu — block-sparse SDDMM on tcgen05 tensor cores: the score half of sparse attention
// (batched SDDMM of sparse transformers; the reference's SDDMM is the CSR nest of
// kernels.cpp:110-136 — here on the BSR pattern, SURVEY §8f item 2 "multi-head batched BSR
// SpMM/SDDMM").
//
//   S_h[q][blk][ii][ji] = A_bsr[q][ii][ji] * sum_f Q_h[br*32 + ii][f] * K_h[JO[q]*32 + ji][f]
//
// for every stored block q of block row br, per head h.  One CTA per (block row, head): the
// block row's Q tile (32 x d) is loaded once and reused as the B operand; the stored blocks'
// K tiles arrive four at a time (four TMA boxes {64 features x 32 rows}, 128-byte swizzle) as the
// 128-row A operand, so one tcgen05.mma computes D[128 keys][32 queries] = four blocks at once
// (M = 128, N = 32, K = d in K16 steps).  A producer thread streams key groups through an
// mbarrier ring; the MMA thread double-buffers the TMEM accumulator; warp w of the epilogue
// owns block w of the group (TMEM lanes 32w..32w+31 = that block's keys) and writes
// S[blk][ii][ji] = A * D[ji][ii] with one coalesced 128-byte row per instruction.
#include <algorithm>
#include <cuda_bf16.h>

#include "capi_internal.h"
#include "common.cuh"
#include "tc_common.cuh"

using namespace strata_b200;

namespace {

constexpr int kB = 32, kGroup = 4, kStages = 4, kThreads = 192;  // warp 0 producer, 1 MMA, 2-5 epilogue

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
bsr_sddmm_tc_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                    const int32_t* __restrict__ jo_indptr, const int32_t* __restrict__ jo_indices,
                    const float* __restrict__ avals, long long nblocks, long long q_rows,
                    long long k_rows, float* __restrict__ S) {
  constexpr int kAtoms = D / 64;                 // 64-feature (128-byte) swizzle atoms
  constexpr int kKT = kGroup * kB * D * 2;       // four key blocks (A operand)
  constexpr int kQT = kB * D * 2;                // the query tile (B operand)
  constexpr uint32_t kIdesc = tc::make_idesc_bf16(kGroup * kB, kB, /*A K-major*/ false, /*B K-major*/ false);
  static_assert(D == 64 || D == 128, "d must be 64 or 128");

  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (tc::smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sQ = smem + kStages * kKT;
  __shared__ uint64_t full[kStages], empty[kStages], qbar, acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long br = blockIdx.x, head = blockIdx.y;
  // Prologue that touches no input (overlaps the previous kernel under PDL).
  if (warp == 0) tc::tmem_alloc<64>(&tmem_slot);
  if (threadIdx.x == 32) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&qbar, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&acc_full[i], 1);
      tc::mbar_init(&acc_empty[i], 4);
    }
    tc::mbar_fence_init();
  }
  if (threadIdx.x == 64) {
    tc::prefetch_tensormap(&qmap);
    tc::prefetch_tensormap(&kmap);
  }
  tc::pdl_wait();  // inputs (Q, K, structure) may come from the previous kernel
  const int q0 = jo_indptr[br], nblk = jo_indptr[br + 1] - q0;
  const int ngroups = (nblk + kGroup - 1) / kGroup;
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  tc::pdl_launch();
  const uint32_t tmem = tmem_slot;

  if (warp == 0) {
    if (lane == 0 && ngroups > 0) {  // producer
      tc::mbar_arrive_expect_tx(&qbar, kQT);
      for (int a = 0; a < kAtoms; ++a)
        tc::tma_load_2d(sQ + a * (kB * 128), &qmap, a * 64, static_cast<int>(head * q_rows + br * kB), &qbar);
      for (int g = 0; g < ngroups; ++g) {
        const int s = g % kStages;
        if (g >= kStages) tc::mbar_wait(&empty[s], ((g / kStages) - 1) & 1);
        const int nb = min(kGroup, nblk - g * kGroup);
        uint8_t* sK = smem + s * kKT;
        tc::mbar_arrive_expect_tx(&full[s], nb * kB * D * 2);
        for (int b = 0; b < nb; ++b) {
          const int col = jo_indices[q0 + g * kGroup + b];
          for (int a = 0; a < kAtoms; ++a)  // block b = rows 32b..32b+31 of atom column a
            tc::tma_load_2d(sK + a * (kGroup * kB * 128) + b * (kB * 128), &kmap, a * 64,
                            static_cast<int>(head * k_rows + col * kB), &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && ngroups > 0) {  // MMA issuer
      tc::mbar_wait(&qbar, 0);
      for (int g = 0; g < ngroups; ++g) {
        const int s = g % kStages, bsel = g & 1;
        tc::mbar_wait(&full[s], (g / kStages) & 1);
        if (g >= 2) tc::mbar_wait(&acc_empty[bsel], ((g / 2) - 1) & 1);
        tc::fence_after_sync();
        const uint32_t ka = tc::smem_u32(smem + s * kKT), qa = tc::smem_u32(sQ);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          // K-major SW128: 8-row groups 1 KB apart; 16 features = 32 B inside the swizzled row;
          // the next 64-feature atom column starts a whole tile later.
          const uint32_t aoff = (kk / 4) * (kGroup * kB * 128) + (kk % 4) * 32;
          const uint32_t boff = (kk / 4) * (kB * 128) + (kk % 4) * 32;
          tc::mma_bf16(tmem + bsel * 32, tc::make_desc_sw128(ka + aoff, 0, 1024),
                       tc::make_desc_sw128(qa + boff, 0, 1024), kIdesc, kk > 0);
        }
        tc::mma_commit(&empty[s]);
        tc::mma_commit(&acc_full[bsel]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warp w (w % 4 = its TMEM lane quarter) owns block (w % 4) of each group
    const int qtr = warp & 3;
    for (int g = 0; g < ngroups; ++g) {
      const int bsel = g & 1;
      tc::mbar_wait(&acc_full[bsel], (g / 2) & 1);
      tc::fence_after_sync();
      uint32_t v[32];
      tc::tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(qtr * 32) << 16) + bsel * 32, v);
      tc::tmem_ld_wait();
      const int b = g * kGroup + qtr;  // block index inside the block row
      if (b < nblk) {
        const long long blk = q0 + b;
        const float* a = avals + blk * (kB * kB);
        float* out = S + (head * nblocks + blk) * (kB * kB);
        // thread = key ji (= lane); v[ii] = D[ji][ii]: for each query row ii one 128-byte row
#pragma unroll
        for (int ii = 0; ii < kB; ++ii)
          __stcs(out + ii * kB + lane, __ldg(a + ii * kB + lane) * __uint_as_float(v[ii]));
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[bsel]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc<64>(tmem);
}

template <int D>
void launch_sddmm(const strata_bsr& h, const __nv_bfloat16* Q, const __nv_bfloat16* K,
                  long long heads, float* S, cudaStream_t s) {
  constexpr int smem = kStages * kGroup * kB * D * 2 + kB * D * 2 + 1024;
  static PerDeviceOnce once;
  once([&] {
    STRATA_CUDA_CHECK(cudaFuncSetAttribute(bsr_sddmm_tc_kernel<D>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  const long long q_rows = h.mb * kB, k_rows = h.nb * kB;
  const CUtensorMap qmap = make_tensor_map_bf16_2d(Q, heads * q_rows, D, 64, kB, CU_TENSOR_MAP_SWIZZLE_128B);
  const CUtensorMap kmap = make_tensor_map_bf16_2d(K, heads * k_rows, D, 64, kB, CU_TENSOR_MAP_SWIZZLE_128B);
  // Programmatic dependent launch, as the BSR SpMM (bsr.cu): the prologue overlaps the
  // previous kernel; no input is read before griddepcontrol.wait.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(h.mb), static_cast<unsigned>(heads));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  STRATA_CUDA_CHECK(cudaLaunchKernelEx(&cfg, bsr_sddmm_tc_kernel<D>, qmap, kmap,
                                       static_cast<const int32_t*>(h.indptr.p),
                                       static_cast<const int32_t*>(h.indices.p),
                                       static_cast<const float*>(h.values.p),
                                       static_cast<long long>(h.nblocks), q_rows, k_rows, S));
}

}  // namespace

extern "C" int strata_bsr_sddmm_bf16(const strata_bsr* h, const void* Q_bf16, const void* K_bf16,
                                     float* S, int64_t heads, int64_t d, void* stream) {
  try {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null bsr handle");
    if (h->b != kB) throw ApiError(STRATA_ERR_USAGE, "bsr_sddmm_bf16: tensor-core path needs b == 32");
    if (d != 64 && d != 128) throw ApiError(STRATA_ERR_USAGE, "bsr_sddmm_bf16: d must be 64 or 128");
    if (heads < 1 || heads > 65535) throw ApiError(STRATA_ERR_USAGE, "bsr_sddmm_bf16: heads must be in [1, 65535]");
    if (h->mb == 0 || h->nblocks == 0) return STRATA_OK;
    int dev = 0, major = 0;
    STRATA_CUDA_CHECK(cudaGetDevice(&dev));
    STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const auto* Q = static_cast<const __nv_bfloat16*>(Q_bf16);
    const auto* K = static_cast<const __nv_bfloat16*>(K_bf16);
    if (d == 64) launch_sddmm<64>(*h, Q, K, heads, S, s);
    else launch_sddmm<128>(*h, Q, K, heads, S, s);
    return STRATA_OK;
  } catch (const ApiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return STRATA_ERR_INTERNAL;
  }
}
