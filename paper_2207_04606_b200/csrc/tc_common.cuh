// tc_common.cuh — sm_100a tensor-core plumbing written directly in PTX: tcgen05 (UMMA) MMA
// issue, TMEM alloc / load, UMMA shared-memory descriptors, mbarriers and cp.async.
//
// Operand layouts used by the kernels (SWIZZLE_NONE "interleaved" canonical layouts, in bytes,
// bf16 elements; a "core matrix" is 8 rows x 16 B stored contiguously as 128 B):
//   K-major  (K contiguous):  off(mn, k) = (mn/8)*SBO + (k/8)*LBO + (mn%8)*16 + (k%8)*2
//   MN-major (MN contiguous): off(k, mn) = (mn/8)*SBO + (k/8)*LBO + (k%8)*16 + (mn%8)*2
// with LBO = 128 (consecutive K groups of 8 adjacent) throughout, so one K=16 MMA step
// advances the start address by 256 B for either major-ness.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace strata_b200 {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// UMMA shared-memory descriptor (tcgen05 "matrix descriptor"): start address, leading /
// stride byte offsets (16-byte units), version 1 (sm_100), SWIZZLE_NONE layout.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (Blackwell)
  return d;                             // base_offset 0, lbo_mode 0, layout_type 0 (none)
}

// Same with the 128-byte swizzle layout (what a TMA tensor map with CU_TENSOR_MAP_SWIZZLE_128B
// writes; atoms of 8 rows x 128 B, 16-byte chunk c of row r stored at c ^ (r % 8); the
// atom's base must be 1024-byte aligned).  MN-major: LBO = stride between 128-byte MN atoms,
// SBO = stride between 8-row K groups.
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return make_desc(saddr, lbo, sbo) | (static_cast<uint64_t>(2) << 61);
}

// 64-byte swizzle (CU_TENSOR_MAP_SWIZZLE_64B): atoms of 8 rows x 64 B (512 B, 512-aligned).
// K-major with K <= 32 bf16: SBO = stride between 8-row groups, LBO unused.
__device__ __forceinline__ uint64_t make_desc_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return make_desc(saddr, lbo, sbo) | (static_cast<uint64_t>(4) << 61);
}

// 32-byte swizzle (CU_TENSOR_MAP_SWIZZLE_32B): atoms of 8 rows x 32 B (256 B, 256-aligned).
__device__ __forceinline__ uint64_t make_desc_sw32(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return make_desc(saddr, lbo, sbo) | (static_cast<uint64_t>(6) << 61);
}

// Instruction descriptor, kind::f16 with bf16 inputs and f32 accumulation.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N, bool a_mn_major,
                                                       bool b_mn_major) {
  return (1u << 4)                                   // D format: f32
         | (1u << 7)                                 // A format: bf16
         | (1u << 10)                                // B format: bf16
         | (static_cast<uint32_t>(a_mn_major) << 15) // A major
         | (static_cast<uint32_t>(b_mn_major) << 16) // B major
         | (static_cast<uint32_t>(N >> 3) << 17)     // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);    // M / 16
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by one thread for the whole CTA.
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
      :: "r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)));
}

// Arrive on an mbarrier once every previously issued tcgen05.mma of this thread completes.
__device__ __forceinline__ void mma_commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
               :: "r"(smem_u32(mbar)) : "memory");
}

__device__ __forceinline__ void fence_before_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void fence_after_sync() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}

// Generic-proxy smem writes (st.shared / cp.async) -> visible to the async proxy (UMMA reads).
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// TMEM allocation: executed by one full warp; writes the base address to *slot (smem).
template <int kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* slot) {
  static_assert(kCols >= 32 && (kCols & (kCols - 1)) == 0 && kCols <= 512, "bad TMEM cols");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
               :: "r"(smem_u32(slot)), "n"(kCols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
template <int kCols>
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n"
               :: "r"(base), "n"(kCols) : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread t of the warp gets lane (base lane + t).
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// 32 lanes x 16 / 8 consecutive 32-bit columns (same lane mapping as the x32 form).
__device__ __forceinline__ void tmem_ld_32x32b_x16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_32x32b_x8(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
}
template <int N>
__device__ __forceinline__ void tmem_ld_32x32b(uint32_t taddr, uint32_t* r) {
  static_assert(N == 8 || N == 16 || N == 32, "tmem_ld_32x32b: N in {8, 16, 32}");
  if constexpr (N == 32) {
    tmem_ld_32x32b_x32(taddr, *reinterpret_cast<uint32_t(*)[32]>(r));
  } else if constexpr (N == 16) {
    tmem_ld_32x32b_x16(taddr, r);
  } else {
    tmem_ld_32x32b_x8(taddr, r);
  }
}
__device__ __forceinline__ void tmem_ld_wait() {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_u32(mbar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
// try_wait with a suspend-time hint: a waiting thread is parked until the phase completes (or
// the hint expires) instead of re-issuing try_wait + branch.  Without the hint the waits of the
// warp-specialised RGMS pass spun ~100M times per launch at C4 — 40 % of all issued warp
// instructions, taken from the epilogue warps sharing the SM sub-partitions.
#ifndef STRATA_MBAR_SUSPEND_NS  // A/B knob; 0 = no hint
#define STRATA_MBAR_SUSPEND_NS 0x989680
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* mbar, uint32_t parity) {
#if STRATA_MBAR_SUSPEND_NS
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1, %2;\n\t"
      "@!done bra WAIT_%=;\n\t}\n"
      :: "r"(smem_u32(mbar)), "r"(parity), "n"(STRATA_MBAR_SUSPEND_NS) : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n\t}\n"
      :: "r"(smem_u32(mbar)), "r"(parity) : "memory");
#endif
}

// 16-byte asynchronous global -> shared copy (L1-bypassing).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
// 4-byte asynchronous global -> shared copy (L1-allocating form required for sizes < 16).
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" :: "r"(smem_u32(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" :: "n"(N) : "memory");
}

// ---- TMA / bulk async copies completing on an mbarrier (byte-counted) -----------------
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n"
               :: "r"(smem_u32(mbar)), "r"(bytes) : "memory");
}
// 1D bulk copy global -> shared (size multiple of 16, both 16-byte aligned).
__device__ __forceinline__ void bulk_copy_g2s(void* smem, const void* gmem, uint32_t bytes,
                                              uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      :: "r"(smem_u32(smem)), "l"(gmem), "r"(bytes), "r"(smem_u32(mbar)) : "memory");
}
// 2D TMA tile load (tensor map in param / const / global space), coordinates innermost first.
__device__ __forceinline__ void tma_load_2d(void* smem, const void* tmap, int c0, int c1,
                                            uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n"
      :: "r"(smem_u32(smem)), "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(mbar)) : "memory");
}
// TMA tile::gather4: rows r0..r3 (each one box of the 2D map, box height 1) of column c0 land
// consecutively at smem (swizzled by address like a 4-row box).
__device__ __forceinline__ void tma_gather4(void* smem, const void* tmap, int c0, int r0, int r1,
                                            int r2, int r3, uint64_t* mbar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];\n"
      :: "r"(smem_u32(smem)), "l"(tmap), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
         "r"(smem_u32(mbar)) : "memory");
}
// Arrive on an mbarrier once all prior cp.async of this thread complete (counts as one of the
// barrier's expected arrivals: .noinc).
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* mbar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" :: "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* mbar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(smem_u32(mbar)) : "memory");
}
__device__ __forceinline__ void prefetch_tensormap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" :: "l"(tmap) : "memory");
}

// Programmatic dependent launch (launched with cudaLaunchAttributeProgrammaticStreamSerialization):
// pdl_wait() blocks until the preceding grid on the stream has completed and its memory is
// visible — call it before the first global read of anything that grid may have written;
// pdl_launch() lets the next grid start its prologue (TMEM alloc, barrier init) early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// Vector reduction into global memory (sm_90+): 4 consecutive f32 added atomically.
__device__ __forceinline__ void red_add_v4(float* gaddr, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};\n"
               :: "l"(gaddr), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

}  // namespace tc
}  // namespace strata_b200
