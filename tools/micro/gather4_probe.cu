// Development probe: semantics of TMA tile::gather4 on sm_100a (box shape, smem placement,
// 64-byte swizzle).  nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap map, const int* rows, uint16_t* out) {
  __shared__ __align__(1024) uint16_t buf[8 * 32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar)), "r"(512) : "memory");
    for (int h = 0; h < 2; ++h)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
          "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
          :: "r"(smem_u32(buf + h * 128)), "l"(&map), "r"(0), "r"(rows[4 * h]), "r"(rows[4 * h + 1]),
             "r"(rows[4 * h + 2]), "r"(rows[4 * h + 3]), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" :: "r"(smem_u32(&bar)) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int n = 1000, cols = 32;
  std::vector<uint16_t> hx(n * cols);
  for (int r = 0; r < n; ++r) for (int c = 0; c < cols; ++c) hx[r * cols + c] = static_cast<uint16_t>(r * 64 + c);
  uint16_t* dx; cudaMalloc(&dx, hx.size() * 2); cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice);
  int hrows[8] = {7, 500, 3, 999, 42, 0, 123, 77};
  int* drows; cudaMalloc(&drows, sizeof(hrows)); cudaMemcpy(drows, hrows, sizeof(hrows), cudaMemcpyHostToDevice);
  uint16_t* dout; cudaMalloc(&dout, 512);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  for (int swz = 0; swz < 2; ++swz) {
    CUtensorMap map;
    cuuint64_t gdim[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(n)};
    cuuint64_t gstride[1] = {static_cast<cuuint64_t>(cols) * 2};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dx, gdim, gstride, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("swizzle %s: encode rc=%d\n", swz ? "64B" : "none", (int)r);
    if (r) continue;
    cudaMemset(dout, 0xff, 512);
    probe<<<1, 32>>>(map, drows, dout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("  kernel: %s\n", cudaGetErrorString(e));
    if (e) return 1;
    std::vector<uint16_t> ho(256);
    cudaMemcpy(ho.data(), dout, 512, cudaMemcpyDeviceToHost);
    int ok_plain = 1, ok_swz = 1;
    for (int rr = 0; rr < 8; ++rr)
      for (int c = 0; c < 32; ++c) {
        const uint16_t want = static_cast<uint16_t>(hrows[rr] * 64 + c);
        if (ho[rr * 32 + c] != want) ok_plain = 0;
        const int chunk = c / 8, phys = chunk ^ ((rr >> 1) & 3);
        if (ho[rr * 32 + phys * 8 + c % 8] != want) ok_swz = 0;
      }
    printf("  layout row-major: %d   row-major with SW64 chunk xor ((r>>1)&3): %d\n", ok_plain, ok_swz);
    for (int rr = 0; rr < 8; ++rr) printf("  smem row %d: first elems %u %u ... chunk heads %u %u %u %u\n", rr,
                                         ho[rr * 32], ho[rr * 32 + 1], ho[rr * 32], ho[rr * 32 + 8], ho[rr * 32 + 16], ho[rr * 32 + 24]);
  }
  return 0;
}
