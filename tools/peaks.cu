// peaks.cu — measured denominators for the rooflines bench.py reports beside MEASURED_PEAKS.json
// (which holds the HBM copy bandwidth and the dense bf16 rate, not these):
//   * L2 read bandwidth: 256-bit loads (ld.global.nc.v8.f32, the SpMM/attention gathers' own
//     instruction) sweeping an L2-resident buffer again and again, every SM busy;
//   * pinned host <-> device copy rates (the e2e path's bound): H2D alone, D2H alone, and both
//     directions at once on two streams (how strata_spmm_hyb_f32_host_batch overlaps them).
// Prints one JSON line.  Build + run: tools/gpu_peaks.sh (nvcc -gencode arch=compute_100a,...).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

__global__ void __launch_bounds__(512) l2_read_kernel(const float* __restrict__ buf, long long n8,
                                                      int reps, float* __restrict__ sink) {
  float acc = 0.f;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (int r = 0; r < reps; ++r) {
    // rotate the start so consecutive sweeps do not hit the same LTS slice in lock step
    const long long start = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x +
                             static_cast<long long>(r) * 4099) % stride;
    for (long long i = start; i < n8; i += stride) {
      float v[8];
      asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                     "=f"(v[6]), "=f"(v[7])
                   : "l"(buf + i * 8));
      acc += ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
    }
  }
  if (acc == 123.456f) sink[0] = acc;  // never true for the zero buffer; keeps the loads live
}

static float time_ms(cudaStream_t s, cudaEvent_t a, cudaEvent_t b) {
  float ms = 0;
  CK(cudaEventSynchronize(b));
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms;
}

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp prop{};
  CK(cudaGetDeviceProperties(&prop, 0));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2, e3;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  CK(cudaEventCreate(&e3));

  // ---- L2 read bandwidth over several resident footprints ----
  const int sms = prop.multiProcessorCount;
  float* sink = nullptr;
  CK(cudaMalloc(&sink, 4));
  std::printf("{\"device\": \"%s\", \"sms\": %d, \"l2_bytes\": %d", prop.name, sms, prop.l2CacheSize);
  double best_l2 = 0;
  const long long sizes_mb[] = {16, 32, 48, 64, 96};
  std::printf(", \"l2_read_gbs\": {");
  for (int si = 0; si < 5; ++si) {
    const long long bytes = sizes_mb[si] << 20;
    float* buf = nullptr;
    CK(cudaMalloc(&buf, bytes));
    CK(cudaMemset(buf, 0, bytes));
    const long long n8 = bytes / 32;
    const int reps = static_cast<int>(std::max<long long>(4, (8LL << 30) / bytes));  // ~8 GB read
    const int grid = sms * 4;
    l2_read_kernel<<<grid, 512, 0, s0>>>(buf, n8, 2, sink);  // warm: pull into L2
    std::vector<float> t;
    for (int it = 0; it < 5; ++it) {
      CK(cudaEventRecord(e0, s0));
      l2_read_kernel<<<grid, 512, 0, s0>>>(buf, n8, reps, sink);
      CK(cudaEventRecord(e1, s0));
      t.push_back(time_ms(s0, e0, e1));
    }
    CK(cudaGetLastError());
    std::sort(t.begin(), t.end());
    const double gbs = static_cast<double>(bytes) * reps / (t[t.size() / 2] * 1e-3) / 1e9;
    best_l2 = std::max(best_l2, gbs);
    std::printf("%s\"%lld_MB\": %.1f", si ? ", " : "", sizes_mb[si], gbs);
    CK(cudaFree(buf));
  }
  std::printf("}, \"l2_read_peak_gbs\": %.1f", best_l2);

  // ---- pinned host <-> device ----
  const size_t cb = 1253902848;  // the C5 e2e step: 2,449,029 x 128 x 4 bytes each way
  void *h_in = nullptr, *h_out = nullptr, *d_in = nullptr, *d_out = nullptr;
  CK(cudaMallocHost(&h_in, cb));
  CK(cudaMallocHost(&h_out, cb));
  CK(cudaMalloc(&d_in, cb));
  CK(cudaMalloc(&d_out, cb));
  std::memset(h_in, 1, cb);
  auto med = [](std::vector<float> v) {
    std::sort(v.begin(), v.end());
    return v[v.size() / 2];
  };
  std::vector<float> th, td, tb;
  for (int it = 0; it < 6; ++it) {
    CK(cudaEventRecord(e0, s0));
    CK(cudaMemcpyAsync(d_in, h_in, cb, cudaMemcpyHostToDevice, s0));
    CK(cudaEventRecord(e1, s0));
    if (it) th.push_back(time_ms(s0, e0, e1));
    CK(cudaEventRecord(e0, s0));
    CK(cudaMemcpyAsync(h_out, d_out, cb, cudaMemcpyDeviceToHost, s0));
    CK(cudaEventRecord(e1, s0));
    if (it) td.push_back(time_ms(s0, e0, e1));
    // both directions at once
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0, s0));
    CK(cudaStreamWaitEvent(s1, e0, 0));
    CK(cudaMemcpyAsync(d_in, h_in, cb, cudaMemcpyHostToDevice, s0));
    CK(cudaMemcpyAsync(h_out, d_out, cb, cudaMemcpyDeviceToHost, s1));
    CK(cudaEventRecord(e2, s1));
    CK(cudaStreamWaitEvent(s0, e2, 0));
    CK(cudaEventRecord(e1, s0));
    if (it) tb.push_back(time_ms(s0, e0, e1));
  }
  const double h2d = cb / (med(th) * 1e-3) / 1e9, d2h = cb / (med(td) * 1e-3) / 1e9;
  const double both_ms = med(tb);
  std::printf(
      ", \"copy_bytes\": %zu, \"h2d_gbs\": %.2f, \"d2h_gbs\": %.2f, \"bidir_ms\": %.3f, "
      "\"bidir_gbs_each\": %.2f}\n",
      cb, h2d, d2h, both_ms, cb / (both_ms * 1e-3) / 1e9);
  return 0;
}
