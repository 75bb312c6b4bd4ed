// rgms_hyb.cu — RGMS over per-relation hyb decompositions: the `hyb` format of
// build_rgms_pipeline (driver.cpp:290-300 decomposes every relation's slice with
// hyb_rules(k = hyb_auto_k(slice)) and lifts the rules to the relation axis), i.e. SURVEY §8b's
// strata_rgms_hyb_bf16(per-relation parts, X, W, Y, d_in, d_out, stream).
//
// The device reads every relation's ELL parts in place (strata_hyb handles), drops the padding
// slots with the reference's rule (a slot repeating the previous column of its ELL row is a pad,
// storage.cpp:528), and rebuilds the relation-major edge list the RGMS plan takes:
//   1. rgms_hyb_keep_kernel   one thread per ELL slot of all parts: keep flag;
//   2. cub exclusive scan     positions of the kept slots;
//   3. rgms_hyb_emit_kernel   64-bit key (relation, row, col) and the value of each kept slot;
//   4. cub radix sort         key order = relation-major, rows ascending, columns ascending (the
//                             CSR order of every slice, whatever the parts' bucket order was);
//   5. rgms_hyb_split_kernel  decode (dst, src), rel_ptr by lower bound;
// then strata_rgms_plan / strata_rgms_run_bf16 as for the CSR form.  The product is the
// reference's (pads multiply by zero there; summation order is irrelevant on its integer
// operands and within the bf16 bar on real ones).
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "common.cuh"

using namespace strata_b200;

namespace {

struct PartDesc {
  const int32_t* I;   // ELL row -> matrix row
  const int32_t* J;   // [nrows][width] columns
  const float* V;     // [nrows][width] values
  long long slot0;    // first global slot of this part
  long long nslots;   // nrows * width
  int width_log2;
  int rel;
};

__device__ __forceinline__ int find_part(const PartDesc* __restrict__ d, int np, long long g) {
  int lo = 0, hi = np - 1;  // last part with slot0 <= g
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (d[mid].slot0 <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void rgms_hyb_keep_kernel(const PartDesc* __restrict__ d, int np, long long total,
                                     int32_t* __restrict__ keep) {
  for (long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    const PartDesc& P = d[find_part(d, np, g)];
    const long long s = g - P.slot0;
    const int k = static_cast<int>(s & ((1ll << P.width_log2) - 1));
    keep[g] = (k == 0 || P.J[s] != P.J[s - 1]) ? 1 : 0;
  }
}

__global__ void rgms_hyb_emit_kernel(const PartDesc* __restrict__ d, int np, long long total,
                                     const int32_t* __restrict__ keep, const int32_t* __restrict__ pos,
                                     unsigned long long rows, unsigned long long cols,
                                     unsigned long long* __restrict__ key, float* __restrict__ val) {
  for (long long g = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; g < total;
       g += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (!keep[g]) continue;
    const PartDesc& P = d[find_part(d, np, g)];
    const long long s = g - P.slot0;
    const unsigned long long row = static_cast<unsigned long long>(P.I[s >> P.width_log2]);
    const unsigned long long col = static_cast<unsigned long long>(P.J[s]);
    key[pos[g]] = (static_cast<unsigned long long>(P.rel) * rows + row) * cols + col;
    val[pos[g]] = P.V[s];
  }
}

__global__ void rgms_hyb_split_kernel(const unsigned long long* __restrict__ key, long long nnz,
                                      unsigned long long rows, unsigned long long cols,
                                      int32_t* __restrict__ dst, int32_t* __restrict__ src) {
  for (long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long rem = key[e] % (rows * cols);
    dst[e] = static_cast<int32_t>(rem / cols);
    src[e] = static_cast<int32_t>(rem % cols);
  }
}

__global__ void rgms_hyb_relptr_kernel(const unsigned long long* __restrict__ key, long long nnz,
                                       long long R, unsigned long long rows_cols,
                                       int32_t* __restrict__ rel_ptr) {
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r <= R;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long t = static_cast<unsigned long long>(r) * rows_cols;
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (key[mid] < t) lo = mid + 1; else hi = mid;
    }
    rel_ptr[r] = static_cast<int32_t>(lo);
  }
}

unsigned grid_of(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, num_sms() * 16LL)));
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return STRATA_OK;
  } catch (const ApiError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return STRATA_ERR_INTERNAL;
  }
}

}  // namespace

extern "C" int strata_rgms_plan_hyb(const strata_hyb* const* hybs, int64_t R, strata_rgms** out,
                                    void* stream) {
  int rc_plan = STRATA_OK;
  const int rc = guarded([&] {
    if (!out || !hybs) throw ApiError(STRATA_ERR_USAGE, "null argument");
    *out = nullptr;
    if (R < 1) throw ApiError(STRATA_ERR_USAGE, "RGMS requires at least one relation");  // kernels.cpp:139
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t rows = -1, cols = -1;
    std::vector<PartDesc> parts;
    long long total = 0;
    for (int64_t r = 0; r < R; ++r) {
      if (!hybs[r]) throw ApiError(STRATA_ERR_USAGE, "null hyb handle for relation " + std::to_string(r));
      const strata_hyb_impl& H = *hybs[r];
      if (r == 0) { rows = H.rows; cols = H.cols; }
      if (H.rows != rows || H.cols != cols)
        throw ApiError(STRATA_ERR_USAGE, "all relations must share dims");
      for (const HybPart& P : H.parts) {
        PartDesc d{H.I.p + P.row_off, H.J.p + P.slot_off, H.V.p + P.slot_off, total,
                   P.nrows * P.width, P.bucket, static_cast<int>(r)};
        total += d.nslots;
        parts.push_back(d);
      }
    }
    const unsigned long long urows = static_cast<unsigned long long>(std::max<int64_t>(rows, 1));
    const unsigned long long ucols = static_cast<unsigned long long>(std::max<int64_t>(cols, 1));
    if (static_cast<double>(R) * static_cast<double>(urows) * static_cast<double>(ucols) > 9.0e18)
      throw ApiError(STRATA_ERR_CAPACITY, "relations x rows x cols exceeds the 64-bit edge key");
    if (total > INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "nnz exceeds int32");
    long long nnz = 0;
    unsigned long long* keys = nullptr;
    float* vals = nullptr;
    if (total > 0) {
      DevBuf<PartDesc> dparts(parts.size(), s);
      STRATA_CUDA_CHECK(cudaMemcpyAsync(dparts.p, parts.data(), parts.size() * sizeof(PartDesc),
                                        cudaMemcpyHostToDevice, s));
      const int np = static_cast<int>(parts.size());
      DevBuf<int32_t> keep(total + 1, s), pos(total + 1, s);
      STRATA_CUDA_CHECK(cudaMemsetAsync(keep.p + total, 0, sizeof(int32_t), s));
      rgms_hyb_keep_kernel<<<grid_of(total), 256, 0, s>>>(dparts.p, np, total, keep.p);
      size_t tb = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, tb, keep.p, pos.p, total + 1, s);
      {
        DevBuf<unsigned char> tmp(tb, s);
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, keep.p, pos.p, total + 1, s);
      }
      int32_t hn = 0;
      STRATA_CUDA_CHECK(cudaMemcpyAsync(&hn, pos.p + total, sizeof(hn), cudaMemcpyDeviceToHost, s));
      STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
      nnz = hn;
      keys = static_cast<unsigned long long*>(workspace_alloc(sizeof(unsigned long long) * nnz * 2, s));
      vals = static_cast<float*>(workspace_alloc(sizeof(float) * nnz * 2, s));
      rgms_hyb_emit_kernel<<<grid_of(total), 256, 0, s>>>(dparts.p, np, total, keep.p, pos.p, urows,
                                                          ucols, keys, vals);
      STRATA_CUDA_CHECK(cudaGetLastError());
      int end_bit = 1;
      const unsigned long long maxkey = static_cast<unsigned long long>(R) * urows * ucols;
      while (end_bit < 64 && (1ull << end_bit) < maxkey) ++end_bit;
      size_t sb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, sb, keys, keys + nnz, vals, vals + nnz, nnz, 0, end_bit, s);
      DevBuf<unsigned char> stmp(sb, s);
      cub::DeviceRadixSort::SortPairs(stmp.p, sb, keys, keys + nnz, vals, vals + nnz, nnz, 0, end_bit, s);
      STRATA_CUDA_CHECK(cudaGetLastError());
    }
    DevBuf<int32_t> rel_ptr(R + 1, s), dst(std::max<long long>(nnz, 1), s), src(std::max<long long>(nnz, 1), s);
    if (nnz > 0) {
      rgms_hyb_split_kernel<<<grid_of(nnz), 256, 0, s>>>(keys + nnz, nnz, urows, ucols, dst.p, src.p);
      rgms_hyb_relptr_kernel<<<grid_of(R + 1), 256, 0, s>>>(keys + nnz, nnz, R, urows * ucols, rel_ptr.p);
    } else {
      STRATA_CUDA_CHECK(cudaMemsetAsync(rel_ptr.p, 0, sizeof(int32_t) * (R + 1), s));
    }
    STRATA_CUDA_CHECK(cudaGetLastError());
    rc_plan = strata_rgms_plan(rel_ptr.p, dst.p, src.p, nnz > 0 ? vals + nnz : nullptr, R,
                               std::max<int64_t>(rows, 0), std::max<int64_t>(cols, 0), nnz, out, stream);
    std::string err = rc_plan != STRATA_OK ? strata_last_error() : "";
    if (keys) STRATA_CUDA_CHECK(cudaFreeAsync(keys, s));
    if (vals) STRATA_CUDA_CHECK(cudaFreeAsync(vals, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));  // rel_ptr / dst / src are freed on return
    if (rc_plan != STRATA_OK) throw ApiError(rc_plan, err);
  });
  return rc;
}

extern "C" int strata_rgms_hyb_bf16(const strata_hyb* const* hybs, int64_t R, const void* X_bf16,
                                    const void* W_bf16, float* Y, int64_t d_in, int64_t d_out,
                                    void* stream) {
  strata_rgms* h = nullptr;
  int rc = strata_rgms_plan_hyb(hybs, R, &h, stream);
  if (rc != STRATA_OK) return rc;
  rc = strata_rgms_run_bf16(h, X_bf16, W_bf16, Y, d_in, d_out, stream);
  if (rc == STRATA_OK)
    rc = guarded([&] { STRATA_CUDA_CHECK(cudaStreamSynchronize(static_cast<cudaStream_t>(stream))); });
  strata_rgms_destroy(h);
  return rc;
}
