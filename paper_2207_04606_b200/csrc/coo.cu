// coo.cu — device build_csr (storage.cpp:89-124): COO triplets -> CSR (SURVEY §8f "device-side
// ingest"; the reference sorts 24-byte triplets with std::sort on one core: 8.3 s at C5).
//
//   range check  -> any coordinate outside [0, rows) x [0, cols): Validation "coordinate out of
//                   range" (checked first, like the reference)
//   key sort     -> 64-bit keys row * cols + col, radix-sorted with the triplet ids
//   duplicates   -> the first sorted position whose key equals its predecessor's: Validation
//                   "duplicate coordinate (r, c)" naming that pair, exactly the reference's message
//   scatter      -> indices[q] = key % cols, values[q] = vals[id]; indptr[r] = first q with
//                   key >= r * cols (lower bound per row)
// Keys are unique once duplicates are rejected, so the result is the reference's bit for bit.
#include <cub/cub.cuh>

#include <algorithm>
#include <string>

#include "capi_internal.h"
#include "common.cuh"

namespace strata_b200 {
namespace {

__global__ void coo_keys_kernel(const int32_t* __restrict__ r, const int32_t* __restrict__ c,
                                long long nnz, long long rows, long long cols,
                                unsigned long long* __restrict__ keys, int32_t* __restrict__ ids,
                                int* __restrict__ bad) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long ri = r[i], ci = c[i];
    if (ri < 0 || ri >= rows || ci < 0 || ci >= cols) {
      atomicOr(bad, 1);
      keys[i] = 0;
    } else {
      keys[i] = static_cast<unsigned long long>(ri) * static_cast<unsigned long long>(cols) +
                static_cast<unsigned long long>(ci);
    }
    ids[i] = static_cast<int32_t>(i);
  }
}

// first duplicate (smallest sorted position q with key[q] == key[q-1]); values / indices.
__global__ void coo_scatter_kernel(const unsigned long long* __restrict__ keys,
                                   const int32_t* __restrict__ ids, const float* __restrict__ v,
                                   long long nnz, long long cols, int32_t* __restrict__ indices,
                                   float* __restrict__ values, unsigned long long* __restrict__ dup) {
  for (long long q = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; q < nnz;
       q += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long k = keys[q];
    if (q > 0 && keys[q - 1] == k) atomicMin(dup, static_cast<unsigned long long>(q));
    indices[q] = static_cast<int32_t>(k % static_cast<unsigned long long>(cols));
    values[q] = v[ids[q]];
  }
}

__global__ void coo_indptr_kernel(const unsigned long long* __restrict__ keys, long long nnz,
                                  long long rows, long long cols, int32_t* __restrict__ indptr) {
  for (long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; r <= rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long t = static_cast<unsigned long long>(r) * static_cast<unsigned long long>(cols);
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (keys[mid] < t) lo = mid + 1; else hi = mid;
    }
    indptr[r] = static_cast<int32_t>(lo);
  }
}

}  // namespace

void csr_from_coo_device(const int32_t* r, const int32_t* c, const float* v, int64_t nnz,
                         int64_t rows, int64_t cols, int32_t* indptr, int32_t* indices,
                         float* values, cudaStream_t s) {
  if (rows < 0 || cols < 0 || nnz < 0) throw ApiError(STRATA_ERR_USAGE, "negative dims");
  if (nnz > INT32_MAX) throw ApiError(STRATA_ERR_CAPACITY, "nnz exceeds int32 index range");
  const unsigned g = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((nnz + 255) / 256, num_sms() * 16LL)));
  if (nnz == 0) {
    STRATA_CUDA_CHECK(cudaMemsetAsync(indptr, 0, sizeof(int32_t) * (rows + 1), s));
    return;
  }
  if (rows == 0 || cols == 0) throw ApiError(STRATA_ERR_VALIDATION, "coordinate out of range");
  auto* keys = static_cast<unsigned long long*>(workspace_alloc(sizeof(unsigned long long) * nnz * 2, s));
  auto* ids = static_cast<int32_t*>(workspace_alloc(sizeof(int32_t) * nnz * 2, s));
  auto* flags = static_cast<unsigned long long*>(workspace_alloc(sizeof(unsigned long long) * 2, s));
  int* bad = reinterpret_cast<int*>(flags);
  unsigned long long* dup = flags + 1;
  STRATA_CUDA_CHECK(cudaMemsetAsync(flags, 0, sizeof(unsigned long long), s));
  STRATA_CUDA_CHECK(cudaMemsetAsync(dup, 0xFF, sizeof(unsigned long long), s));
  coo_keys_kernel<<<g, 256, 0, s>>>(r, c, nnz, rows, cols, keys, ids, bad);
  int end_bit = 1;
  const unsigned long long maxkey = static_cast<unsigned long long>(rows) * static_cast<unsigned long long>(std::max<int64_t>(cols, 1));
  while (end_bit < 64 && (1ULL << end_bit) < maxkey) ++end_bit;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys, keys + nnz, ids, ids + nnz, nnz, 0, end_bit, s);
  void* tmp = workspace_alloc(tb, s);
  cub::DeviceRadixSort::SortPairs(tmp, tb, keys, keys + nnz, ids, ids + nnz, nnz, 0, end_bit, s);
  coo_scatter_kernel<<<g, 256, 0, s>>>(keys + nnz, ids + nnz, v, nnz, cols, indices, values, dup);
  const unsigned gr = static_cast<unsigned>(std::max<long long>(1, std::min<long long>((rows + 1 + 255) / 256, num_sms() * 16LL)));
  coo_indptr_kernel<<<gr, 256, 0, s>>>(keys + nnz, nnz, rows, cols, indptr);
  STRATA_CUDA_CHECK(cudaGetLastError());
  unsigned long long hf[2];
  STRATA_CUDA_CHECK(cudaMemcpyAsync(hf, flags, sizeof(hf), cudaMemcpyDeviceToHost, s));
  unsigned long long dkey = 0;
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));  // the one host sync: validation result
  if (hf[1] != ~0ULL)
    STRATA_CUDA_CHECK(cudaMemcpy(&dkey, keys + nnz + hf[1], sizeof(dkey), cudaMemcpyDeviceToHost));
  STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(flags, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(ids, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(keys, s));
  if (static_cast<int>(hf[0] & 0xFFFFFFFFu) != 0)
    throw ApiError(STRATA_ERR_VALIDATION, "coordinate out of range");
  if (hf[1] != ~0ULL) {
    const unsigned long long uc = static_cast<unsigned long long>(cols);
    throw ApiError(STRATA_ERR_VALIDATION, "duplicate coordinate (" + std::to_string(dkey / uc) +
                                              ", " + std::to_string(dkey % uc) + ")");
  }
}

}  // namespace strata_b200
