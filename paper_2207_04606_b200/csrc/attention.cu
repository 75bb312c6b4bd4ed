// attention.cu — fused GNN attention layer step: SDDMM -> edge softmax -> SpMM in one pass
// ("GAT-style"; the reference composes these as separate stage-III
// programs: SDDMM kernels.cpp:110-136, then SpMM kernels.cpp:85-108).
//
//   s_ij = A_ij * <Q_i, K_j>                  (SDDMM on the sparsity pattern of A)
//   a_ij = exp(s_ij - max_j s_ij) / sum_j exp(s_ij - max_j s_ij)     (row softmax over stored j)
//   Z_i  = sum_j a_ij * V_j                    (SpMM with the attention weights)
//
// One pass over each row's edges with the online-softmax recurrence (running max m, running
// sum l, rescaled accumulator), so neither the scores nor the weights touch HBM: per edge the
// K_j and V_j rows are gathered once (128-bit per lane), the dot is reduced across the virtual
// warp by butterfly shuffles.  Power-law rows: rows longer than kChunk edges are cut into
// chunks whose (m, l, acc) partials are merged in chunk order by a second kernel (log-sum-exp
// merge), so a hub row does not serialise one warp.  Deterministic (fixed orders, no atomics).
// Empty rows give Z_i = 0.
#include <cub/cub.cuh>

#include <algorithm>
#include <memory>

#include "capi_internal.h"
#include "common.cuh"

using namespace strata_b200;

struct strata_attn_plan {
  int device = 0;
  int64_t m = 0, nnz = 0, nitems = 0, nchunks = 0;
  DevBuf<int2> items;        // work item: (row, first edge offset inside the row) ...
  DevBuf<int32_t> item_len;  // ... and its edge count
  DevBuf<int32_t> long_rows; // rows split into chunks, and their first chunk index
  DevBuf<int32_t> long_off;  // [nlong + 1]
  int64_t nlong = 0;
};  // per call: long-row chunk partials [nchunks][d + 4] = acc[d], m, l (16-byte records)

namespace {

constexpr int kChunk = 256;  // rows longer than this are split into kChunk-edge chunks

// Items: one per row of length <= kChunk, else one per kChunk-edge chunk of the row.
__global__ void attn_items_kernel(const int32_t* __restrict__ indptr, long long m,
                                  const long long* __restrict__ off, int2* __restrict__ items,
                                  int32_t* __restrict__ len_out) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long len = indptr[i + 1] - indptr[i];
    const long long n = len > kChunk ? (len + kChunk - 1) / kChunk : 1;
    for (long long c = 0; c < n; ++c) {
      items[off[i] + c] = make_int2(static_cast<int>(i), static_cast<int>(c * kChunk));
      len_out[off[i] + c] = static_cast<int>(len > kChunk ? min64(kChunk, len - c * kChunk) : len);
    }
  }
}

template <int L>
__device__ __forceinline__ float vw_allreduce(float v, unsigned mask) {
#pragma unroll
  for (int o = L / 2; o >= 1; o >>= 1) v += __shfl_xor_sync(mask, v, o, L);
  return v;
}

// One virtual warp (L lanes, one float4 of the D features each) per work item.
// Items from nlong_items_begin on are long-row chunks: they write their (acc, m, l) partial.
#ifndef STRATA_ATTN_U  // A/B knobs: edges in flight per batch, CTAs per SM the registers allow
#define STRATA_ATTN_U 2  // C2 with 256-bit slices: U = 1 / 2 / 3 / 4 / 8 -> 6.18 / 5.41 / 5.87 / 5.67 / 9.82 ms
#endif
#ifndef STRATA_ATTN_FASTEXP  // A/B knob: MUFU __expf in the edge loop (C2: 6.13 vs 6.18 ms; off)
#define STRATA_ATTN_FASTEXP 0
#endif
#if STRATA_ATTN_FASTEXP
#define ATTN_EXP(x) __expf(x)
#else
#define ATTN_EXP(x) expf(x)
#endif
#ifndef STRATA_ATTN_MB  // A/B knob: chunk partials in flight per merge step
#define STRATA_ATTN_MB 8
#endif
#ifndef STRATA_ATTN_MINB
#define STRATA_ATTN_MINB 1
#endif

#ifndef STRATA_ATTN_VEC  // A/B knob: float4s per lane (2 = one 256-bit load per K / V row slice)
#define STRATA_ATTN_VEC 2
#endif

// VEC consecutive float4 of a row slice: one 256-bit load (sm_100 LDG.256) when VEC = 2.
template <int VEC>
__device__ __forceinline__ void ld_row(const float* __restrict__ p, float4 (&v)[VEC]) {
  if constexpr (VEC == 2) {
    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[0].z), "=f"(v[0].w), "=f"(v[1].x),
                   "=f"(v[1].y), "=f"(v[1].z), "=f"(v[1].w)
                 : "l"(p));
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) v[i] = ld_gather4(reinterpret_cast<const float4*>(p) + i);
  }
}

template <int L, int VEC = 1>
__global__ void __launch_bounds__(256, STRATA_ATTN_MINB)
attn_kernel(const int32_t* __restrict__ indptr, const int32_t* __restrict__ indices,
            const float* __restrict__ A, const float* __restrict__ Q, const float* __restrict__ K,
            const float* __restrict__ V, const int2* __restrict__ items,
            const int32_t* __restrict__ item_len, long long nitems, long long nlong_items_begin,
            float* __restrict__ Z, float* __restrict__ partial) {
  constexpr int D = 4 * VEC * L;
  constexpr int U = STRATA_ATTN_U;  // edges in flight per batch
  const int wl = threadIdx.x & 31, lane = threadIdx.x & (L - 1);
  const unsigned vmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (wl & ~(L - 1)));
  const long long it = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  if (it >= nitems) return;
  const int2 item = items[it];
  const long long row = item.x;
  const int len = item_len[it];
  const long long e0 = static_cast<long long>(indptr[row]) + item.y;
  float4 q[VEC];
  ld_row<VEC>(Q + row * D + lane * 4 * VEC, q);
  float m = -INFINITY, l = 0.f;
  float4 acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int b = 0; b < len; b += U) {
    const int n = min(U, len - b);
    int32_t col[U];
    float a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      col[u] = u < n ? __ldg(indices + e0 + b + u) : 0;
      a[u] = u < n ? __ldg(A + e0 + b + u) : 0.f;
    }
    float4 kv[U][VEC], vv[U][VEC];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < n) {
        ld_row<VEC>(K + static_cast<long long>(col[u]) * D + lane * 4 * VEC, kv[u]);
        ld_row<VEC>(V + static_cast<long long>(col[u]) * D + lane * 4 * VEC, vv[u]);
      }
    }
    float s[U];
    float bm = -INFINITY;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float part = 0.f;
      if (u < n) {
#pragma unroll
        for (int i = 0; i < VEC; ++i)
          part += q[i].x * kv[u][i].x + q[i].y * kv[u][i].y + q[i].z * kv[u][i].z + q[i].w * kv[u][i].w;
      }
      s[u] = a[u] * vw_allreduce<L>(part, vmask);
      if (u < n) bm = fmaxf(bm, s[u]);
    }
    const float mn = fmaxf(m, bm);
    const float scale = ATTN_EXP(m - mn);  // m = -inf on the first batch -> 0
    l *= scale;
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      acc[i].x *= scale; acc[i].y *= scale; acc[i].z *= scale; acc[i].w *= scale;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (u < n) {
        const float p = ATTN_EXP(s[u] - mn);
        l += p;
#pragma unroll
        for (int i = 0; i < VEC; ++i) fma4(acc[i], p, vv[u][i]);
      }
    }
    m = mn;
  }
  if (it >= nlong_items_begin) {  // long-row chunk: hand (acc, m, l) to the merge kernel
    float* pp = partial + (it - nlong_items_begin) * (D + 4);
#pragma unroll
    for (int i = 0; i < VEC; ++i) reinterpret_cast<float4*>(pp)[lane * VEC + i] = acc[i];
    if (lane == 0) {
      pp[D] = m;
      pp[D + 1] = l;
    }
  } else {
    const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
    for (int i = 0; i < VEC; ++i)
      st_stream4(reinterpret_cast<float4*>(Z + row * D) + lane * VEC + i,
                 make_float4(acc[i].x * inv, acc[i].y * inv, acc[i].z * inv, acc[i].w * inv));
  }
}

// One virtual warp per long row: log-sum-exp merge of its chunk partials in chunk order.
template <int L>
__global__ void __launch_bounds__(256)
attn_merge_kernel(const int32_t* __restrict__ long_rows, const int32_t* __restrict__ long_off,
                  long long nlong, const float* __restrict__ partial, float* __restrict__ Z) {
  constexpr int D = 4 * L;
  const int lane = threadIdx.x & (L - 1);
  const long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) / L;
  if (r >= nlong) return;
  const int c0 = long_off[r], c1 = long_off[r + 1];
  // Dense hub rows have ~900 chunks: the partials are read kMB at a time (independent loads in
  // flight) and combined in chunk order — the same arithmetic as one chunk per step.
  constexpr int kMB = STRATA_ATTN_MB;
  // Row max: lane-strided over the chunks, then a max across the virtual warp (exact in any
  // order, so identical to the sequential scan).
  const int wl = threadIdx.x & 31;
  const unsigned vmask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (wl & ~(L - 1)));
  float M = -INFINITY;
  for (int c = c0; c < c1; c += L * kMB) {
    float mv[kMB];
#pragma unroll
    for (int u = 0; u < kMB; ++u) {
      const int q = c + u * L + lane;
      mv[u] = q < c1 ? partial[static_cast<long long>(q) * (D + 4) + D] : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < kMB; ++u) M = fmaxf(M, mv[u]);
  }
#pragma unroll
  for (int o = L / 2; o >= 1; o >>= 1) M = fmaxf(M, __shfl_xor_sync(vmask, M, o, L));
  float lsum = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int c = c0; c < c1; c += kMB) {
    float mv[kMB], lv[kMB];
    float4 av[kMB];
#pragma unroll
    for (int u = 0; u < kMB; ++u) {
      if (c + u < c1) {
        const float* pp = partial + static_cast<long long>(c + u) * (D + 4);
        mv[u] = pp[D];
        lv[u] = pp[D + 1];
        av[u] = reinterpret_cast<const float4*>(pp)[lane];
      }
    }
#pragma unroll
    for (int u = 0; u < kMB; ++u) {
      if (c + u < c1) {
        const float w = expf(mv[u] - M);
        lsum += w * lv[u];
        fma4(acc, w, av[u]);
      }
    }
  }
  const float inv = lsum > 0.f ? 1.f / lsum : 0.f;
  st_stream4(reinterpret_cast<float4*>(Z + static_cast<long long>(long_rows[r]) * D) + lane,
             make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv));
}

__global__ void long_rows_kernel(const int32_t* __restrict__ indptr, long long m,
                                 const long long* __restrict__ off, long long short_items,
                                 const long long* __restrict__ lpos, int32_t* __restrict__ long_rows,
                                 int32_t* __restrict__ long_off) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long len = indptr[i + 1] - indptr[i];
    if (len > kChunk) {
      long_rows[lpos[i]] = static_cast<int32_t>(i);
      long_off[lpos[i]] = static_cast<int32_t>(off[i] - short_items);
    }
  }
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

__global__ void is_long_kernel(const int32_t* __restrict__ indptr, long long m, long long* __restrict__ f) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i <= m;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    f[i] = i < m && indptr[i + 1] - indptr[i] > kChunk ? 1 : 0;
}

// Short-row items first (rows in order), then the long rows' chunks (rows in order): the item
// offset of row i is short_rank(i) for a short row and short_total + chunk_rank(i) otherwise.
__global__ void item_off_kernel(const int32_t* __restrict__ indptr, long long m,
                                const long long* __restrict__ is_long_scan,
                                const long long* __restrict__ chunk_scan, long long short_total,
                                long long* __restrict__ off) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool lg = indptr[i + 1] - indptr[i] > kChunk;
    off[i] = lg ? short_total + chunk_scan[i] : i - is_long_scan[i];
  }
}

__global__ void long_chunks_kernel(const int32_t* __restrict__ indptr, long long m, long long* __restrict__ c) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i <= m;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long len = i < m ? indptr[i + 1] - indptr[i] : 0;
    c[i] = len > kChunk ? (len + kChunk - 1) / kChunk : 0;
  }
}

template <int L>  // L = d / 4
void launch_attn(const strata_attn_plan& p, const int32_t* indptr, const int32_t* indices,
                 const float* A, const float* Q, const float* K, const float* V, float* Z,
                 float* partial, cudaStream_t s) {
  // 256-bit row slices (VEC = 2, half the lanes per edge) when Q / K / V are 32-byte aligned:
  // C2 6.27 -> 5.72 ms (twice the edges in flight per warp, one fewer shuffle step)
  constexpr int VEC = (STRATA_ATTN_VEC == 2 && L >= 16) ? 2 : 1;
  constexpr int LE = L / VEC;  // lanes per edge-loop virtual warp
  const bool a32 = (reinterpret_cast<uintptr_t>(Q) | reinterpret_cast<uintptr_t>(K) |
                    reinterpret_cast<uintptr_t>(V)) % 32 == 0;
  const long long short_items = p.nitems - p.nchunks;
  if (p.nitems > 0) {
    if (VEC == 2 && a32)
      attn_kernel<LE, VEC><<<static_cast<unsigned>((p.nitems * LE + 255) / 256), 256, 0, s>>>(
          indptr, indices, A, Q, K, V, p.items.p, p.item_len.p, p.nitems, short_items, Z, partial);
    else
      attn_kernel<L, 1><<<static_cast<unsigned>((p.nitems * L + 255) / 256), 256, 0, s>>>(
          indptr, indices, A, Q, K, V, p.items.p, p.item_len.p, p.nitems, short_items, Z, partial);
  }
  if (p.nlong > 0)
    attn_merge_kernel<L><<<static_cast<unsigned>((p.nlong * L + 255) / 256), 256, 0, s>>>(
        p.long_rows.p, p.long_off.p, p.nlong, partial, Z);
  STRATA_CUDA_CHECK(cudaGetLastError());
}

}  // namespace

extern "C" {

int strata_attn_plan_create(const int32_t* indptr, int64_t m, int64_t nnz, strata_attn_plan** out,
                            void* stream) {
  return guarded([&] {
    if (!out) throw ApiError(STRATA_ERR_USAGE, "null output handle");
    *out = nullptr;
    if (m < 0 || nnz < 0 || nnz > INT32_MAX) throw ApiError(STRATA_ERR_USAGE, "bad dimensions");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto p = std::make_unique<strata_attn_plan>();
    STRATA_CUDA_CHECK(cudaGetDevice(&p->device));
    p->m = m;
    p->nnz = nnz;
    if (m == 0) {
      *out = p.release();
      return;
    }
    const unsigned g = static_cast<unsigned>(std::min<long long>((m + 256) / 256, num_sms() * 16LL));
    DevBuf<long long> isl(m + 1), isl_scan(m + 1), ch(m + 1), ch_scan(m + 1), off(m);
    is_long_kernel<<<g, 256, 0, s>>>(indptr, m, isl.p);
    long_chunks_kernel<<<g, 256, 0, s>>>(indptr, m, ch.p);
    size_t tb = 0, tb2 = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tb, isl.p, isl_scan.p, m + 1, s);
    cub::DeviceScan::ExclusiveSum(nullptr, tb2, ch.p, ch_scan.p, m + 1, s);
    DevBuf<unsigned char> tmp(std::max(tb, tb2));
    cub::DeviceScan::ExclusiveSum(tmp.p, tb, isl.p, isl_scan.p, m + 1, s);
    cub::DeviceScan::ExclusiveSum(tmp.p, tb2, ch.p, ch_scan.p, m + 1, s);
    long long hl[2] = {0, 0};
    STRATA_CUDA_CHECK(cudaMemcpyAsync(&hl[0], isl_scan.p + m, sizeof(long long), cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaMemcpyAsync(&hl[1], ch_scan.p + m, sizeof(long long), cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    p->nlong = hl[0];
    p->nchunks = hl[1];
    const long long short_items = m - p->nlong;
    p->nitems = short_items + p->nchunks;
    p->items.alloc(std::max<long long>(p->nitems, 1));
    p->item_len.alloc(std::max<long long>(p->nitems, 1));
    p->long_rows.alloc(std::max<long long>(p->nlong, 1));
    p->long_off.alloc(p->nlong + 1);
    item_off_kernel<<<g, 256, 0, s>>>(indptr, m, isl_scan.p, ch_scan.p, short_items, off.p);
    attn_items_kernel<<<g, 256, 0, s>>>(indptr, m, off.p, p->items.p, p->item_len.p);
    long_rows_kernel<<<g, 256, 0, s>>>(indptr, m, off.p, short_items, isl_scan.p, p->long_rows.p,
                                       p->long_off.p);
    const int32_t total = static_cast<int32_t>(p->nchunks);
    STRATA_CUDA_CHECK(cudaMemcpyAsync(p->long_off.p + p->nlong, &total, sizeof(total),
                                      cudaMemcpyHostToDevice, s));
    STRATA_CUDA_CHECK(cudaGetLastError());
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    *out = p.release();
  });
}

int strata_attn_plan_destroy(strata_attn_plan* p) {
  delete p;
  return STRATA_OK;
}

int strata_attn_csr_f32(const strata_attn_plan* p, const int32_t* indptr, const int32_t* indices,
                        const float* A, const float* Q, const float* K, const float* V, float* Z,
                        int64_t d, void* stream) {
  return guarded([&] {
    if (!p) throw ApiError(STRATA_ERR_USAGE, "null attention plan");
    if (d != 32 && d != 64 && d != 128)
      throw ApiError(STRATA_ERR_USAGE, "attention: d must be 32, 64 or 128");
    for (const void* ptr : {static_cast<const void*>(Q), static_cast<const void*>(K),
                            static_cast<const void*>(V), static_cast<const void*>(Z)})
      if (reinterpret_cast<uintptr_t>(ptr) % 16) throw ApiError(STRATA_ERR_USAGE, "attention: 16-byte aligned operands");
    int dev = 0, major = 0;
    STRATA_CUDA_CHECK(cudaGetDevice(&dev));
    STRATA_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    if (major != 10) throw ApiError(STRATA_ERR_CUDA, "strata_b200 kernels are built for sm_100a");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // long-row chunk partials: per-call scratch from the stream-ordered pool (a plan may serve
    // several streams at once)
    float* partial = p->nchunks > 0
        ? static_cast<float*>(workspace_alloc(sizeof(float) * p->nchunks * (d + 4), s)) : nullptr;
    switch (d) {
      case 32: launch_attn<8>(*p, indptr, indices, A, Q, K, V, Z, partial, s); break;
      case 64: launch_attn<16>(*p, indptr, indices, A, Q, K, V, Z, partial, s); break;
      case 128: launch_attn<32>(*p, indptr, indices, A, Q, K, V, Z, partial, s); break;
    }
    if (partial) STRATA_CUDA_CHECK(cudaFreeAsync(partial, s));
  });
}

}  // extern "C"
