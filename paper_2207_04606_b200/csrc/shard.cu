// shard.cu — row-partitioned multi-GPU SpMM / SDDMM behind the C ABI.
//
// One process per GPU.  Output rows are independent (kernels.cpp:85-108 / :110-136 write row
// i from row i's non-zeros only), so the path shards by contiguous nnz-balanced row ranges
// (strata_partition_rows: cut p = first row with indptr >= nnz*p/P) with no exchange before
// the compute; the only collective reassembles the outputs every rank needs next:
//   SpMM   this rank's range is cut again into `chunks` nnz-balanced sub-ranges, each
//          decomposed to hyb(c, k) on this device (shard-concatenated buckets equal the global
//          decomposition).  X[cols][d] is replicated, Y[rows][d] is a full replica
//          on every rank.  Reassembly:
//            nccl  chunk q of every rank is broadcast from its owner (one ncclGroup of P
//                  ncclBroadcast = an uneven all-gather, in place) on the plan's comm stream,
//                  overlapping the SpMM of chunk q+1;
//            p2p   the fused peer-store kernel (spmm_hyb_kernel<..., kMulti>) writes every
//                  finished row into all ranks' replicas (CUDA IPC mappings) — no collective.
//   SDDMM  the same row ranges give contiguous nnz ranges of B[nnz]; each rank computes its
//          range (X[rows][d] and Y[d][n] replicated) and, if asked, the ranges are all-gathered
//          the same way (grouped broadcasts), else B stays sharded.
// NCCL is resolved at run time (dlopen of the libnccl.so.2 already in the process — e.g.
// PyTorch's — or the system one), so loading this library never pins an NCCL build.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "common.cuh"

using namespace strata_b200;

struct strata_shard_plan {
  int device = 0;
  int rank = 0, world = 1, chunks = 1;
  int64_t rows = 0, cols = 0, nnz = 0;
  std::vector<int64_t> indptr_host;              // [rows+1]
  std::vector<std::vector<int64_t>> sub;         // sub[q] = chunks+1 row cuts of rank q
  std::vector<std::unique_ptr<strata_hyb>> hyb;  // this rank's chunks
  DevBuf<int32_t> sddmm_indptr;                  // this rank's rows, rebased to 0
  const int32_t* indices = nullptr;              // caller's full CSR (kept alive by the caller)
  const float* values = nullptr;
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ev;                   // chunks + 1
  ~strata_shard_plan() {
    for (auto e : ev) cudaEventDestroy(e);
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
};

namespace {

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

void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw ApiError(code, msg);
}

// ---- NCCL, resolved at run time ---------------------------------------------------------------
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  static std::string err;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL, if any
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      err = std::string("NCCL unavailable: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) err = std::string("NCCL symbol missing: ") + name;
      return p;
    };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.CommCount = reinterpret_cast<decltype(n.CommCount)>(sym("ncclCommCount"));
    n.CommUserRank = reinterpret_cast<decltype(n.CommUserRank)>(sym("ncclCommUserRank"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty()) throw ApiError(STRATA_ERR_USAGE, err);
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw ApiError(STRATA_ERR_CUDA, std::string(what) + ": " + nccl().GetErrorString(r));
}

// Cuts of the row range [r0, r1) into `parts` nnz-balanced contiguous ranges: cut p is the
// first row whose indptr reaches base + floor(total*p/parts) — strata_partition_rows' rule.
std::vector<int64_t> cuts(const std::vector<int64_t>& ip, int64_t r0, int64_t r1, int parts) {
  std::vector<int64_t> b(parts + 1);
  const int64_t base = ip[r0], total = ip[r1] - base;
  b[0] = r0;
  b[parts] = r1;
  for (int p = 1; p < parts; ++p) {
    const int64_t target = base + (total * p) / parts;
    b[p] = std::lower_bound(ip.begin() + r0, ip.begin() + r1 + 1, target) - ip.begin();
    b[p] = std::max(b[p - 1], std::min(b[p], r1));
  }
  return b;
}

__global__ void rebase_kernel(const int32_t* __restrict__ in, long long n, int32_t* __restrict__ out) {
  const int32_t base = in[0];
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    out[i] = in[i] - base;
}

const strata_shard_plan& plan_of(const strata_shard_plan* p) {
  require(p != nullptr, STRATA_ERR_USAGE, "null shard plan");
  return *p;
}

ncclComm_t comm_of(const void* comm, int ndev, const strata_shard_plan& P) {
  require(ndev == P.world, STRATA_ERR_USAGE,
          "sharded call: ndev " + std::to_string(ndev) + " != plan world " + std::to_string(P.world));
  if (comm == nullptr) return nullptr;  // no reassembly: this rank's rows / range only
  ncclComm_t c = *static_cast<const ncclComm_t*>(comm);
  int n = 0, r = 0;
  nccl_check(nccl().CommCount(c, &n), "ncclCommCount");
  nccl_check(nccl().CommUserRank(c, &r), "ncclCommUserRank");
  require(n == P.world && r == P.rank, STRATA_ERR_USAGE,
          "sharded call: communicator is rank " + std::to_string(r) + " of " + std::to_string(n) +
              ", plan is rank " + std::to_string(P.rank) + " of " + std::to_string(P.world));
  return c;
}

}  // namespace

extern "C" {

int strata_nccl_unique_id(void* id_out) {
  return guarded([&] {
    require(id_out != nullptr, STRATA_ERR_USAGE, "null id buffer");
    static_assert(sizeof(ncclUniqueId) == STRATA_NCCL_ID_BYTES, "ncclUniqueId size");
    nccl_check(nccl().GetUniqueId(static_cast<ncclUniqueId*>(id_out)), "ncclGetUniqueId");
  });
}

int strata_nccl_comm_init(const void* id, int nranks, int rank, void* comm_out) {
  return guarded([&] {
    require(id && comm_out, STRATA_ERR_USAGE, "null argument");
    require(nranks >= 1 && rank >= 0 && rank < nranks, STRATA_ERR_USAGE, "bad rank / nranks");
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    nccl_check(nccl().CommInitRank(static_cast<ncclComm_t*>(comm_out), nranks, uid, rank),
               "ncclCommInitRank");
  });
}

int strata_nccl_comm_destroy(void* comm) {
  return guarded([&] {
    if (!comm) return;
    nccl_check(nccl().CommDestroy(*static_cast<ncclComm_t*>(comm)), "ncclCommDestroy");
  });
}

int strata_shard_plan_create(const int32_t* indptr, const int32_t* indices, const float* values,
                             int64_t rows, int64_t cols, int rank, int world, int chunks, int c,
                             int k, strata_shard_plan** out, void* stream) {
  return guarded([&] {
    require(out != nullptr, STRATA_ERR_USAGE, "null output handle");
    require(world >= 1 && rank >= 0 && rank < world, STRATA_ERR_USAGE, "bad rank / world");
    require(chunks >= 1 && chunks <= 64, STRATA_ERR_USAGE, "chunks must be in [1, 64]");
    require(rows >= 0 && cols >= 0 && (rows == 0 || indptr), STRATA_ERR_USAGE, "bad CSR");
    require(c >= 1 && k >= 0, STRATA_ERR_USAGE, "hyb requires c >= 1 and k >= 0");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto P = std::make_unique<strata_shard_plan>();
    STRATA_CUDA_CHECK(cudaGetDevice(&P->device));
    P->rank = rank;
    P->world = world;
    P->chunks = chunks;
    P->rows = rows;
    P->cols = cols;
    P->indices = indices;
    P->values = values;
    // The host indptr decides every rank's cuts identically (one D2H of rows+1 ints).
    std::vector<int32_t> ip32(rows + 1);
    STRATA_CUDA_CHECK(cudaMemcpyAsync(ip32.data(), indptr, (rows + 1) * sizeof(int32_t),
                                      cudaMemcpyDeviceToHost, s));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    P->indptr_host.assign(ip32.begin(), ip32.end());
    P->nnz = P->indptr_host[rows];
    require(P->nnz == 0 || (indices && values), STRATA_ERR_USAGE, "null CSR arrays");
    const std::vector<int64_t> ranks = cuts(P->indptr_host, 0, rows, world);
    P->sub.resize(world);
    for (int q = 0; q < world; ++q) P->sub[q] = cuts(P->indptr_host, ranks[q], ranks[q + 1], chunks);
    // This rank's chunks: hyb over the un-rebased row slice (indptr values index the full
    // indices / values arrays directly).
    for (int ch = 0; ch < chunks; ++ch) {
      const int64_t a = P->sub[rank][ch], b = P->sub[rank][ch + 1];
      strata_hyb* h = nullptr;
      const int rc = strata_hyb_decompose(indptr + a, indices, values, b - a, cols,
                                          P->indptr_host[b] - P->indptr_host[a], c, k, stream, &h);
      if (rc != STRATA_OK) throw ApiError(rc, strata_last_error());
      P->hyb.emplace_back(h);
    }
    // SDDMM walks non-zero chunks from 0: a rebased indptr of this rank's rows.
    const int64_t r0 = ranks[rank], r1 = ranks[rank + 1];
    P->sddmm_indptr.alloc(r1 - r0 + 1);
    rebase_kernel<<<static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>((r1 - r0 + 256) / 256, 1184))),
                    256, 0, s>>>(indptr + r0, r1 - r0 + 1, P->sddmm_indptr.p);
    STRATA_CUDA_CHECK(cudaGetLastError());
    STRATA_CUDA_CHECK(cudaStreamCreateWithFlags(&P->comm_stream, cudaStreamNonBlocking));
    P->ev.resize(chunks + 1);
    for (auto& e : P->ev) STRATA_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    *out = P.release();
  });
}

int strata_shard_plan_rows(const strata_shard_plan* p, int rank, int chunk, int64_t* row0,
                           int64_t* row1) {
  return guarded([&] {
    const auto& P = plan_of(p);
    require(rank >= 0 && rank < P.world, STRATA_ERR_USAGE, "rank out of range");
    require(chunk >= -1 && chunk < P.chunks, STRATA_ERR_USAGE, "chunk out of range");
    const auto& s = P.sub[rank];
    if (row0) *row0 = chunk < 0 ? s.front() : s[chunk];
    if (row1) *row1 = chunk < 0 ? s.back() : s[chunk + 1];
  });
}

int strata_shard_plan_destroy(strata_shard_plan* p) {
  return guarded([&] {
    if (!p) return;
    DeviceGuard g(p->device);
    delete p;
  });
}

int strata_spmm_hyb_f32_sharded(const strata_shard_plan* p, const float* X, float* Y, int64_t d,
                                const void* comm, int ndev, void* stream) {
  return guarded([&] {
    const auto& P = plan_of(p);
    require(d >= 1 && X && Y, STRATA_ERR_USAGE, "sharded spmm: bad operands");
    const ncclComm_t cm = comm_of(comm, ndev, P);
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const Nccl* n = cm ? &nccl() : nullptr;
    if (cm) {  // the comm stream must not touch Y before the caller's prior work on it
      STRATA_CUDA_CHECK(cudaEventRecord(P.ev[P.chunks], s));
      STRATA_CUDA_CHECK(cudaStreamWaitEvent(P.comm_stream, P.ev[P.chunks], 0));
    }
    for (int ch = 0; ch < P.chunks; ++ch) {
      float* y = Y + P.sub[P.rank][ch] * d;
      spmm_hyb_launch(*P.hyb[ch], X, &y, 1, d, s);
      if (!cm) continue;
      STRATA_CUDA_CHECK(cudaEventRecord(P.ev[ch], s));
      STRATA_CUDA_CHECK(cudaStreamWaitEvent(P.comm_stream, P.ev[ch], 0));
      nccl_check(n->GroupStart(), "ncclGroupStart");
      for (int q = 0; q < P.world; ++q) {
        float* buf = Y + P.sub[q][ch] * d;
        const size_t count = static_cast<size_t>((P.sub[q][ch + 1] - P.sub[q][ch]) * d);
        nccl_check(n->Broadcast(buf, buf, count, ncclFloat32, q, cm, P.comm_stream), "ncclBroadcast");
      }
      nccl_check(n->GroupEnd(), "ncclGroupEnd");
    }
    if (cm) {
      STRATA_CUDA_CHECK(cudaEventRecord(P.ev[P.chunks], P.comm_stream));
      STRATA_CUDA_CHECK(cudaStreamWaitEvent(s, P.ev[P.chunks], 0));
    }
  });
}

int strata_spmm_hyb_f32_sharded_p2p(const strata_shard_plan* p, const float* X,
                                    float* const* Y_dsts, int ndev, int64_t d, void* stream) {
  return guarded([&] {
    const auto& P = plan_of(p);
    require(d >= 1 && X && Y_dsts, STRATA_ERR_USAGE, "sharded spmm: bad operands");
    require(ndev == P.world && ndev <= STRATA_MAX_Y_DESTS, STRATA_ERR_USAGE,
            "sharded p2p spmm: one destination per rank (<= " + std::to_string(STRATA_MAX_Y_DESTS) + ")");
    for (int ch = 0; ch < P.chunks; ++ch) {
      float* dst[STRATA_MAX_Y_DESTS];
      for (int q = 0; q < ndev; ++q) {
        require(Y_dsts[q] != nullptr, STRATA_ERR_USAGE, "sharded p2p spmm: null destination");
        dst[q] = Y_dsts[q] + P.sub[P.rank][ch] * d;
      }
      // the own replica first: the multi-destination kernel stores it, then the peers'
      std::swap(dst[0], dst[P.rank]);
      spmm_hyb_launch(*P.hyb[ch], X, dst, ndev, d, static_cast<cudaStream_t>(stream));
    }
  });
}

int strata_sddmm_csr_f32_sharded(const strata_shard_plan* p, const float* X, const float* Yd,
                                 float* B, int64_t d, int gather, const void* comm, int ndev,
                                 void* stream) {
  return guarded([&] {
    const auto& P = plan_of(p);
    require(d >= 1 && X && Yd && B, STRATA_ERR_USAGE, "sharded sddmm: bad operands");
    const ncclComm_t cm = gather ? comm_of(comm, ndev, P) : nullptr;
    require(ndev == P.world, STRATA_ERR_USAGE, "sharded sddmm: ndev != plan world");
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t r0 = P.sub[P.rank].front(), r1 = P.sub[P.rank].back();
    const int64_t q0 = P.indptr_host[r0], q1 = P.indptr_host[r1];
    if (q1 > q0)
      sddmm_csr_launch(P.sddmm_indptr.p, P.indices + q0, P.values + q0, X + r0 * d, Yd, B + q0,
                       r1 - r0, P.cols, q1 - q0, d, s);
    if (!cm) return;
    const Nccl& n = nccl();
    STRATA_CUDA_CHECK(cudaEventRecord(P.ev[0], s));
    STRATA_CUDA_CHECK(cudaStreamWaitEvent(P.comm_stream, P.ev[0], 0));
    nccl_check(n.GroupStart(), "ncclGroupStart");
    for (int q = 0; q < P.world; ++q) {
      const int64_t a = P.indptr_host[P.sub[q].front()], b = P.indptr_host[P.sub[q].back()];
      nccl_check(n.Broadcast(B + a, B + a, static_cast<size_t>(b - a), ncclFloat32, q, cm, P.comm_stream),
                 "ncclBroadcast");
    }
    nccl_check(n.GroupEnd(), "ncclGroupEnd");
    STRATA_CUDA_CHECK(cudaEventRecord(P.ev[0], P.comm_stream));
    STRATA_CUDA_CHECK(cudaStreamWaitEvent(s, P.ev[0], 0));
  });
}

}  // extern "C"
