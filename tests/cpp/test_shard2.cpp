// test_shard2.cpp — the sharded C ABI with two ranks, one process each,
// driven from C++ exactly as a reference-side caller would: fork() before any CUDA call, each
// process builds its world-2 shard plan (strata_shard_plan_create) on the same device (the only
// GPU a test box has), exports its full-size Y replica with strata_ipc_get_handle, maps the
// peer's with strata_ipc_open_handle, and runs the fused peer-store SpMM
// (strata_spmm_hyb_f32_sharded_p2p) into both replicas, then the sharded SDDMM (gather = 0).
// Each replica must equal the single-GPU SpMM bitwise, each SDDMM range the single-GPU SDDMM.
// (NCCL refuses two ranks on one device; the NCCL reassembly is covered at world 1 by
// test_facade.cpp and tests/test_gpu_shard.py.)  Run by tests/test_gpu_cpp.py.
#include <sys/wait.h>
#include <unistd.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

#include "strata_b200.hpp"

using namespace strata_b200;

namespace {

struct Pipe {
  int to_peer, from_peer;
  void send(const void* p, size_t n) const {
    const char* c = static_cast<const char*>(p);
    while (n) {
      const ssize_t w = write(to_peer, c, n);
      if (w <= 0) fail(ErrKind::Internal, "pipe write");
      c += w;
      n -= static_cast<size_t>(w);
    }
  }
  void recv(void* p, size_t n) const {
    char* c = static_cast<char*>(p);
    while (n) {
      const ssize_t r = read(from_peer, c, n);
      if (r <= 0) fail(ErrKind::Internal, "pipe read");
      c += r;
      n -= static_cast<size_t>(r);
    }
  }
  void barrier() const {
    const char x = 1;
    char y = 0;
    send(&x, 1);
    recv(&y, 1);
  }
};

int run_rank(int rank, const Pipe& pipe) {
  cuda_check(cudaSetDevice(0));
  const CooMatrix a = generate_matrix("powerlaw", 20000, 18000, 0, 0, 0, 12.0, 6);
  const TensorStorage csr = build_csr(a);
  DeviceCsr dc(csr);
  const int64_t d = 64;
  std::mt19937 rng(9);
  std::uniform_int_distribution<int> val(-3, 3);
  std::vector<float> x(static_cast<size_t>(a.cols * d));
  for (auto& v : x) v = static_cast<float>(val(rng));
  DeviceArray<float> X(x);

  strata_shard_plan* plan = nullptr;
  check(strata_shard_plan_create(dc.indptr.data(), dc.indices.data(), dc.values.data(), dc.rows,
                                 dc.cols, rank, 2, /*chunks*/ 2, /*c*/ 1, /*k*/ 3, &plan, nullptr));
  // Full-size Y replica, NaN-filled, exported to the peer.
  DeviceArray<float> Y(static_cast<size_t>(a.rows * d));
  std::vector<float> nan(Y.size(), std::nanf(""));
  cuda_check(cudaMemcpy(Y.data(), nan.data(), Y.size() * 4, cudaMemcpyHostToDevice));
  char handle[STRATA_IPC_HANDLE_BYTES];
  int64_t off = 0;
  check(strata_ipc_get_handle(Y.data(), handle, &off));
  pipe.send(handle, sizeof(handle));
  pipe.send(&off, sizeof(off));
  char peer_handle[STRATA_IPC_HANDLE_BYTES];
  int64_t peer_off = 0;
  pipe.recv(peer_handle, sizeof(peer_handle));
  pipe.recv(&peer_off, sizeof(peer_off));
  void* peer_base = nullptr;
  check(strata_ipc_open_handle(peer_handle, &peer_base));
  float* dsts[2];
  dsts[rank] = Y.data();
  dsts[1 - rank] = reinterpret_cast<float*>(static_cast<char*>(peer_base) + peer_off);
  cuda_check(cudaDeviceSynchronize());
  pipe.barrier();  // both replicas NaN before anyone stores

  check(strata_spmm_hyb_f32_sharded_p2p(plan, X.data(), dsts, 2, d, nullptr));
  cuda_check(cudaDeviceSynchronize());
  pipe.barrier();  // both ranks' stores complete

  // the single-GPU reference of the whole graph
  DeviceHyb h(dc, 1, 3);
  DeviceArray<float> Yref(Y.size());
  h.spmm(X.data(), Yref.data(), d);
  const bool spmm_ok = Y.host() == Yref.host();

  // sharded SDDMM, B kept sharded: this rank's nnz range only
  std::vector<float> xs(static_cast<size_t>(a.rows * 32)), yd(static_cast<size_t>(32 * a.cols));
  for (auto& v : xs) v = static_cast<float>(val(rng));
  for (auto& v : yd) v = static_cast<float>(val(rng));
  DeviceArray<float> Xs(xs), Yd(yd), B(static_cast<size_t>(csr.nnz)), Bref(static_cast<size_t>(csr.nnz));
  std::vector<float> bnan(B.size(), std::nanf(""));
  cuda_check(cudaMemcpy(B.data(), bnan.data(), B.size() * 4, cudaMemcpyHostToDevice));
  check(strata_sddmm_csr_f32_sharded(plan, Xs.data(), Yd.data(), B.data(), 32, 0, nullptr, 2, nullptr));
  check(strata_sddmm_csr_f32(dc.indptr.data(), dc.indices.data(), dc.values.data(), Xs.data(),
                             Yd.data(), Bref.data(), a.rows, a.cols, csr.nnz, 32, nullptr));
  int64_t r0 = 0, r1 = 0;
  check(strata_shard_plan_rows(plan, rank, -1, &r0, &r1));
  const IntArray& ip = csr.arr("J_indptr");
  const auto b = B.host(), bref = Bref.host();
  bool sddmm_ok = true;
  for (int64_t q = 0; q < csr.nnz; ++q) {
    const bool mine = q >= ip[r0] && q < ip[r1];
    sddmm_ok &= mine ? b[q] == bref[q] : std::isnan(b[q]);
  }
  pipe.barrier();  // the peer is done with this replica before it is unmapped / freed
  check(strata_ipc_close(peer_base));
  check(strata_shard_plan_destroy(plan));
  std::printf("rank %d: rows [%lld, %lld) spmm %s sddmm %s\n", rank, static_cast<long long>(r0),
              static_cast<long long>(r1), spmm_ok ? "ok" : "MISMATCH", sddmm_ok ? "ok" : "MISMATCH");
  return spmm_ok && sddmm_ok ? 0 : 1;
}

}  // namespace

int main() {
  int p2c[2], c2p[2];
  if (pipe(p2c) != 0 || pipe(c2p) != 0) return 2;
  const pid_t pid = fork();  // before any CUDA call
  if (pid < 0) return 2;
  int rc = 0;
  try {
    if (pid == 0) {
      rc = run_rank(1, Pipe{c2p[1], p2c[0]});
    } else {
      rc = run_rank(0, Pipe{p2c[1], c2p[0]});
    }
  } catch (const std::exception& e) {
    std::printf("rank %d: EXCEPTION %s\n", pid == 0 ? 1 : 0, e.what());
    rc = 1;
  }
  if (pid == 0) _exit(rc);
  int status = 0;
  waitpid(pid, &status, 0);
  const int child = WIFEXITED(status) ? WEXITSTATUS(status) : 3;
  std::printf("two-rank sharded ABI: %s\n", rc == 0 && child == 0 ? "passed" : "FAILED");
  return rc == 0 && child == 0 ? 0 : 1;
}
