// mtx.cu — device Matrix Market ingest: read_matrix_market
// (mmio.hpp:22-23, mmio.cpp:17-55) with the entry lines segmented and parsed on the GPU.
//
// The reference reads the banner line, skips comment / empty lines, reads the size line, then
// getline()s exactly nnz entry lines and parses each with an istringstream (`>> i >> j`, then
// `>> v` unless the field is "pattern"), pushing (i-1, j-1, v) and, for a symmetric file, the
// mirrored (j-1, i-1, v) right after it (mmio.cpp:43-52).  Here:
//   host    banner / comments / size line (a few bytes; parsed with the same istringstream
//           extraction so the reference's messages and corner cases carry over);
//   device  1. mtx_nl_count_kernel   newlines per 4 KB block of the entry region;
//           2. cub exclusive scan     block bases;
//           3. mtx_nl_pos_kernel     byte offset of newline q for q < nnz (block scan);
//           4. mtx_parse_kernel      one thread per line: libstdc++ num_get grammar for int64
//                                    and double (checked against the linked reference in
//                                    tests/test_gpu_mtx.py), decimal -> double correctly
//                                    rounded (Clinger fast path, else exact big-integer
//                                    rounding, subnormals included), range check, first
//                                    failing line by atomicMin;
//           5. symmetric files only: scan of 1 + (i != j) per line, mtx_mirror_kernel.
// Only the verdict (first failing line, newline count) comes back to the host; the failing
// line's text for the message is read from the caller's host buffer.
// Values are kept as the reference's f64 triplet values plus their f32 rounding (what
// build_csr stores for the F32 pipeline, storage.cpp:57-61 / :117), ready for
// strata_csr_from_coo.
#include <cub/cub.cuh>
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cfloat>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.h"
#include "common.cuh"

using namespace strata_b200;

struct strata_mtx {
  int device = 0;
  int64_t rows = 0, cols = 0, ntrip = 0;
  DevBuf<int32_t> row, col;
  DevBuf<double> v64;
  DevBuf<float> v32;
};

namespace {

constexpr int kBlockBytes = 4096;  // newline-count block: 256 threads x 16 bytes
constexpr int kNlThreads = 256;

__device__ __forceinline__ int nl_in(const uint4& q) {
  int n = 0;
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    // bytes equal to '\n' (0x0a): zero bytes of w ^ 0x0a0a0a0a, counted exactly
    const uint32_t x = w[i] ^ 0x0a0a0a0au;
    const uint32_t t = ((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x;
    n += __popc(~t & 0x80808080u);
  }
  return n;
}

// 16 bytes of the region at byte offset o (o % 16 == 0), zero-padded past the end.
__device__ __forceinline__ uint4 load16(const uint8_t* __restrict__ buf, long long o, long long n) {
  if (o + 16 <= n) return *reinterpret_cast<const uint4*>(buf + o);
  uint8_t b[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) b[i] = o + i < n ? buf[o + i] : 0;
  uint4 q;
  memcpy(&q, b, 16);
  return q;
}

__global__ void __launch_bounds__(kNlThreads)
mtx_nl_count_kernel(const uint8_t* __restrict__ buf, long long n, long long* __restrict__ cnt) {
  using Reduce = cub::BlockReduce<int, kNlThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  const long long o = static_cast<long long>(blockIdx.x) * kBlockBytes + threadIdx.x * 16;
  const int c = o < n ? nl_in(load16(buf, o, n)) : 0;
  const int tot = Reduce(tmp).Sum(c);
  if (threadIdx.x == 0) cnt[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kNlThreads)
mtx_nl_pos_kernel(const uint8_t* __restrict__ buf, long long n, const long long* __restrict__ base,
                  long long want, long long* __restrict__ pos) {
  using Scan = cub::BlockScan<int, kNlThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const long long b0 = base[blockIdx.x];
  if (b0 >= want) return;  // uniform per block
  const long long o = static_cast<long long>(blockIdx.x) * kBlockBytes + threadIdx.x * 16;
  const uint4 q = o < n ? load16(buf, o, n) : make_uint4(0, 0, 0, 0);
  int before = 0;
  Scan(tmp).ExclusiveSum(nl_in(q), before);
  long long k = b0 + before;
  const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    if (((w[i >> 2] >> (8 * (i & 3))) & 0xffu) == 0x0au && o + i < n) {
      if (k < want) pos[k] = o + i;
      ++k;
    }
  }
}

// ---- decimal -> double, correctly rounded (round half to even), as strtod -----------------
constexpr int kLimbs = 30;  // 960 bits: w (64) * 5^308 and (5^343 << 57) both fit
struct Big {
  uint32_t l[kLimbs];
  int n;  // limbs in use (l[n-1] != 0 unless n == 0)
};

__device__ void big_set(Big& a, unsigned long long v) {
  a.n = 0;
  while (v) { a.l[a.n++] = static_cast<uint32_t>(v); v >>= 32; }
}
__device__ void big_mul(Big& a, uint32_t m) {
  unsigned long long carry = 0;
  for (int i = 0; i < a.n; ++i) {
    const unsigned long long t = static_cast<unsigned long long>(a.l[i]) * m + carry;
    a.l[i] = static_cast<uint32_t>(t);
    carry = t >> 32;
  }
  if (carry) a.l[a.n++] = static_cast<uint32_t>(carry);
}
__device__ void big_pow5(Big& a, int e) {  // a *= 5^e
  while (e >= 13) { big_mul(a, 1220703125u); e -= 13; }  // 5^13
  uint32_t m = 1;
  while (e-- > 0) m *= 5;
  if (m > 1) big_mul(a, m);
}
__device__ int big_bits(const Big& a) {
  return a.n == 0 ? 0 : 32 * (a.n - 1) + (32 - __clz(a.l[a.n - 1]));
}
__device__ void big_shl(Big& a, int s) {
  if (a.n == 0 || s == 0) return;
  const int w = s / 32, b = s % 32;
  int n = a.n + w + 1;
  for (int i = n - 1; i >= 0; --i) {
    const int j = i - w;
    uint32_t hi = j >= 0 && j < a.n ? a.l[j] : 0;
    uint32_t lo = j - 1 >= 0 && j - 1 < a.n ? a.l[j - 1] : 0;
    a.l[i] = b ? (hi << b) | (lo >> (32 - b)) : hi;
  }
  a.n = n;
  while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}
__device__ void big_shr1(Big& a) {
  for (int i = 0; i < a.n; ++i) a.l[i] = (a.l[i] >> 1) | (i + 1 < a.n ? a.l[i + 1] << 31 : 0u);
  while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}
__device__ int big_cmp(const Big& a, const Big& b) {
  if (a.n != b.n) return a.n < b.n ? -1 : 1;
  for (int i = a.n - 1; i >= 0; --i)
    if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
  return 0;
}
__device__ void big_sub(Big& a, const Big& b) {  // a -= b, a >= b
  long long borrow = 0;
  for (int i = 0; i < a.n; ++i) {
    long long t = static_cast<long long>(a.l[i]) - (i < b.n ? b.l[i] : 0u) - borrow;
    borrow = t < 0;
    a.l[i] = static_cast<uint32_t>(t + (borrow << 32));
  }
  while (a.n > 0 && a.l[a.n - 1] == 0) --a.n;
}
// Bits [lo, hi) of a as an integer (hi - lo <= 64).
__device__ unsigned long long big_bits_range(const Big& a, int lo, int hi) {
  unsigned long long r = 0;
  for (int b = hi - 1; b >= lo; --b) r = (r << 1) | ((a.l[b >> 5] >> (b & 31)) & 1u);
  return r;
}
__device__ bool big_any_below(const Big& a, int bits) {
  for (int i = 0; i < a.n && 32 * i < bits; ++i) {
    const int take = min(32, bits - 32 * i);
    const uint32_t m = take == 32 ? 0xffffffffu : ((1u << take) - 1u);
    if (a.l[i] & m) return true;
  }
  return false;
}

// Round (Q + frac) * 2^E0 to the nearest double (ties to even; frac > 0 iff sticky).
__device__ double round_to_double(unsigned long long Q, bool sticky, int E0) {
  if (Q == 0) return 0.0;
  const int bq = 64 - __clzll(Q);
  const int E = max(E0 + bq - 53, -1074);
  const int drop = E - E0;
  if (drop <= 0) return scalbn(static_cast<double>(Q), E0);  // exact, Q < 2^53
  unsigned long long mant, half, rest;
  if (drop >= 65) { mant = 0; half = 0; rest = Q; }
  else if (drop == 64) { mant = 0; half = Q >> 63; rest = Q & ~(1ull << 63); }
  else {
    mant = Q >> drop;
    half = (Q >> (drop - 1)) & 1ull;
    rest = drop - 1 == 0 ? 0 : (Q & ((1ull << (drop - 1)) - 1ull));
  }
  if (half && (rest || sticky || (mant & 1ull))) ++mant;
  return scalbn(static_cast<double>(mant), E);  // mant <= 2^53: exact (or overflow to inf)
}

// w * 10^q for w < 10^19 (exact decimal significand), correctly rounded.
__device__ double decimal_to_double(unsigned long long w, int q) {
  if (w == 0) return 0.0;
  if (q > 308) return __longlong_as_double(0x7ff0000000000000ll);  // >= 1e309: inf
  if (q < -343) return 0.0;      // < 1e-324 < 2^-1075
  if (w <= (1ull << 53) && q >= -22 && q <= 22) {  // Clinger: one rounding of exact operands
    double p = 1.0;
    for (int i = 0; i < (q < 0 ? -q : q); ++i) p *= 10.0;  // exact up to 1e22
    return q < 0 ? __ddiv_rn(static_cast<double>(w), p) : __dmul_rn(static_cast<double>(w), p);
  }
  Big num;
  big_set(num, w);
  if (q >= 0) {
    big_pow5(num, q);  // value = num * 2^q
    const int nb = big_bits(num);
    if (nb <= 64) return round_to_double(big_bits_range(num, 0, nb), false, q);
    const int s = nb - 60;
    return round_to_double(big_bits_range(num, s, nb), big_any_below(num, s), q + s);
  }
  Big den;
  big_set(den, 1);
  big_pow5(den, -q);  // value = num / den * 2^q
  // Scale so that the quotient lands in [2^54, 2^57): num <<= a, or den <<= -a.
  const int a = 55 + big_bits(den) - big_bits(num);
  if (a >= 0) big_shl(num, a); else big_shl(den, -a);
  // Q = floor(num / den) < 2^57 by restoring division against den << 56 .. den.
  Big D = den;
  big_shl(D, 56);
  unsigned long long Q = 0;
  for (int bit = 56; bit >= 0; --bit) {
    if (big_cmp(num, D) >= 0) {
      big_sub(num, D);
      Q |= 1ull << bit;
    }
    big_shr1(D);
  }
  return round_to_double(Q, num.n != 0, q - a);
}

__device__ __forceinline__ bool is_space(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}
__device__ __forceinline__ bool is_digit(uint8_t c) { return c >= '0' && c <= '9'; }

// istringstream >> int64_t (libstdc++ num_get): skip whitespace, [+-] digits; no digit or
// overflow fails.
__device__ bool parse_i64(const uint8_t* s, long long& p, long long e, long long& out) {
  while (p < e && is_space(s[p])) ++p;
  bool neg = false;
  if (p < e && (s[p] == '+' || s[p] == '-')) { neg = s[p] == '-'; ++p; }
  if (p >= e || !is_digit(s[p])) return false;
  unsigned long long v = 0;
  bool ovf = false;
  const unsigned long long lim = neg ? 9223372036854775808ull : 9223372036854775807ull;
  while (p < e && is_digit(s[p])) {
    const unsigned d = s[p++] - '0';
    if (v > (lim - d) / 10) ovf = true; else v = v * 10 + d;
  }
  if (ovf) return false;
  out = neg ? static_cast<long long>(0ull - v) : static_cast<long long>(v);
  return true;
}

// istringstream >> double (libstdc++ num_get + strtod): [+-] digits [. digits] [(e|E) [+-]
// digits]; a mantissa without digits, or an exponent marker without digits, fails with v = 0;
// overflow gives +-DBL_MAX (failbit, mmio.cpp ignores it); an exhausted line leaves `out`
// (mmio.cpp's v = 1.0) untouched.  Returns false only when more than
// 19 significant digits leave the rounding undecided (reported as unsupported).
__device__ bool parse_f64(const uint8_t* s, long long& p, long long e, double& out) {
  while (p < e && is_space(s[p])) ++p;
  if (p >= e) return true;  // nothing left: the sentry fails before num_get, `out` unchanged
  out = 0.0;
  bool neg = false;
  if (p < e && (s[p] == '+' || s[p] == '-')) { neg = s[p] == '-'; ++p; }
  unsigned long long w = 0;
  int nd = 0, qadj = 0;
  bool any = false, dropped = false;
  while (p < e && is_digit(s[p])) {
    const unsigned d = s[p++] - '0';
    any = true;
    if (nd == 0 && d == 0) continue;
    if (nd < 19) { w = w * 10 + d; ++nd; } else { ++qadj; dropped |= d != 0; }
  }
  if (p < e && s[p] == '.') {
    ++p;
    while (p < e && is_digit(s[p])) {
      const unsigned d = s[p++] - '0';
      any = true;
      if (nd == 0 && d == 0) { --qadj; continue; }
      if (nd < 19) { w = w * 10 + d; ++nd; --qadj; } else { dropped |= d != 0; }
    }
  }
  if (!any) return true;  // v = 0
  long long ex = 0;
  if (p < e && (s[p] == 'e' || s[p] == 'E')) {
    ++p;
    bool eneg = false;
    if (p < e && (s[p] == '+' || s[p] == '-')) { eneg = s[p] == '-'; ++p; }
    if (p >= e || !is_digit(s[p])) return true;  // "1e", "1e+": extraction fails, v = 0
    while (p < e && is_digit(s[p])) {
      ex = ex * 10 + (s[p++] - '0');
      if (ex > 100000) ex = 100000;
    }
    if (eneg) ex = -ex;
  }
  const int q = static_cast<int>(max(-200000ll, min(200000ll, ex + qadj)));
  double v = decimal_to_double(w, q);
  if (dropped) {  // significand truncated to 19 digits: decided iff w and w + 1 agree
    const double v2 = decimal_to_double(w + 1, q);
    if (v2 != v) return false;
  }
  if (isinf(v)) v = DBL_MAX;
  out = neg ? -v : v;
  return true;
}

enum : int { kOk = 0, kBadEntry = 1, kOutOfRange = 2, kUnsupported = 3 };

__global__ void mtx_parse_kernel(const uint8_t* __restrict__ buf, long long nbytes,
                                 const long long* __restrict__ nlpos, long long nl_have,
                                 long long nlines, long long rows, long long cols, int pattern,
                                 int symmetric, int32_t* __restrict__ r, int32_t* __restrict__ c,
                                 double* __restrict__ v, int32_t* __restrict__ mult,
                                 unsigned long long* __restrict__ first_bad) {
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < nlines;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long p = k == 0 ? 0 : nlpos[k - 1] + 1;
    const long long e = k < nl_have ? nlpos[k] : nbytes;
    long long i = 0, j = 0;
    double val = 1.0;
    int st = kOk;
    if (!parse_i64(buf, p, e, i) || !parse_i64(buf, p, e, j)) {
      st = kBadEntry;
    } else {
      if (!pattern && !parse_f64(buf, p, e, val)) st = kUnsupported;
      if (st == kOk && (i < 1 || i > rows || j < 1 || j > cols)) st = kOutOfRange;
    }
    if (st != kOk) {
      atomicMin(first_bad, (static_cast<unsigned long long>(k) << 2) | static_cast<unsigned>(st));
      continue;
    }
    r[k] = static_cast<int32_t>(i - 1);
    c[k] = static_cast<int32_t>(j - 1);
    v[k] = val;
    if (symmetric) mult[k] = i != j ? 2 : 1;
  }
}

// Symmetric files: triplet positions from the scan of 1 + (i != j); mirrored entry follows.
__global__ void mtx_mirror_kernel(const int32_t* __restrict__ r, const int32_t* __restrict__ c,
                                  const double* __restrict__ v, const int32_t* __restrict__ off,
                                  long long nlines, int32_t* __restrict__ ro, int32_t* __restrict__ co,
                                  double* __restrict__ vo, float* __restrict__ vf) {
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < nlines;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long o = off[k];
    ro[o] = r[k]; co[o] = c[k]; vo[o] = v[k]; vf[o] = static_cast<float>(v[k]);
    if (r[k] != c[k]) {
      ro[o + 1] = c[k]; co[o + 1] = r[k]; vo[o + 1] = v[k]; vf[o + 1] = static_cast<float>(v[k]);
    }
  }
}

__global__ void to_f32_kernel(const double* __restrict__ v, long long n, float* __restrict__ f) {
  for (long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    f[k] = static_cast<float>(v[k]);
}

unsigned grid_for(long long n) {
  return static_cast<unsigned>(std::max<long long>(1, std::min<long long>((n + 255) / 256, num_sms() * 16LL)));
}

// Host part of mmio.cpp:17-38: banner, comments, size line.  Returns the byte offset of the
// first entry line.
long long read_preamble(const char* text, long long bytes, bool& pattern, bool& symmetric,
                        long long& rows, long long& cols, long long& nnz) {
  long long p = 0;
  auto getline = [&](std::string& line) -> bool {
    line.clear();
    if (p >= bytes) return false;
    const void* nl = memchr(text + p, '\n', static_cast<size_t>(bytes - p));
    const long long e = nl ? static_cast<const char*>(nl) - text : bytes;
    line.assign(text + p, static_cast<size_t>(e - p));
    p = nl ? e + 1 : bytes;
    return true;
  };
  std::string line;
  if (!getline(line)) throw ApiError(STRATA_ERR_USAGE, "empty matrix market stream");
  std::istringstream hdr(line);
  std::string banner, object, fmt, field, symmetry;
  hdr >> banner >> object >> fmt >> field >> symmetry;
  if (banner != "%%MatrixMarket" || object != "matrix" || fmt != "coordinate")
    throw ApiError(STRATA_ERR_USAGE, "unsupported matrix market header: " + line);
  pattern = field == "pattern";
  symmetric = symmetry == "symmetric";
  if (field != "real" && field != "integer" && !pattern)
    throw ApiError(STRATA_ERR_USAGE, "unsupported matrix market field: " + field);
  while (getline(line))
    if (!line.empty() && line[0] != '%') break;
  std::istringstream dims(line);
  int64_t r = 0, c = 0, z = 0;
  if (!(dims >> r >> c >> z)) throw ApiError(STRATA_ERR_USAGE, "bad matrix market size line");
  rows = r; cols = c; nnz = z;
  return p;
}

// Host text -> device for large pageable buffers: host threads copy 32 MB chunks into a ring of
// pinned buffers (two sets of kStageThreads) while the copy engine drains the other set, so the
// transfer runs at the threads' memcpy rate overlapped with DMA instead of the driver's
// single-threaded pageable staging (C5 text, 1.1 GB: ~100 ms pageable).  The ring is allocated
// once per process (portable pinned memory) and serialised by a mutex.
constexpr int kStageThreads = 4;
constexpr size_t kStageChunk = size_t(32) << 20;

struct StageRing {
  std::mutex mu;
  char* buf[2 * kStageThreads] = {};
  bool ok = false, tried = false;
  bool ensure() {
    if (tried) return ok;
    tried = true;
    for (int i = 0; i < 2 * kStageThreads; ++i) {
      void* p = nullptr;
      if (cudaHostAlloc(&p, kStageChunk, cudaHostAllocPortable) != cudaSuccess) {
        cudaGetLastError();
        return ok = false;
      }
      buf[i] = static_cast<char*>(p);
    }
    return ok = true;
  }
};

StageRing& stage_ring() {
  static StageRing* r = new StageRing;  // process lifetime (no teardown-order CUDA calls)
  return *r;
}

void copy_text_h2d(uint8_t* dst, const char* src, long long n, cudaStream_t s) {
  cudaPointerAttributes pa{};
  const bool pinned = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  StageRing& R = stage_ring();
  std::unique_lock<std::mutex> lock(R.mu);
  // small, already page-locked or no pinned memory: one copy
  const bool ring = !pinned && n >= static_cast<long long>(4 * kStageChunk) && R.ensure();
  if (std::getenv("STRATA_MTX_DEBUG"))
    std::fprintf(stderr, "[strata mtx] %lld bytes: %s\n", n,
                 ring ? "pinned staging ring" : (pinned ? "page-locked source" : "driver pageable copy"));
  if (!ring) {
    lock.unlock();
    STRATA_CUDA_CHECK(cudaMemcpyAsync(dst, src, static_cast<size_t>(n), cudaMemcpyHostToDevice, s));
    return;
  }
  cudaEvent_t ev[2 * kStageThreads];
  for (auto& e : ev) STRATA_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const long long nchunks = (n + static_cast<long long>(kStageChunk) - 1) / static_cast<long long>(kStageChunk);
  bool used[2 * kStageThreads] = {};
  try {
    for (long long w = 0; w * kStageThreads < nchunks; ++w) {
      const int set = static_cast<int>(w & 1) * kStageThreads;
      const long long c0 = w * kStageThreads;
      const int nc = static_cast<int>(std::min<long long>(kStageThreads, nchunks - c0));
      for (int t = 0; t < nc; ++t)  // the set's previous DMA must have drained
        if (used[set + t]) STRATA_CUDA_CHECK(cudaEventSynchronize(ev[set + t]));
      std::thread th[kStageThreads];
      for (int t = 0; t < nc; ++t) {
        const long long o = (c0 + t) * static_cast<long long>(kStageChunk);
        const size_t len = static_cast<size_t>(std::min<long long>(kStageChunk, n - o));
        try {
          th[t] = std::thread([&R, set, t, src, o, len] { std::memcpy(R.buf[set + t], src + o, len); });
        } catch (...) {  // no thread: copy on this one
          std::memcpy(R.buf[set + t], src + o, len);
        }
      }
      for (int t = 0; t < nc; ++t)
        if (th[t].joinable()) th[t].join();
      for (int t = 0; t < nc; ++t) {
        const long long o = (c0 + t) * static_cast<long long>(kStageChunk);
        const size_t len = static_cast<size_t>(std::min<long long>(kStageChunk, n - o));
        STRATA_CUDA_CHECK(cudaMemcpyAsync(dst + o, R.buf[set + t], len, cudaMemcpyHostToDevice, s));
        STRATA_CUDA_CHECK(cudaEventRecord(ev[set + t], s));
        used[set + t] = true;
      }
    }
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));  // the ring is free for the next caller
  } catch (...) {
    cudaStreamSynchronize(s);
    for (auto& e : ev) cudaEventDestroy(e);
    throw;
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

std::string line_at(const char* text, long long bytes, long long start) {
  const void* nl = memchr(text + start, '\n', static_cast<size_t>(bytes - start));
  const long long e = nl ? static_cast<const char*>(nl) - text : bytes;
  return std::string(text + start, static_cast<size_t>(e - start));
}

void mtx_parse(const char* text, long long bytes, strata_mtx& h, cudaStream_t s) {
  bool pattern = false, symmetric = false;
  long long rows = 0, cols = 0, nnz = 0;
  const long long off = read_preamble(text, bytes, pattern, symmetric, rows, cols, nnz);
  if (nnz < 0) throw ApiError(STRATA_ERR_USAGE, "bad matrix market size line");
  if (rows > INT32_MAX || cols > INT32_MAX)
    throw ApiError(STRATA_ERR_CAPACITY, "matrix market dimensions exceed the int32 index range");
  h.rows = rows;
  h.cols = cols;
  h.ntrip = 0;
  if (nnz == 0) return;
  STRATA_CUDA_CHECK(cudaGetDevice(&h.device));
  const long long n = bytes - off;  // entry region
  if (n <= 0) throw ApiError(STRATA_ERR_USAGE, "truncated matrix market entries");

  auto* buf = static_cast<uint8_t*>(workspace_alloc(static_cast<size_t>(n) + 16, s));
  copy_text_h2d(buf, text + off, n, s);
  const long long nblk = (n + kBlockBytes - 1) / kBlockBytes;
  auto* cnt = static_cast<long long*>(workspace_alloc(sizeof(long long) * (nblk + 1) * 2, s));
  long long* base = cnt + nblk + 1;
  STRATA_CUDA_CHECK(cudaMemsetAsync(cnt + nblk, 0, sizeof(long long), s));
  mtx_nl_count_kernel<<<static_cast<unsigned>(nblk), kNlThreads, 0, s>>>(buf, n, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, base, nblk + 1, s);
  void* tmp = workspace_alloc(tb, s);
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, base, nblk + 1, s);
  auto* nlpos = static_cast<long long*>(workspace_alloc(sizeof(long long) * nnz, s));
  mtx_nl_pos_kernel<<<static_cast<unsigned>(nblk), kNlThreads, 0, s>>>(buf, n, base, nnz, nlpos);
  long long nl_total = 0;
  STRATA_CUDA_CHECK(cudaMemcpyAsync(&nl_total, base + nblk, sizeof(long long), cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  STRATA_CUDA_CHECK(cudaGetLastError());
  // Lines getline() can deliver: one per newline, plus a non-empty unterminated tail.
  long long last_nl = -1;
  if (nl_total > 0 && nl_total <= nnz)
    STRATA_CUDA_CHECK(cudaMemcpy(&last_nl, nlpos + nl_total - 1, sizeof(long long), cudaMemcpyDeviceToHost));
  long long nlines = std::min(nl_total, nnz);
  if (nl_total < nnz && n - (last_nl + 1) > 0) ++nlines;

  // Outputs from the stream-ordered pool (persistent: freed with the handle); cudaMalloc /
  // cudaFree of ~1 GB per parse cost more than the parse kernels at C5.
  DevBuf<int32_t> r, c, mult;
  DevBuf<double> v;
  r.alloc_async(nlines, s, true);
  c.alloc_async(nlines, s, true);
  v.alloc_async(nlines, s, true);
  if (symmetric) mult.alloc_async(nlines + 1, s, true);
  auto* bad = static_cast<unsigned long long*>(workspace_alloc(sizeof(unsigned long long), s));
  STRATA_CUDA_CHECK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
  if (nlines > 0)
    mtx_parse_kernel<<<grid_for(nlines), 256, 0, s>>>(buf, n, nlpos, std::min(nl_total, nnz), nlines,
                                                       rows, cols, pattern, symmetric, r.p, c.p, v.p,
                                                       mult.p, bad);
  STRATA_CUDA_CHECK(cudaGetLastError());
  unsigned long long hb = 0;
  STRATA_CUDA_CHECK(cudaMemcpyAsync(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  long long bad_start = -1;
  if (hb != ~0ull) {
    const long long k = static_cast<long long>(hb >> 2);
    bad_start = 0;
    if (k > 0) {
      STRATA_CUDA_CHECK(cudaMemcpy(&bad_start, nlpos + k - 1, sizeof(long long), cudaMemcpyDeviceToHost));
      ++bad_start;
    }
  }
  STRATA_CUDA_CHECK(cudaFreeAsync(bad, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(nlpos, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(tmp, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(cnt, s));
  STRATA_CUDA_CHECK(cudaFreeAsync(buf, s));
  if (hb != ~0ull) {
    const std::string line = line_at(text + off, n, bad_start);
    switch (static_cast<int>(hb & 3u)) {
      case kBadEntry: throw ApiError(STRATA_ERR_USAGE, "bad matrix market entry: " + line);
      case kOutOfRange: throw ApiError(STRATA_ERR_USAGE, "matrix market entry out of range: " + line);
      default:
        throw ApiError(STRATA_ERR_USAGE,
                       "matrix market value needs more than 19 significant digits to round: " + line);
    }
  }
  if (nlines < nnz) throw ApiError(STRATA_ERR_USAGE, "truncated matrix market entries");

  if (!symmetric) {
    h.row = std::move(r);
    h.col = std::move(c);
    h.v64 = std::move(v);
    h.ntrip = nlines;
    h.v32.alloc_async(nlines, s, true);
    to_f32_kernel<<<grid_for(nlines), 256, 0, s>>>(h.v64.p, nlines, h.v32.p);
    STRATA_CUDA_CHECK(cudaGetLastError());
    STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
    return;
  }
  DevBuf<int32_t> offs(nlines + 1, s);
  STRATA_CUDA_CHECK(cudaMemsetAsync(mult.p + nlines, 0, sizeof(int32_t), s));
  tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, mult.p, offs.p, nlines + 1, s);
  DevBuf<uint8_t> t2(tb, s);
  cub::DeviceScan::ExclusiveSum(t2.p, tb, mult.p, offs.p, nlines + 1, s);
  int32_t total = 0;
  STRATA_CUDA_CHECK(cudaMemcpyAsync(&total, offs.p + nlines, sizeof(total), cudaMemcpyDeviceToHost, s));
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
  h.ntrip = total;
  h.row.alloc_async(total, s, true);
  h.col.alloc_async(total, s, true);
  h.v64.alloc_async(total, s, true);
  h.v32.alloc_async(total, s, true);
  mtx_mirror_kernel<<<grid_for(nlines), 256, 0, s>>>(r.p, c.p, v.p, offs.p, nlines, h.row.p, h.col.p,
                                                      h.v64.p, h.v32.p);
  STRATA_CUDA_CHECK(cudaGetLastError());
  STRATA_CUDA_CHECK(cudaStreamSynchronize(s));
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

extern "C" {

int strata_mtx_parse(const char* text, int64_t bytes, strata_mtx** out, void* stream) {
  return guarded([&] {
    if (!out || (bytes > 0 && !text)) throw ApiError(STRATA_ERR_USAGE, "null argument");
    if (bytes < 0) throw ApiError(STRATA_ERR_USAGE, "negative byte count");
    auto h = std::make_unique<strata_mtx>();
    mtx_parse(text, bytes, *h, static_cast<cudaStream_t>(stream));
    *out = h.release();
  });
}

int strata_mtx_read_file(const char* path, strata_mtx** out, void* stream) {
  return guarded([&] {
    if (!out || !path) throw ApiError(STRATA_ERR_USAGE, "null argument");
    // The file is mapped, not read: the page cache is the host copy (a fresh 1 GB read buffer
    // cost ~0.3 s of first-touch page faults alone), and mtx_parse's staging threads fault the
    // mapped pages in parallel while they copy them to pinned buffers.
    const int fd = open(path, O_RDONLY);
    if (fd < 0) throw ApiError(STRATA_ERR_USAGE, std::string("cannot open ") + path);  // mmio.cpp:59
    struct stat st {};
    if (fstat(fd, &st) != 0) {
      close(fd);
      throw ApiError(STRATA_ERR_USAGE, std::string("cannot open ") + path);
    }
    const long long bytes = static_cast<long long>(st.st_size);
    void* map = bytes > 0 ? mmap(nullptr, static_cast<size_t>(bytes), PROT_READ, MAP_PRIVATE, fd, 0) : nullptr;
    close(fd);
    if (bytes > 0 && map == MAP_FAILED) throw ApiError(STRATA_ERR_USAGE, std::string("cannot open ") + path);
    if (map) madvise(map, static_cast<size_t>(bytes), MADV_SEQUENTIAL);
    struct Unmap {
      void* p;
      size_t n;
      ~Unmap() { if (p) munmap(p, n); }
    } hold{map, static_cast<size_t>(bytes)};
    const char* text = static_cast<const char*>(map);
    auto h = std::make_unique<strata_mtx>();
    mtx_parse(text, bytes, *h, static_cast<cudaStream_t>(stream));
    *out = h.release();
  });
}

int strata_mtx_info(const strata_mtx* h, int64_t* rows, int64_t* cols, int64_t* ntriplets) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null mtx handle");
    if (rows) *rows = h->rows;
    if (cols) *cols = h->cols;
    if (ntriplets) *ntriplets = h->ntrip;
  });
}

int strata_mtx_device(const strata_mtx* h, const int32_t** row, const int32_t** col,
                      const double** val64, const float** val32) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null mtx handle");
    if (row) *row = h->row.p;
    if (col) *col = h->col.p;
    if (val64) *val64 = h->v64.p;
    if (val32) *val32 = h->v32.p;
  });
}

int strata_mtx_read(const strata_mtx* h, int64_t* row, int64_t* col, double* val) {
  return guarded([&] {
    if (!h) throw ApiError(STRATA_ERR_USAGE, "null mtx handle");
    DeviceGuard g(h->device);
    const size_t n = static_cast<size_t>(h->ntrip);
    std::vector<int32_t> r(n), c(n);
    if (n) {
      STRATA_CUDA_CHECK(cudaMemcpy(r.data(), h->row.p, n * 4, cudaMemcpyDeviceToHost));
      STRATA_CUDA_CHECK(cudaMemcpy(c.data(), h->col.p, n * 4, cudaMemcpyDeviceToHost));
      if (val) STRATA_CUDA_CHECK(cudaMemcpy(val, h->v64.p, n * 8, cudaMemcpyDeviceToHost));
    }
    for (size_t i = 0; i < n; ++i) {
      if (row) row[i] = r[i];
      if (col) col[i] = c[i];
    }
  });
}

int strata_mtx_destroy(strata_mtx* h) {
  return guarded([&] {
    if (!h) return;
    DeviceGuard g(h->device);
    delete h;
  });
}

}  // extern "C"
