// Shared device/host helpers for the IVF-RaBitQ sm_100a kernels.
//
// The reference computes almost everything in float64 through NumPy; the
// helpers here reproduce NumPy's reduction orders bit-for-bit where the
// reference's result is host-independent:
//   * np.einsum("ij,ij->i") : 2 accumulator lanes, 8-element blocks visited
//     as sub-blocks 3,2,1,0, each product rounded separately (no FMA), then
//     0.0 + (acc0 + acc1);
//   * ndarray.sum()         : NumPy pairwise summation (blocks of <= 128 with 8
//     strided accumulators, recursive halving at multiples of 8).
// Every float64 operation that must match the reference is written with the
// explicit round-to-nearest intrinsics so nvcc can never contract it into an
// FMA.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/ivrq_b200.h"

namespace ivrq {

// ------------------------------------------------------------------ errors
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int check_launch(const char* what);
// The library's own stream-ordered memory pool on the current device (never the
// process-wide default pool): freed workspace stays mapped up to a bounded
// release threshold (IVRQ_POOL_KEEP_BYTES), so per-call workspaces do not
// re-map pages every call, and ivrq_release_memory() trims it.
cudaMemPool_t library_pool();
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t s);
int sm_count_of_current_device();

// Scratch memory of one C-ABI call: every block allocated through it is freed
// (stream-ordered, on the stream given at construction) when it goes out of
// scope, on the success path and on every early error return alike.
class Workspace {
 public:
  explicit Workspace(cudaStream_t s) : s_(s) {}
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() {
    for (int i = 0; i < n_; ++i) cudaFreeAsync(p_[i], s_);
  }
  // count elements of T (at least one); false (with the error set) on failure
  template <typename T>
  bool alloc(T*& out, size_t count, cudaStream_t on = nullptr) {
    out = nullptr;
    if (n_ == kMax) return false;
    void* p = nullptr;
    if (pool_malloc(&p, (count ? count : 1) * sizeof(T), on ? on : s_) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    p_[n_++] = p;
    out = static_cast<T*>(p);
    return true;
  }

 private:
  static constexpr int kMax = 48;
  cudaStream_t s_;
  void* p_[kMax] = {};
  int n_ = 0;
};

// Fork/join of a side stream inside one call: join() makes `main` wait for the
// side stream's work; the destructor joins too, so an early return never leaves
// work on the side stream that the caller's stream does not wait for.
class StreamFork {
 public:
  StreamFork(cudaStream_t main, cudaStream_t side) : main_(main), side_(side) {
    if (side_ && cudaEventCreateWithFlags(&ev_, cudaEventDisableTiming) == cudaSuccess) {
      cudaEventRecord(ev_, main_);
      cudaStreamWaitEvent(side_, ev_, 0);
    } else {
      side_ = nullptr;
    }
  }
  StreamFork(const StreamFork&) = delete;
  StreamFork& operator=(const StreamFork&) = delete;
  ~StreamFork() { join(); }
  cudaStream_t side() const { return side_ ? side_ : main_; }
  void join() {
    if (!side_) return;
    cudaEventRecord(ev_, side_);
    cudaStreamWaitEvent(main_, ev_, 0);
    cudaEventDestroy(ev_);
    side_ = nullptr;
  }

 private:
  cudaStream_t main_, side_;
  cudaEvent_t ev_ = nullptr;
};
// A non-blocking stream per device (and host thread) for intra-call fork/join.
cudaStream_t side_stream();

// Optional per-kernel timing (ivrq_kernel_timing / ivrq_kernel_time): while
// enabled, a KernelTimer around a launch records CUDA events on the launching
// stream; disabled (the default) it does nothing.
bool kernel_timing_enabled();
void kernel_timing_record(const char* name, cudaEvent_t begin, cudaEvent_t end);
struct KernelTimer {
  const char* name;
  cudaStream_t stream;
  cudaEvent_t begin = nullptr;
  KernelTimer(const char* n, cudaStream_t s) : name(n), stream(s) {
    if (kernel_timing_enabled() && cudaEventCreate(&begin) == cudaSuccess) cudaEventRecord(begin, stream);
  }
  ~KernelTimer() {
    cudaEvent_t end = nullptr;
    if (begin && cudaEventCreate(&end) == cudaSuccess) {
      cudaEventRecord(end, stream);
      kernel_timing_record(name, begin, end);
    }
  }
};

#define IVRQ_TRY(expr)              \
  do {                              \
    int _rc = (expr);               \
    if (_rc != IVRQ_OK) return _rc; \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

constexpr int kWarp = 32;

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int words_per_vector(int dims) { return (dims + 31) / 32; }

// ------------------------------------------------------------------ refine code layout
// rcodes rows hold the full unsigned code u per dim for the int8 MMA refine:
// K is padded to a multiple of 64 (two m16n8k32 steps); bits <= 4 packs two
// dims per byte (dim 2j low nibble), bits >= 5 one dim per byte.
__host__ __device__ inline int kpad64(int dims) { return (dims + 63) / 64 * 64; }
__host__ __device__ inline bool rcode_nibbles(int bits) { return bits <= 4; }
__host__ __device__ inline int64_t rcode_row_bytes_of(int dims, int bits) {
  if (bits <= 1) return 0;
  return rcode_nibbles(bits) ? kpad64(dims) / 2 : kpad64(dims);
}
// MMA K position -> dimension.  Lane t4 of a quad loads 16 codes per pair of
// k-steps (one 128-bit load of bytes, or one 64-bit load of nibbles); the
// fragment registers a0/a2 (k ranges 4t4.., 16+4t4..) are filled from them as
// below, and the query slices are laid out in the same K order.
__host__ __device__ inline int refine_kdim(int k, bool nibbles) {
  const int s = k >> 5, w = k & 31, t4 = (w & 15) >> 2, j = w & 3, half = w >> 4;
  const int p = s >> 1, odd = s & 1;
  const int base = 16 * (4 * p + t4) + 8 * odd;
  return nibbles ? base + 2 * j + half : base + 4 * half + j;
}

// ------------------------------------------------------------------ exact fp64 ops
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }
// np.maximum / np.minimum on non-NaN operands
__device__ __forceinline__ double dmax(double a, double b) { return a >= b ? a : b; }
__device__ __forceinline__ double dmin(double a, double b) { return a <= b ? a : b; }

// ------------------------------------------------------------------ einsum order
// Running state of NumPy's einsum("ij,ij->i") inner loop for one row.  Feed
// the products of an 8-aligned block with `block8`, the tail with `tail`,
// then read `result()`.
struct EinsumAcc {
  double a0 = 0.0, a1 = 0.0;
  // p[k] = x[i+k]*y[i+k] (already rounded), k = 0..7
  __device__ __forceinline__ void block8(const double p[8]) {
    a0 = dadd(p[6], a0);
    a1 = dadd(p[7], a1);
    a0 = dadd(p[4], a0);
    a1 = dadd(p[5], a1);
    a0 = dadd(p[2], a0);
    a1 = dadd(p[3], a1);
    a0 = dadd(p[0], a0);
    a1 = dadd(p[1], a1);
  }
  // tail pair starting at an even offset; `has1` false when the pair is cut.
  __device__ __forceinline__ void pair(double p0, double p1, bool has1) {
    a0 = dadd(p0, a0);
    a1 = dadd(has1 ? p1 : 0.0, a1);
  }
  __device__ __forceinline__ double result() const { return dadd(0.0, dadd(a0, a1)); }
};

// Einsum of a row held contiguously in memory (any T convertible to double).
template <typename TA, typename TB>
__device__ inline double einsum_row(const TA* x, const TB* y, int n) {
  EinsumAcc acc;
  int i = 0;
  for (; i + 8 <= n; i += 8) {
    double p[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = dmul((double)x[i + k], (double)y[i + k]);
    acc.block8(p);
  }
  for (; i < n; i += 2) {
    double p0 = dmul((double)x[i], (double)y[i]);
    bool has1 = (i + 1) < n;
    double p1 = has1 ? dmul((double)x[i + 1], (double)y[i + 1]) : 0.0;
    acc.pair(p0, p1, has1);
  }
  return acc.result();
}

template <typename T>
__device__ inline double einsum_sq_row(const T* x, int n) {
  return einsum_row(x, x, n);
}

// ------------------------------------------------------------------ pairwise sum
// NumPy pairwise_sum over a contiguous float64 array of length n, evaluated
// sequentially by one thread (n is small: a vector of `dims` values).
__device__ inline double pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = dadd(res, a[i]);
    return res;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], a[i + j]);
  }
  double res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
  for (; i < n; ++i) res = dadd(res, a[i]);
  return res;
}

__device__ inline double pairwise_sum_seq(const double* a, int64_t n) {
  // explicit stack instead of recursion: (start, len, state)
  struct Frame { int64_t s, n; double left; int stage; };
  Frame st[48];
  int sp = 0;
  st[0] = {0, n, 0.0, 0};
  double ret = 0.0;
  while (sp >= 0) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf(a + f.s, f.n);
      --sp;
      continue;
    }
    int64_t n2 = f.n / 2;
    n2 -= n2 % 8;
    if (f.stage == 0) {
      f.stage = 1;
      st[sp + 1] = {f.s, n2, 0.0, 0};
      ++sp;
    } else if (f.stage == 1) {
      f.left = ret;
      f.stage = 2;
      st[sp + 1] = {f.s + n2, f.n - n2, 0.0, 0};
      ++sp;
    } else {
      ret = dadd(f.left, ret);
      --sp;
    }
  }
  return dadd(0.0, ret);
}

// ------------------------------------------------------------------ ordering keys
// (dist, id) lexicographic order used by every top-k in the reference
// (np.lexsort((ids, dists)), search.py:374, 386).
__device__ __forceinline__ bool key_less(double da, int64_t ia, double db, int64_t ib) {
  return da < db || (da == db && ia < ib);
}

}  // namespace ivrq
