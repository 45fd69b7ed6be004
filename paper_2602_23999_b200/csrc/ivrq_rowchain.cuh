// Row-wise float64 reductions in NumPy's einsum order,
// at memory speed.
//
// np.einsum("ij,ij->i") keeps two independent accumulator lanes per row; here
// each lane is one thread (threads 2r and 2r+1 own row r), so a row's two
// dependent add chains run in parallel.  Rows are staged through shared
// memory in [ROWS x CH] tiles loaded with 128-bit coalesced loads, all issued
// before any is consumed.  The per-element product is a functor so the same
// body serves |x|^2, |x - c|^2 with a broadcast centre, and residuals of
// gathered rows.
#pragma once

#include "ivrq_common.cuh"

namespace ivrq {
namespace rowchain {

constexpr int ROWS = 64;              // rows per CTA
constexpr int CH = 64;                // dims per chunk (multiple of 8: einsum blocks stay whole)
constexpr int THREADS = 2 * ROWS;     // two accumulator lanes per row

template <typename T>
struct Tile {
  static constexpr int VEC = 16 / sizeof(T);  // elements per 128-bit load
  static constexpr int PAD = CH + VEC;        // row pitch: 16-byte aligned, spreads banks
  T v[ROWS][PAD];
};

template <typename T>
struct Vec16;
template <>
struct Vec16<float> {
  using type = float4;
};
template <>
struct Vec16<double> {
  using type = double2;
};

// Stage rows [row0, row0+ROWS) x dims [c0, c0+cw) of a matrix whose row r
// starts at src(r).  vec: every row pointer is 16-byte aligned and cw is a
// multiple of the vector width.
template <typename T, typename RowPtr>
__device__ __forceinline__ void stage_tile(Tile<T>& tile, const RowPtr& src, int64_t row0, int64_t n, int c0, int cw,
                                           bool vec) {
  using V = typename Vec16<T>::type;
  constexpr int W = Tile<T>::VEC;
  const int t = threadIdx.x;
  if (vec) {
    constexpr int PER = ROWS * CH / W / THREADS;
    V v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = t + u * THREADS;
      const int rr = idx / (CH / W), cv = idx % (CH / W);
      const int64_t gr = row0 + rr;
      if (gr < n && cv * W < cw) {
        v[u] = __ldg(reinterpret_cast<const V*>(src(gr) + c0) + cv);
      } else {
        T* z = reinterpret_cast<T*>(&v[u]);
#pragma unroll
        for (int e = 0; e < W; ++e) z[e] = (T)0;
      }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = t + u * THREADS;
      const int rr = idx / (CH / W), cv = idx % (CH / W);
      *reinterpret_cast<V*>(&tile.v[rr][cv * W]) = v[u];
    }
  } else {
    constexpr int PER = ROWS * CH / THREADS;
    T v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = t + u * THREADS;
      const int rr = idx / CH, cc = idx % CH;
      const int64_t gr = row0 + rr;
      v[u] = (gr < n && cc < cw) ? __ldg(src(gr) + c0 + cc) : (T)0;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int idx = t + u * THREADS;
      tile.v[idx / CH][idx % CH] = v[u];
    }
  }
}

// Walk one accumulator lane of a row through a staged chunk in einsum order.
// prod(k) returns the rounded product for chunk-local dim k.
template <typename Prod>
__device__ __forceinline__ double chain_chunk(double acc, int lane, int cw, const Prod& prod) {
  int i = 0;
  for (; i + 8 <= cw; i += 8) {
#pragma unroll
    for (int blk = 3; blk >= 0; --blk) acc = dadd(prod(i + 2 * blk + lane), acc);
  }
  for (; i < cw; i += 2) {  // tail pairs: only in the last chunk (CH % 8 == 0)
    const int kk = i + lane;
    acc = dadd(kk < cw ? prod(kk) : 0.0, acc);
  }
  return acc;
}

// Combine the two lanes of a row: 0.0 + (acc0 + acc1); valid on both threads.
__device__ __forceinline__ double finish(double acc) {
  const double other = __shfl_xor_sync(0xffffffffu, acc, 1);
  const double a0 = (threadIdx.x & 1) ? other : acc;
  const double a1 = (threadIdx.x & 1) ? acc : other;
  return dadd(0.0, dadd(a0, a1));
}

}  // namespace rowchain
}  // namespace ivrq
