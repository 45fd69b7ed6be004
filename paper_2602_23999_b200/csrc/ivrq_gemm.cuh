// Float64 "NT" GEMM tiles on the fp64 tensor cores:  C[m][n] = sum_k A(m,k) * B(n,k)
//
// The reference evaluates every distance identity and rotation with an
// OpenBLAS dgemm (clustering.py:50, search.py:241/422, index.py:238); parity of
// the discrete outputs (labels, probes, codes) needs float64 accumulation.
// On B200 the DMMA m16n8k16 path issues twice the float64 MACs per clock of
// the DFMA pipe (measured: 121.7 vs 61.8 MAC/clk/SM, tools/microbench.cu), so
// the tiles use mma.sync.m16n8k16.f64: 128x128 CTA tile, 32-deep k slab,
// 16 warps in a 4x4 grid each owning a 32x32 sub-tile (2x4 fragments), so an
// SM keeps 16 warps in flight (the 8-warp variant was latency bound at 12.5%
// occupancy, profiles/round1).
// Operand loaders and epilogues are functors so one kernel body serves the
// query rotation, probe distances, k-means labelling and residual rotation.
#pragma once

#include <algorithm>

#include "ivrq_common.cuh"

namespace ivrq {
namespace gemm {

constexpr int BM = 128, BN = 128, BK = 32, THREADS = 512;
constexpr int MF = 2, NF = 4;  // m16 / n8 fragments per warp
constexpr int LDA = BM + 8;  // k-major smem pitch (doubles): conflict-free fragment loads
constexpr int SMEM_BYTES = 2 * 2 * BK * LDA * (int)sizeof(double);  // double-buffered A and B

// Row-major [rows x ld] operand of element type T (float or double).
// load8: 8 consecutive k of row r as float64, through 128-bit loads when aligned.
template <typename T>
struct RowMajor {
  const T* p;
  int64_t rows;
  int64_t ld;
  __device__ __forceinline__ double operator()(int64_t r, int k) const { return (double)p[r * ld + k]; }
  __device__ __forceinline__ void load8(int64_t r, int k, int K, double (&out)[8]) const {
    const T* src = p + r * ld + k;
    constexpr int W = 16 / sizeof(T);
    if (k + 8 <= K && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
#pragma unroll
      for (int v = 0; v < 8 / W; ++v) {
        if constexpr (sizeof(T) == 4) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(src) + v);
          out[4 * v] = f.x;
          out[4 * v + 1] = f.y;
          out[4 * v + 2] = f.z;
          out[4 * v + 3] = f.w;
        } else {
          const double2 f = __ldg(reinterpret_cast<const double2*>(src) + v);
          out[2 * v] = f.x;
          out[2 * v + 1] = f.y;
        }
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) out[e] = (k + e < K) ? (double)src[e] : 0.0;
    }
  }
};

__device__ __forceinline__ void dmma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// Accumulator tile of one thread: acc[mf][nf][r], r = 0,1: row gid, cols 2t4+r;
// r = 2,3: row gid+8.  Rows: wm*32 + mf*16 (+gid), cols: wn*32 + nf*8 (+2t4).
struct Acc {
  double v[MF][NF][4];
};

__device__ __forceinline__ int64_t acc_row(int64_t m0, int mf, int r) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  return m0 + (w >> 2) * 32 + mf * 16 + (lane >> 2) + (r >= 2 ? 8 : 0);
}
__device__ __forceinline__ int64_t acc_col(int64_t n0, int nf, int r) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  return n0 + (w & 3) * 32 + nf * 8 + 2 * (lane & 3) + (r & 1);
}

// Per-CTA mainloop over K for rows [m0, m0+128) x cols [n0, n0+128).
template <typename LA, typename LB>
__device__ __forceinline__ void mainloop(const LA& la, int64_t M, const LB& lb, int64_t N, int K, int64_t m0,
                                         int64_t n0, double* smem, Acc& acc) {
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int gid = lane >> 2, t4 = lane & 3;
  const int wm = w >> 2, wn = w & 3;
  double* As = smem;                // [2][BK][LDA]
  double* Bs = smem + 2 * BK * LDA;  // [2][BK][LDA]
#pragma unroll
  for (int i = 0; i < MF; ++i)
#pragma unroll
    for (int j = 0; j < NF; ++j)
#pragma unroll
      for (int r = 0; r < 4; ++r) acc.v[i][j][r] = 0.0;

  // global->smem: each thread moves 8 consecutive k of one row per operand
  const int lr = tid >> 2, lk0 = (tid & 3) * 8;
  double ra[8], rb[8];
  auto load_regs = [&](int k0) {
    const int64_t gm = m0 + lr, gn = n0 + lr;
    if (gm < M) {
      la.load8(gm, k0 + lk0, K, ra);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) ra[e] = 0.0;
    }
    if (gn < N) {
      lb.load8(gn, k0 + lk0, K, rb);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) rb[e] = 0.0;
    }
  };
  auto store_smem = [&](int buf) {
    double* a = As + buf * BK * LDA;
    double* b = Bs + buf * BK * LDA;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      a[(lk0 + e) * LDA + lr] = ra[e];
      b[(lk0 + e) * LDA + lr] = rb[e];
    }
  };

  const int nk = (K + BK - 1) / BK;
  load_regs(0);
  store_smem(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_regs((kt + 1) * BK);
#pragma unroll
    for (int ks = 0; ks < BK / 16; ++ks) {
      const double* a = As + buf * BK * LDA + ks * 16 * LDA;
      const double* b = Bs + buf * BK * LDA + ks * 16 * LDA;
      // B fragments of the warp's column blocks: b_j = B[k = t4 + 4j][n = gid]
      double bf[NF][4];
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[nf][j] = b[(t4 + 4 * j) * LDA + wn * 32 + nf * 8 + gid];
#pragma unroll
      for (int mf = 0; mf < MF; ++mf) {
        // A fragment: a_{2j} = A[row gid][k = t4 + 4j], a_{2j+1} = A[row gid + 8][k = t4 + 4j]
        double af[8];
        const int rbase = wm * 32 + mf * 16 + gid;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          af[2 * j] = a[(t4 + 4 * j) * LDA + rbase];
          af[2 * j + 1] = a[(t4 + 4 * j) * LDA + rbase + 8];
        }
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) dmma16816(acc.v[mf][nf], af, bf[nf]);
      }
    }
    if (kt + 1 < nk) store_smem(buf ^ 1);
    __syncthreads();
  }
}

// Plain tiled GEMM: grid (ceil(N/BN), ceil(M/BM)); epilogue(row, col, acc).
template <typename LA, typename LB, typename EPI>
__global__ void __launch_bounds__(THREADS, 1) gemm_kernel(LA la, int64_t M, LB lb, int64_t N, int K, EPI epi,
                                                          int64_t n_base) {
  extern __shared__ __align__(16) double smem_d[];
  // row tiles on grid.x (up to 2^31-1: 10M rows is 78K tiles), column tiles on
  // grid.y (launched in slices of 65535 tiles from n_base)
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int64_t n0 = n_base + (int64_t)blockIdx.y * BN;
  Acc acc;
  mainloop(la, M, lb, N, K, m0, n0, smem_d, acc);
#pragma unroll
  for (int mf = 0; mf < MF; ++mf)
#pragma unroll
    for (int nf = 0; nf < NF; ++nf)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t row = acc_row(m0, mf, r), col = acc_col(n0, nf, r);
        if (row < M && col < N) epi(row, col, acc.v[mf][nf][r]);
      }
}

// Row-argmin GEMM: one CTA per 128-row block sweeps every column tile and
// keeps, per row, the first column minimising dist(row, col, acc).
// Writes labels[row] and dmin[row] = max(best, 0).
template <typename LA, typename LB, typename DIST>
__global__ void __launch_bounds__(THREADS, 1) gemm_argmin_kernel(LA la, int64_t M, LB lb, int64_t N, int K,
                                                                 DIST dist, int32_t* labels, double* dmin) {
  extern __shared__ __align__(16) double smem_d[];
  __shared__ double red_d[4][BM];
  __shared__ int32_t red_i[4][BM];
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double best_d[2 * MF];
  int32_t best_i[2 * MF];  // [mf*2 + (r>=2)]
#pragma unroll
  for (int i = 0; i < 2 * MF; ++i) {
    best_d[i] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    best_i[i] = 0x7fffffff;
  }
  Acc acc;
  for (int64_t n0 = 0; n0 < N; n0 += BN) {
    mainloop(la, M, lb, N, K, m0, n0, smem_d, acc);
#pragma unroll
    for (int mf = 0; mf < MF; ++mf)
#pragma unroll
      for (int nf = 0; nf < NF; ++nf)
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int64_t row = acc_row(m0, mf, r), col = acc_col(n0, nf, r);
          if (row < M && col < N) {
            const double dv = dist(row, col, acc.v[mf][nf][r]);
            const int s = mf * 2 + (r >> 1);
            if (dv < best_d[s] || (dv == best_d[s] && (int32_t)col < best_i[s])) {
              best_d[s] = dv;
              best_i[s] = (int32_t)col;
            }
          }
        }
  }
  // reduce over the 4 lanes (t4) sharing a row, then over the 4 column warps
#pragma unroll
  for (int s = 0; s < 2 * MF; ++s) {
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, best_d[s], o);
      const int32_t oi = __shfl_xor_sync(0xffffffffu, best_i[s], o);
      if (od < best_d[s] || (od == best_d[s] && oi < best_i[s])) {
        best_d[s] = od;
        best_i[s] = oi;
      }
    }
  }
  if ((lane & 3) == 0) {
#pragma unroll
    for (int s = 0; s < 2 * MF; ++s) {
      const int lrow = (w >> 2) * 32 + (s >> 1) * 16 + (lane >> 2) + (s & 1) * 8;
      red_d[w & 3][lrow] = best_d[s];
      red_i[w & 3][lrow] = best_i[s];
    }
  }
  __syncthreads();
  if (threadIdx.x < BM) {
    const int lrow = threadIdx.x;
    double bd = red_d[0][lrow];
    int32_t bi = red_i[0][lrow];
    for (int t = 1; t < 4; ++t) {
      const double d = red_d[t][lrow];
      const int32_t ii = red_i[t][lrow];
      if (d < bd || (d == bd && ii < bi)) {
        bd = d;
        bi = ii;
      }
    }
    const int64_t r = m0 + lrow;
    if (r < M) {
      labels[r] = bi;
      if (dmin) dmin[r] = dmax(bd, 0.0);
    }
  }
}

template <typename LA, typename LB, typename EPI>
inline int launch_gemm(const LA& la, int64_t M, const LB& lb, int64_t N, int K, const EPI& epi, cudaStream_t s,
                       const char* what) {
  if (M == 0 || N == 0) return IVRQ_OK;
  auto kern = gemm_kernel<LA, LB, EPI>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  const int64_t nt = ceil_div(N, BN);
  for (int64_t t0 = 0; t0 < nt; t0 += 65535) {
    dim3 grid((unsigned)ceil_div(M, BM), (unsigned)std::min<int64_t>(65535, nt - t0));
    kern<<<grid, THREADS, SMEM_BYTES, s>>>(la, M, lb, N, K, epi, t0 * BN);
  }
  return check_launch(what);
}

template <typename LA, typename LB, typename DIST>
inline int launch_gemm_argmin(const LA& la, int64_t M, const LB& lb, int64_t N, int K, const DIST& dist,
                              int32_t* labels, double* dmin, cudaStream_t s, const char* what) {
  if (M == 0) return IVRQ_OK;
  auto kern = gemm_argmin_kernel<LA, LB, DIST>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  dim3 grid((unsigned)ceil_div(M, BM));
  kern<<<grid, THREADS, SMEM_BYTES, s>>>(la, M, lb, N, K, dist, labels, dmin);
  return check_launch(what);
}

}  // namespace gemm
}  // namespace ivrq
