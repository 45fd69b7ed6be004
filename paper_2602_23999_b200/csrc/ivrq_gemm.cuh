// Float64 "NT" GEMM tiles:  C[m][n] = sum_k A(m,k) * B(n,k)
//
// The reference evaluates every distance identity and rotation with an
// OpenBLAS dgemm (clustering.py:50, search.py:241/422, index.py:238); parity of
// the discrete outputs (labels, probes, codes) needs float64 accumulation, so
// these tiles run on the float64 FMA pipe.  128x128 CTA tile, 16-deep k-slab,
// 256 threads each owning an 8x8 register tile split into two 4-row/4-column
// halves 64 apart so that the 128-bit shared loads are bank-conflict free.
// Operand loaders and epilogues are functors so one kernel body serves the
// query rotation, probe distances, k-means labelling and residual rotation.
#pragma once

#include "ivrq_common.cuh"

namespace ivrq {
namespace gemm {

constexpr int BM = 128, BN = 128, BK = 16, THREADS = 256;
constexpr int SMEM_BYTES = 2 * 2 * BK * BM * (int)sizeof(double);  // double-buffered A and B

// Row-major [rows x ld] operand of element type T (float or double).
template <typename T>
struct RowMajor {
  const T* p;
  int64_t rows;
  int64_t ld;
  __device__ __forceinline__ double operator()(int64_t r, int k) const { return (double)p[r * ld + k]; }
};

// Per-CTA mainloop; accumulates rows [m0, m0+128) x cols [n0, n0+128) into acc.
// acc[i][j]: i<4 -> row m0 + ty*4+i, i>=4 -> row m0 + 64 + ty*4 + (i-4); same for j/cols.
template <typename LA, typename LB>
__device__ __forceinline__ void mainloop(const LA& la, int64_t M, const LB& lb, int64_t N, int K,
                                         int64_t m0, int64_t n0, double* smem, double (&acc)[8][8]) {
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  double* As = smem;                 // [2][BK][BM]
  double* Bs = smem + 2 * BK * BM;   // [2][BK][BN]
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  // global->smem mapping: each thread loads 8 (row, k) elements per operand:
  // row = tid / 2, k = (tid % 2) * 8 + e
  const int lr = tid / 2;
  const int lk0 = (tid % 2) * 8;
  double ra[8], rb[8];
  auto load_regs = [&](int k0) {
    int64_t gm = m0 + lr, gn = n0 + lr;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      int k = k0 + lk0 + e;
      ra[e] = (gm < M && k < K) ? la(gm, k) : 0.0;
      rb[e] = (gn < N && k < K) ? lb(gn, k) : 0.0;
    }
  };
  auto store_smem = [&](int buf) {
    double* a = As + buf * BK * BM;
    double* b = Bs + buf * BK * BN;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      a[(lk0 + e) * BM + lr] = ra[e];
      b[(lk0 + e) * BN + lr] = rb[e];
    }
  };

  const int nk = (K + BK - 1) / BK;
  load_regs(0);
  store_smem(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_regs((kt + 1) * BK);
    const double* a = As + buf * BK * BM;
    const double* b = Bs + buf * BK * BN;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      double av[8], bv[8];
      const double2* ap0 = reinterpret_cast<const double2*>(a + k * BM + ty * 4);
      const double2* ap1 = reinterpret_cast<const double2*>(a + k * BM + 64 + ty * 4);
      const double2* bp0 = reinterpret_cast<const double2*>(b + k * BN + tx * 4);
      const double2* bp1 = reinterpret_cast<const double2*>(b + k * BN + 64 + tx * 4);
      double2 t;
      t = ap0[0]; av[0] = t.x; av[1] = t.y;
      t = ap0[1]; av[2] = t.x; av[3] = t.y;
      t = ap1[0]; av[4] = t.x; av[5] = t.y;
      t = ap1[1]; av[6] = t.x; av[7] = t.y;
      t = bp0[0]; bv[0] = t.x; bv[1] = t.y;
      t = bp0[1]; bv[2] = t.x; bv[3] = t.y;
      t = bp1[0]; bv[4] = t.x; bv[5] = t.y;
      t = bp1[1]; bv[6] = t.x; bv[7] = t.y;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store_smem(buf ^ 1);
    __syncthreads();
  }
}

__device__ __forceinline__ int64_t acc_row(int64_t m0, int i) {
  const int ty = threadIdx.x / 16;
  return m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
}
__device__ __forceinline__ int64_t acc_col(int64_t n0, int j) {
  const int tx = threadIdx.x % 16;
  return n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
}

// Plain tiled GEMM: grid (ceil(N/BN), ceil(M/BM)); epilogue(row, col, acc).
template <typename LA, typename LB, typename EPI>
__global__ void __launch_bounds__(THREADS) gemm_kernel(LA la, int64_t M, LB lb, int64_t N, int K, EPI epi) {
  extern __shared__ __align__(16) double smem_d[];
  const int64_t m0 = (int64_t)blockIdx.y * BM;
  const int64_t n0 = (int64_t)blockIdx.x * BN;
  double acc[8][8];
  mainloop(la, M, lb, N, K, m0, n0, smem_d, acc);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int64_t r = acc_row(m0, i);
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      int64_t c = acc_col(n0, j);
      if (c < N) epi(r, c, acc[i][j]);
    }
  }
}

// Row-argmin GEMM: one CTA per 128-row block sweeps every column tile and
// keeps, per row, the first column minimising dist(row, col, acc).
// Writes labels[row] and dmin[row] = max(best, 0).
template <typename LA, typename LB, typename DIST>
__global__ void __launch_bounds__(THREADS) gemm_argmin_kernel(LA la, int64_t M, LB lb, int64_t N, int K,
                                                              DIST dist, int32_t* labels, double* dmin) {
  extern __shared__ __align__(16) double smem_d[];
  __shared__ double red_d[16][BM];
  __shared__ int32_t red_i[16][BM];
  const int64_t m0 = (int64_t)blockIdx.x * BM;
  const int tx = threadIdx.x % 16;
  double best_d[8];
  int32_t best_i[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    best_d[i] = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    best_i[i] = 0x7fffffff;
  }
  double acc[8][8];
  for (int64_t n0 = 0; n0 < N; n0 += BN) {
    mainloop(la, M, lb, N, K, m0, n0, smem_d, acc);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int64_t r = acc_row(m0, i);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int64_t c = acc_col(n0, j);
        if (r < M && c < N) {
          double d = dist(r, c, acc[i][j]);
          if (d < best_d[i] || (d == best_d[i] && (int32_t)c < best_i[i])) {
            best_d[i] = d;
            best_i[i] = (int32_t)c;
          }
        }
      }
    }
  }
  // reduce over the 16 column-threads sharing each row
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    int ty = threadIdx.x / 16;
    int lrow = i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4);
    red_d[tx][lrow] = best_d[i];
    red_i[tx][lrow] = best_i[i];
  }
  __syncthreads();
  if (threadIdx.x < BM) {
    int lrow = threadIdx.x;
    double bd = red_d[0][lrow];
    int32_t bi = red_i[0][lrow];
    for (int t = 1; t < 16; ++t) {
      double d = red_d[t][lrow];
      int32_t ii = red_i[t][lrow];
      if (d < bd || (d == bd && ii < bi)) {
        bd = d;
        bi = ii;
      }
    }
    int64_t r = m0 + lrow;
    if (r < M) {
      labels[r] = bi;
      if (dmin) dmin[r] = dmax(bd, 0.0);
    }
  }
}

template <typename LA, typename LB, typename EPI>
inline int launch_gemm(const LA& la, int64_t M, const LB& lb, int64_t N, int K, const EPI& epi,
                       cudaStream_t s, const char* what) {
  if (M == 0 || N == 0) return IVRQ_OK;
  auto kern = gemm_kernel<LA, LB, EPI>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  dim3 grid((unsigned)ceil_div(N, BN), (unsigned)ceil_div(M, BM));
  kern<<<grid, THREADS, SMEM_BYTES, s>>>(la, M, lb, N, K, epi);
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
