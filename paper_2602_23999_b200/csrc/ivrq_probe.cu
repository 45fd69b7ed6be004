// Coarse probe on the 5th-generation tensor cores (select_clusters,
// search.py:226-244): exact top-n_probe of d = max((|q|^2 + |c|^2) - 2<q,c>, 0).
//
//  1. digits: every query row (float64) and centroid row (float32) becomes a
//     28-bit fixed-point integer vector relative to its row maximum,
//     x = X * 2^(e-27) + r (|r| <= 2^(e-28)), split into 4 balanced base-128
//     int8 digits X = sum_s D_s 128^(3-s).
//  2. tc_probe_kernel: <Q, C> exactly from int8 tcgen05 MMAs.  A rows are
//     (query, digit s) pairs (32 queries x 4), B rows (centroid, digit t)
//     pairs (64 centroids x 4): one M=128, N=256 MMA per 32-dim step gives all
//     16 digit products; the epilogue assembles them exactly (two int64
//     halves, one float64 rounding) and writes float32 bounds L <= d <= U that
//     provably bracket the float64 distance the rescoring below computes
//     (representation error (s_q s_c / 2)(|Q|_1 + |C|_1 + K/2), doubled, plus
//     float64 rounding slack).
//  3. probe_rescore_kernel: per query, tau = n_probe-th smallest U (radix
//     select), candidates = {c : L_c <= tau} (a superset of the exact top
//     n_probe), their float64 distances recomputed by a warp-wide dot product,
//     and the n_probe smallest by (distance, id) kept (ordered by id or by
//     (distance, id)).
#include <algorithm>

#include "ivrq_common.cuh"
#include "ivrq_tc.cuh"

namespace ivrq {
namespace probe {

// NDIG digits per row: queries per tile 128 / NDIG (A rows = TMEM lanes), centroids 256 / NDIG (N = 256)
template <int NDIG> constexpr int QT_ = 128 / NDIG;
template <int NDIG> constexpr int CT_ = 256 / NDIG;
constexpr int KC = 128;  // K bytes per stage
constexpr int ST = 3;    // stages
constexpr int EPW = 16;       // epilogue warps (4 per TMEM lane quarter: the epilogue, not the MMAs, bounds the tile)
constexpr int THREADS = 32 * (2 + EPW);  // warp 0 TMA, warp 1 MMA, warps 2.. epilogue
constexpr int NCOL = 256;  // accumulator columns per tile

// ---------------------------------------------------------------- digits
// One warp per row.  out: digit s of row r at out[(s * rows + r) * kp + k] (queries,
// slice_major) or out[(4 r + s) * kp + k] (centroids).  e_out: scale exponent e
// (x = X 2^(e-27)), l1_out: |X|_1.
template <typename T, int NDIG>
__global__ void digits_kernel(const T* __restrict__ x, int64_t rows, int d, int kp, int slice_major,
                              int8_t* __restrict__ out, int32_t* __restrict__ e_out, double* __restrict__ l1_out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const T* xr = x + r * d;
  double mx = 0.0;
  for (int k = lane; k < d; k += 32) mx = fmax(mx, fabs((double)xr[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
  double l1 = 0.0;
  for (int k = lane; k < kp; k += 32) {
    long long X = k < d ? llrint(ldexp((double)xr[k], 7 * NDIG - 1 - e)) : 0;  // |X| <= 2^(7 NDIG - 1)
    l1 += (double)(X < 0 ? -X : X);
    int8_t dg[NDIG];
#pragma unroll
    for (int s = NDIG - 1; s >= 0; --s) {
      const long long rr = ((X + 64) & 127) - 64;
      dg[s] = (int8_t)rr;
      X = (X - rr) >> 7;
    }
    dg[0] = (int8_t)(dg[0] + (int8_t)(X * 128));  // the top digit absorbs the remainder (|D_0| <= 65)
#pragma unroll
    for (int s = 0; s < NDIG; ++s) {
      const int64_t row = slice_major ? (int64_t)s * rows + r : NDIG * r + s;
      out[row * kp + k] = dg[s];
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) l1 += __shfl_xor_sync(0xffffffffu, l1, o);
  if (lane == 0) {
    e_out[r] = e;
    l1_out[r] = l1;
  }
}

// ---------------------------------------------------------------- bounds GEMM
struct TpArgs {
  CUtensorMap map_q;  // query digits  [nq rows x 4 digits, kp], box 128 B x 128 rows
  CUtensorMap map_c;  // centroid digits [4 * nlist rows x kp], box 128 B x 256 rows
  int64_t nq, q0, nrows;  // this chunk: query rows [q0, q0 + nrows)
  int nlist, kp, d;
  const double* q_sq;   // [nq]
  const double* c_sq;   // [nlist]
  const int32_t* q_e;
  const int32_t* c_e;
  const double* q_l1;
  const double* c_l1;
  float* bnd;           // [nrows][2][nlist]: lower bounds L, then upper bounds U
};

// 2^e as a float64 (exact multiplier for ldexp when 2^e is normal)
__device__ __forceinline__ double pow2(int e) {
  return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(e + 1023) << 52) : ldexp(1.0, e);
}

template <int NDIG>
__global__ void __launch_bounds__(THREADS, 1) tc_probe_kernel(const __grid_constant__ TpArgs a) {
  constexpr int QT = QT_<NDIG>, CT = CT_<NDIG>;
  extern __shared__ __align__(1024) unsigned char psm_raw[];
  unsigned char* psm = reinterpret_cast<unsigned char*>(((uintptr_t)psm_raw + 1023) & ~(uintptr_t)1023);
  int8_t* sA = reinterpret_cast<int8_t*>(psm);                       // [ST][128 rows x 128 B]
  int8_t* sB = reinterpret_cast<int8_t*>(psm + ST * 128 * KC);       // [ST][256 rows x 128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(psm + ST * (128 + NCOL) * KC);
  uint64_t* full = bars;
  uint64_t* empty = bars + ST;
  uint64_t* accf = bars + 2 * ST;
  uint64_t* acce = bars + 2 * ST + 2;
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(bars + 2 * ST + 4);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&accf[i], 1);
      tc::mbar_init(&acce[i], 32 * EPW);
    }
    tc::fence_mbar_init();
  }
  if (wid == 1) tc::tmem_alloc(s_taddr, 2 * NCOL);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *s_taddr;
  const int nkc = (a.kp + KC - 1) / KC;
  const int nqt = (int)ceil_div(a.nrows, QT), nct = (int)ceil_div(a.nlist, CT);
  const int ntiles = nqt * nct;
  const uint32_t idesc = tc::idesc_i8(128, NCOL, true, true);
  if (wid == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int qt = tile / nct, ct = tile % nct;  // centroid tiles fastest: the query tile stays in L2
        const int64_t qrow = a.q0 + (int64_t)qt * QT;
        for (int kc = 0; kc < nkc; ++kc, ++it) {
          const int st = it % ST;
          tc::mbar_wait(&empty[st], ((it / ST) & 1) ^ 1);
          tc::mbar_expect_tx(&full[st], (128 + NCOL) * KC);
          // A rows 4 j + s: the tile's 32 queries x 4 digits, one box
          tc::tma_load_2d(sA + st * 128 * KC, &a.map_q, kc * KC, (int)(NDIG * qrow), &full[st]);
          tc::tma_load_2d(sB + st * NCOL * KC, &a.map_c, kc * KC, ct * NCOL, &full[st]);
        }
      }
    }
  } else if (wid == 1) {
    uint32_t it = 0, tcount = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
      const int ab = tcount & 1;
      tc::mbar_wait(&acce[ab], ((tcount >> 1) & 1) ^ 1);
      tc::fence_after_sync();
      for (int kc = 0; kc < nkc; ++kc, ++it) {
        const int st = it % ST;
        tc::mbar_wait(&full[st], (it / ST) & 1);
        tc::fence_after_sync();
        if (lane == 0) {
          const int ks = (min(KC, a.kp - kc * KC) + 31) / 32;
          for (int s2 = 0; s2 < ks; ++s2) {
            const uint64_t ad = tc::smem_desc_sw128(sA + st * 128 * KC + 32 * s2);
            const uint64_t bd = tc::smem_desc_sw128(sB + st * NCOL * KC + 32 * s2);
            tc::mma_i8(tbase + ab * NCOL, ad, bd, idesc, kc > 0 || s2 > 0);
          }
          tc::commit(&empty[st]);
          if (kc == nkc - 1) tc::commit(&accf[ab]);
        }
        __syncwarp();
      }
    }
  } else {
    // epilogue: TMEM lane = A row = NDIG j + s (query j of the tile, digit s); column NDIG c + t
    const int quarter = wid & 3;
    constexpr int PARTS = EPW / 4;      // warps per TMEM lane quarter
    const int part = (wid - 2) >> 2;  // which part of the tile's centroids this warp finishes
    const int s = lane % NDIG;
    const int jq = quarter * (32 / NDIG) + lane / NDIG;  // query within the tile
    const int b1 = (lane >> 1) & 1, b0 = lane & 1;
    constexpr int CPC = 32 / NDIG;  // centroids per 32-column chunk
    uint32_t tcount = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++tcount) {
      const int ab = tcount & 1;
      const int qt = tile / nct, ct = tile % nct;
      const int64_t qr = (int64_t)qt * QT + jq;  // row within the chunk
      const int64_t qg = a.q0 + qr;
      double qsq = 0.0, ql1 = 0.0;
      int qe = 0;
      if (qr < a.nrows) {
        qsq = a.q_sq[qg];
        ql1 = a.q_l1[qg];
        qe = a.q_e[qg];
      }
      // the tile's centroid scalars, staged while the MMAs run (double-buffered by tile parity)
      __shared__ double s_csq[2][128], s_cl1[2][128];
      __shared__ int32_t s_ce[2][128];
      __shared__ __align__(16) float s_stage[EPW * 2 * 16 * 16];  // per epilogue warp: 16 queries x 16 centroids, L and U
      {
        const int et = tid - 64;  // 0..32*EPW-1
        if (et < CT) {
          const int64_t c = (int64_t)ct * CT + et;
          s_csq[ab][et] = c < a.nlist ? __ldg(a.c_sq + c) : 0.0;
          s_cl1[ab][et] = c < a.nlist ? __ldg(a.c_l1 + c) : 0.0;
          s_ce[ab][et] = c < a.nlist ? __ldg(a.c_e + c) : 0;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * EPW) : "memory");  // epilogue warps only
      }
      tc::mbar_wait(&accf[ab], (tcount >> 1) & 1);
      tc::fence_after_sync();
      // bounds of (query jq, centroid cl): float64 with exact power-of-two scalings, rounded outwards
      auto bounds = [&](int cl, double dot_scaled_hi, double dot_scaled_lo, int shift_hi, float& lo_b, float& up_b) {
        const int sc = qe + s_ce[ab][cl] - 2 * (7 * NDIG - 1);  // s_q s_c
        const double csq = s_csq[ab][cl];
        const double p2 = pow2(sc);
        double dot;
        if constexpr (NDIG == 2) {  // the whole sum is the low part (hi == 0): the same value, fewer ops
          dot = dmul(dot_scaled_lo, p2);
        } else {
          dot = dadd(dmul(dot_scaled_hi, pow2(sc + shift_hi)), dmul(dot_scaled_lo, p2));
        }
        const double dist = dsub(dadd(qsq, csq), dmul(2.0, dot));
        const double rep = dmul(ql1 + s_cl1[ab][cl] + 0.5 * a.d, p2);  // 2 (s_q s_c / 2)(|Q|_1+|C|_1+K/2)
        const double slack = (qsq + csq + 2.0 * fabs(dot)) * 0x1p-40;
        const double E = rep * 1.0000001 + slack;
        lo_b = __double2float_rd(fmax(dist - E, 0.0));
        up_b = __double2float_ru(fmax(dist + E, 0.0));
      };
      auto emit = [&](int cl, double dot_scaled_hi, double dot_scaled_lo, int shift_hi) {
        const int64_t c = (int64_t)ct * CT + cl;
        if (qr < a.nrows && c < a.nlist) {
          float lb, ub;
          bounds(cl, dot_scaled_hi, dot_scaled_lo, shift_hi, lb, ub);
          float* br = a.bnd + qr * 2 * (int64_t)a.nlist;
          br[c] = lb;
          br[a.nlist + c] = ub;
        }
      };
      // NDIG == 2 stages each 32-column chunk (16 queries x 16 centroids, L and U) in shared memory
      // so that every query row is written as two 64-byte runs
      float* stg = s_stage + (wid - 2) * (2 * 16 * 16);
      for (int cc0 = part * (CT / PARTS); cc0 < (part + 1) * (CT / PARTS); cc0 += CPC) {
        uint32_t v[32];
        tc::tmem_ld32(tbase + ((uint32_t)(quarter * 32) << 16) + ab * NCOL + NDIG * cc0, v);
        tc::tmem_ld_wait();
        if constexpr (NDIG == 4) {
          // weight 128^(6-s-t): hi collects s+t <= 2 (weight 128^(2-s-t)), lo s+t >= 3 (128^(6-s-t))
          long long H[8], L[8];
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            long long h = 0, l = 0;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const long long x = (long long)(int)v[4 * c8 + t];
              const int u = s + t;
              if (u <= 2) h += x << (7 * (2 - u));
              else l += x << (7 * (6 - u));
            }
            H[c8] = h;
            L[c8] = l;
          }
          // sum over the query's 4 digit lanes, transposed: lane s ends with centroids 2s, 2s+1
          long long H1[4], L1[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const long long sh = b1 ? H[i] : H[i + 4], sl = b1 ? L[i] : L[i + 4];
            H1[i] = (b1 ? H[i + 4] : H[i]) + __shfl_xor_sync(0xffffffffu, sh, 2);
            L1[i] = (b1 ? L[i + 4] : L[i]) + __shfl_xor_sync(0xffffffffu, sl, 2);
          }
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const long long sh = b0 ? H1[i] : H1[i + 2], sl = b0 ? L1[i] : L1[i + 2];
            const long long Ht = (b0 ? H1[i + 2] : H1[i]) + __shfl_xor_sync(0xffffffffu, sh, 1);
            const long long Lt = (b0 ? L1[i + 2] : L1[i]) + __shfl_xor_sync(0xffffffffu, sl, 1);
            emit(cc0 + 2 * s + i, (double)Ht, (double)Lt, 28);
          }
        } else {
          // NDIG == 2: weight 128^(2-s-t), the whole sum fits an int64 (|.| < 2^38)
          long long P[16];
#pragma unroll
          for (int c16 = 0; c16 < 16; ++c16) {
            long long p = 0;
#pragma unroll
            for (int t = 0; t < 2; ++t) p += ((long long)(int)v[2 * c16 + t]) << (7 * (2 - s - t));
            P[c16] = p;
          }
          // sum over the 2 digit lanes, transposed: lane s ends with centroids 8s .. 8s+7
          const int jl = lane >> 1;  // query within the warp's 16
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const long long sh = b0 ? P[i] : P[i + 8];
            const long long Pt = (b0 ? P[i + 8] : P[i]) + __shfl_xor_sync(0xffffffffu, sh, 1);
            float lb, ub;
            bounds(cc0 + 8 * s + i, 0.0, (double)Pt, 0, lb, ub);
            stg[jl * 16 + 8 * s + i] = lb;
            stg[256 + jl * 16 + 8 * s + i] = ub;
          }
          __syncwarp();
          const int64_t cb = (int64_t)ct * CT + cc0;  // the chunk's first centroid (a multiple of 16)
          if ((a.nlist & 3) == 0 && cb + 16 <= a.nlist) {
            // 16-byte stores: lane = (query of 4, L/U, 4-centroid quad), four passes over the 16 queries
            const int c4 = lane & 3, which = (lane >> 2) & 1;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              const int j = h * 4 + (lane >> 3);
              const int64_t qrow = (int64_t)qt * QT + quarter * 16 + j;
              if (qrow < a.nrows)
                *reinterpret_cast<float4*>(a.bnd + (qrow * 2 + which) * (int64_t)a.nlist + cb + 4 * c4) =
                    *reinterpret_cast<const float4*>(stg + which * 256 + j * 16 + 4 * c4);
            }
          } else {
            const int ci = lane & 15, which = lane >> 4;  // lanes 0-15: L, 16-31: U
            const int64_t c = cb + ci;
#pragma unroll 4
            for (int j = 0; j < 16; ++j) {
              const int64_t qrow = (int64_t)qt * QT + quarter * 16 + j;
              if (qrow < a.nrows && c < a.nlist)
                a.bnd[qrow * 2 * (int64_t)a.nlist + (int64_t)which * a.nlist + c] = stg[which * 256 + j * 16 + ci];
            }
          }
          __syncwarp();
        }
      }
      tc::fence_before_sync();
      tc::mbar_arrive(&acce[ab]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 1) tc::tmem_dealloc(tbase, 2 * NCOL);
}

size_t tp_smem_bytes() { return 1024 + (size_t)ST * (128 + NCOL) * KC + 256; }

// ---------------------------------------------------------------- rescoring
// One CTA per query: tau = n_probe-th smallest U (3-pass radix on the float32
// bits), candidates L <= tau, float64 distances recomputed (warp per candidate,
// fixed lane order), the n_probe smallest by (distance, id) written out.  If the
// candidate set overflows shared memory (pathological ties), every distance of
// the row is recomputed in float64 into the row's own storage and selected by
// an exact radix select instead.
constexpr int RS_THREADS = 256;
constexpr int MAX_CAND = 1024;
constexpr int RS_REG = 64;  // U values per thread held in registers (nlist <= 16384)

__device__ __forceinline__ double exact_dist(const double* qv, const float* cv, int d, double qs, double cs) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  for (int k = lane; k < d; k += 32) acc = fma(qv[k], (double)cv[k], acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  return dmax(dsub(dadd(qs, cs), dmul(2.0, acc)), 0.0);
}

// k-th smallest (1-based) key among n keys (bits of non-negative numbers): MSB-first radix of
// 8-bit digits; the bin holding the k-th is found by a warp-parallel prefix over the histogram.
// need_out = how many keys equal to the result are among the k smallest.
template <typename K, typename Get>
__device__ K radix_kth(int n, int k, int total_bits, int32_t* hist, Get get, int& need_out) {
  __shared__ unsigned long long s_prefix;
  __shared__ int32_t s_need;
  const int tid = threadIdx.x, lane = tid & 31;
  unsigned long long prefix = 0, mask = 0;
  int need = k;
  for (int shift = total_bits - 8; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i0 = tid - lane; i0 < n; i0 += blockDim.x) {  // whole warps: aggregated atomics (keys cluster)
      const int i = i0 + lane;
      int bin = -1;
      if (i < n) {
        const unsigned long long key = (unsigned long long)get(i);
        if ((key & mask) == prefix) bin = (int)((key >> shift) & 255);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (bin >= 0 && lane == __ffs(peers) - 1) atomicAdd(&hist[bin], __popc(peers));
    }
    __syncthreads();
    if (tid < 32) {
      int h[8], loc = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        h[b] = hist[lane * 8 + b];
        loc += h[b];
      }
      int incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int x = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += x;
      }
      const int excl = incl - loc;
      const unsigned ball = __ballot_sync(0xffffffffu, incl >= need);
      const int first = __ffs(ball) - 1;  // lane whose 8 bins hold the k-th
      if (lane == first) {
        int cum = excl, digit = lane * 8 + 7;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          if (cum + h[b] >= need) {
            digit = lane * 8 + b;
            break;
          }
          cum += h[b];
        }
        s_prefix = prefix | ((unsigned long long)digit << shift);
        s_need = need - cum;
      }
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
    mask |= (unsigned long long)255 << shift;
    __syncthreads();
  }
  need_out = need;
  return (K)prefix;
}

constexpr int SMEM_ROW = 16384;  // upper bounds staged in shared memory up to this many centroids
__host__ __device__ inline bool rs_fast_tau(int nlist, int nprobe) {
  // short rows: the radix select over shared memory is already cheaper than the register pass
  // (measured at C3, nlist 1024: the register pass made the probe 0.45 ms against 0.39)
  return nlist >= 4096 && nlist <= RS_REG * RS_THREADS && nprobe <= RS_THREADS;
}

// FAST: the register-held tau path is compiled in (nlist 4096..16384, 64 bounds per thread in registers,
// three CTAs per SM by registers); otherwise the radix path alone, under a 64-register budget so that four
// CTAs (1024 threads) share an SM: the kernel is latency-bound (long-scoreboard and barrier stalls at
// 37% occupancy with 79 registers, C3 ncu)
template <bool FAST>
__global__ void __launch_bounds__(RS_THREADS, FAST ? 3 : 4) probe_rescore_kernel(float* __restrict__ bnd, int64_t q0, int nlist,
                                                                   int nprobe, int order_by_id,
                                                                   const double* __restrict__ q_rot,
                                                                   const float* __restrict__ cent, int d,
                                                                   const double* __restrict__ q_sq,
                                                                   const double* __restrict__ c_sq,
                                                                   int64_t* __restrict__ ids_out,
                                                                   double* __restrict__ d2_out,
                                                                   unsigned long long* __restrict__ stats) {
  extern __shared__ float s_up[];  // [nlist] when nlist <= SMEM_ROW
  __shared__ int32_t hist[256];
  __shared__ int32_t s_nc;
  __shared__ int32_t s_cid[MAX_CAND];
  __shared__ double s_cd[MAX_CAND];
  __shared__ int32_t s_rank[MAX_CAND];
  const int64_t qr = blockIdx.x;
  const int64_t q = q0 + qr;
  float* lrow = bnd + qr * 2 * (int64_t)nlist;
  float* urow = lrow + nlist;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const double* qv = q_rot + q * d;
  const double qs = q_sq[q];
  int64_t* out_i = ids_out + q * nprobe;
  double* out_d = d2_out + q * nprobe;
  // ---- tau: n_probe-th smallest U.  Fast path (nlist <= RS_REG * RS_THREADS, n_probe <= RS_THREADS):
  // the row is held in registers; T0 = the n_probe-th smallest of the per-thread minima bounds
  // tau from above (n_probe distinct elements are <= T0), the few U <= T0 are gathered and
  // tau is their n_probe-th smallest by rank counting.  Otherwise, or when the gathered set
  // is too large (heavy ties), an MSB-first radix select over the whole row.
  __shared__ float s_sel[MAX_CAND];
  __shared__ int32_t s_ns;
  __shared__ float s_tau;
  __shared__ int s_have;
  if (tid == 0) {
    s_ns = 0;
    s_have = 0;
  }
  __syncthreads();
  const bool fast_tau = FAST && rs_fast_tau(nlist, nprobe);
  if (fast_tau) {
    float u[RS_REG];
    float m = __int_as_float(0x7f800000);  // +inf
#pragma unroll
    for (int j = 0; j < RS_REG; ++j) {
      const int i = tid + j * RS_THREADS;
      u[j] = i < nlist ? urow[i] : __int_as_float(0x7f800000);
      m = fminf(m, u[j]);
    }
    s_sel[tid] = m;  // RS_THREADS <= MAX_CAND
    __syncthreads();
    {
      int lt = 0, le = 0;
      for (int f = 0; f < RS_THREADS; ++f) {
        const float x = s_sel[f];
        lt += x < m;
        le += x <= m;
      }
      __syncthreads();
      if (lt < nprobe && nprobe <= le) s_tau = m;  // every writer holds the same value
      __syncthreads();
    }
    const float t0 = s_tau;
#pragma unroll
    for (int j = 0; j < RS_REG; ++j) {
      if (u[j] <= t0) {
        const int p = atomicAdd(&s_ns, 1);
        if (p < MAX_CAND) s_sel[p] = u[j];
      }
    }
    __syncthreads();
    const int ns = s_ns;
    if (ns <= MAX_CAND) {
      for (int e = tid; e < ns; e += RS_THREADS) {
        const float x = s_sel[e];
        int lt = 0, le = 0;
        for (int f = 0; f < ns; ++f) {
          const float y = s_sel[f];
          lt += y < x;
          le += y <= x;
        }
        if (lt < nprobe && nprobe <= le) {
          s_tau = x;
          s_have = 1;
        }
      }
    }
    __syncthreads();
  }
  float tau;
  if (s_have) {
    tau = s_tau;
  } else {
    const bool staged = nlist <= SMEM_ROW && !fast_tau;  // the fast path launches without the staging buffer
    if (staged) {
      for (int i = tid; i < nlist; i += RS_THREADS) s_up[i] = urow[i];
      __syncthreads();
    }
    const float* up = staged ? s_up : urow;
    int unused;
    const uint32_t tau_bits =
        radix_kth<uint32_t>(nlist, nprobe, 32, hist, [&](int i) { return __float_as_uint(up[i]); }, unused);
    tau = __uint_as_float(tau_bits);
  }
  // ---- candidates: L <= tau (a superset of the exact top n_probe)
  if (tid == 0) s_nc = 0;
  __syncthreads();
  for (int i = tid; i < nlist; i += RS_THREADS) {
    if (lrow[i] <= tau) {
      const int p = atomicAdd(&s_nc, 1);
      if (p < MAX_CAND) s_cid[p] = i;
    }
  }
  __syncthreads();
  const int nc = s_nc;
  if (stats && tid == 0) {
    atomicAdd(stats, (unsigned long long)nc);
    if (nc > MAX_CAND) atomicAdd(stats + 1, 1ull);
  }
  if (nc > MAX_CAND) {
    // ---- fallback: every distance in float64, stored over the row's bounds (8 bytes per centroid)
    double* exact = reinterpret_cast<double*>(lrow);
    __syncthreads();
    for (int c = wid; c < nlist; c += RS_THREADS / 32) {
      const double v = exact_dist(qv, cent + (int64_t)c * d, d, qs, c_sq[c]);
      if (lane == 0) exact[c] = v;
    }
    __syncthreads();
    int need = 0;
    const unsigned long long kth = radix_kth<unsigned long long>(
        nlist, nprobe, 64, hist, [&](int i) { return (unsigned long long)__double_as_longlong(exact[i]); }, need);
    if (tid == 0) {  // every key < kth, then the `need` lowest ids equal to kth (ascending id)
      int n = 0, eq = 0;
      for (int c = 0; c < nlist; ++c) {
        const unsigned long long key = (unsigned long long)__double_as_longlong(exact[c]);
        if (key < kth || (key == kth && eq++ < need)) {
          out_i[n] = c;
          out_d[n] = exact[c];
          ++n;
        }
      }
      if (!order_by_id) {  // insertion sort by (distance, id)
        for (int i = 1; i < n; ++i) {
          const double dv = out_d[i];
          const int64_t iv = out_i[i];
          int j = i - 1;
          while (j >= 0 && key_less(dv, iv, out_d[j], out_i[j])) {
            out_d[j + 1] = out_d[j];
            out_i[j + 1] = out_i[j];
            --j;
          }
          out_d[j + 1] = dv;
          out_i[j + 1] = iv;
        }
      }
    }
    return;
  }
  // ---- float64 distances of the candidates (search.py:240-242 arithmetic)
  for (int ci = wid; ci < nc; ci += RS_THREADS / 32) {
    const int c = s_cid[ci];
    const double v = exact_dist(qv, cent + (int64_t)c * d, d, qs, c_sq[c]);
    if (lane == 0) s_cd[ci] = v;
  }
  __syncthreads();
  // ---- ranks by (distance, id); the n_probe smallest are kept
  for (int ci = tid; ci < nc; ci += RS_THREADS) {
    const double dc = s_cd[ci];
    const int64_t ic = s_cid[ci];
    int rank = 0;
    for (int f = 0; f < nc; ++f) rank += key_less(s_cd[f], (int64_t)s_cid[f], dc, ic) ? 1 : 0;
    s_rank[ci] = rank;
  }
  __syncthreads();
  for (int ci = tid; ci < nc; ci += RS_THREADS) {
    const int r = s_rank[ci];
    if (r >= nprobe) continue;
    int pos = r;
    if (order_by_id) {  // ascending id: selected candidates with a smaller id
      pos = 0;
      for (int f = 0; f < nc; ++f) pos += (s_rank[f] < nprobe && s_cid[f] < s_cid[ci]) ? 1 : 0;
    }
    out_i[pos] = s_cid[ci];
    out_d[pos] = s_cd[ci];
  }
}

}  // namespace probe

// Host: the tensor-core probe for rows [0, nq) (stream-ordered, no host sync).
int probe_tc(const double* q_rot, int64_t nq, int32_t dims, const float* centroids, const double* centroid_sqnorms,
             int32_t n_clusters, int32_t n_probe, int32_t order_by_id, int64_t* ids, double* d2, const double* q_sq,
             cudaStream_t s) {
  using namespace probe;
  const int kp = (dims + 15) / 16 * 16;
  int8_t *qd = nullptr, *cd = nullptr;
  int32_t *qe = nullptr, *ce = nullptr;
  double *ql1 = nullptr, *cl1 = nullptr;
  float* bounds = nullptr;
  // (bound rows in 256 MB chunks; 64 / 100 MB chunks measured slower at C4: probe 2.08 / 1.99 vs 1.78 ms)
  const int64_t rows = std::max<int64_t>(128, std::min<int64_t>(nq, ((int64_t)256 << 20) / ((int64_t)n_clusters * 8)));
  Workspace ws(s);
  if (!ws.alloc(qd, (size_t)4 * nq * kp) || !ws.alloc(cd, (size_t)4 * n_clusters * kp) || !ws.alloc(qe, nq) ||
      !ws.alloc(ce, n_clusters) || !ws.alloc(ql1, nq) || !ws.alloc(cl1, n_clusters) ||
      !ws.alloc(bounds, (size_t)rows * n_clusters * 2))
    return fail(IVRQ_ENOMEM, "ivrq_select_clusters: workspace allocation failed");
  constexpr int ndig = 2;  // 14-bit fixed point per side
  const int QT = QT_<ndig>, CT = CT_<ndig>;
  auto dq = digits_kernel<double, ndig>;
  auto dc = digits_kernel<float, ndig>;
  dq<<<(unsigned)ceil_div(nq, 8), 256, 0, s>>>(q_rot, nq, dims, kp, 0, qd, qe, ql1);
  dc<<<(unsigned)ceil_div(n_clusters, 8), 256, 0, s>>>(centroids, n_clusters, dims, kp, 0, cd, ce, cl1);
  IVRQ_TRY(check_launch("ivrq_select_clusters(digits)"));
  TpArgs ta{};
  if (!tc::make_tmap_u8_sw128(&ta.map_q, qd, (uint64_t)kp, (uint64_t)ndig * nq, (uint64_t)kp, KC, 128) ||
      !tc::make_tmap_u8_sw128(&ta.map_c, cd, (uint64_t)kp, (uint64_t)ndig * n_clusters, (uint64_t)kp, KC, NCOL))
    return fail(IVRQ_ECUDA, "ivrq_select_clusters: TMA tensor map encoding failed");
  ta.nq = nq;
  ta.nlist = n_clusters;
  ta.kp = kp;
  ta.d = dims;
  ta.q_sq = q_sq;
  ta.c_sq = centroid_sqnorms;
  ta.q_e = qe;
  ta.c_e = ce;
  ta.q_l1 = ql1;
  ta.c_l1 = cl1;
  ta.bnd = bounds;
  const size_t sm = tp_smem_bytes();
  auto tk = tc_probe_kernel<ndig>;
  if (cudaFuncSetAttribute(tk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess ||
      cudaFuncSetAttribute(probe_rescore_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ROW * 4) !=
          cudaSuccess ||
      cudaFuncSetAttribute(probe_rescore_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_ROW * 4) !=
          cudaSuccess)
    return fail(IVRQ_EUNSUP, "ivrq_select_clusters: tensor-core probe shared memory");
  cudaFuncSetAttribute(probe_rescore_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  for (int64_t r0 = 0; r0 < nq; r0 += rows) {
    const int64_t rn = std::min(rows, nq - r0);
    ta.q0 = r0;
    ta.nrows = rn;
    const int64_t tiles = ceil_div(rn, QT) * ceil_div(n_clusters, CT);
    const int grid = (int)std::min<int64_t>(tiles, sm_count_of_current_device());
    tk<<<grid, THREADS, sm, s>>>(ta);
    IVRQ_TRY(check_launch("ivrq_select_clusters(tc bounds)"));
    const size_t rsm =
        n_clusters <= SMEM_ROW && !rs_fast_tau(n_clusters, n_probe) ? (size_t)n_clusters * sizeof(float) : 0;
    auto rk = rs_fast_tau(n_clusters, n_probe) ? probe_rescore_kernel<true> : probe_rescore_kernel<false>;
    rk<<<(unsigned)rn, RS_THREADS, rsm, s>>>(bounds, r0, n_clusters, n_probe, order_by_id, q_rot,
                                                               centroids, dims, q_sq, centroid_sqnorms, ids, d2, nullptr);
    IVRQ_TRY(check_launch("ivrq_select_clusters(rescore)"));
  }
  return IVRQ_OK;
}

}  // namespace ivrq
