// Per-call sub-operators of the reference API (search.py:84-375, codec.py:118-151,
// 262-303, 383-401) on the GPU.  These are the building blocks the reference
// exports next to build_index / search_batch; the batched hot path does not use
// them (it fuses the same arithmetic into the list scan), but callers of the
// reference's finer-grained API get the same semantics here:
//
//   ivrq_ip_bitwise            ip_bitwise           search.py:163-183  exact integer AND+POPC
//   ivrq_ip_lut                ip_lut               search.py:146-160  float32 tables summed in float64
//   ivrq_estimate_stage1       estimate_stage1      search.py:270-287  reference operand order
//   ivrq_refine_stage2         refine_stage2        search.py:290-310  ex @ q_rot as a double-double dot
//   ivrq_cluster_local_search  cluster_local_search search.py:326-375  one CTA: stage 1, prune, refine, lexsort
//   ivrq_compute_factors       compute_factors_batch codec.py:322-380  einsum-order reductions
//   ivrq_normalize_residuals   normalize_residual(s) codec.py:118-151
//   ivrq_quantize_oracle       quantize_oracle       codec.py:262-303  exhaustive critical-factor search
//
// Values that the reference takes from a BLAS dot (refine_stage2's `ex @ q_rot`,
// _refine_from_codes' `codes @ q_rot`, cluster_local_search's `diff @ diff`,
// np.linalg.norm) are host dependent there; here they are double-double sums
// rounded once, i.e. the correctly rounded value in all but pathological cases.
#include <cstdint>

#include "ivrq_common.cuh"

namespace ivrq {
namespace ops {

constexpr unsigned FULL = 0xffffffffu;
__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }
constexpr int64_t NO_ID = 0x7fffffffffffffffLL;

// ------------------------------------------------------------ double-double dot
struct DDAcc {
  double s = 0.0, c = 0.0;
  __device__ __forceinline__ void add_prod(double a, double b) {
    const double p = __dmul_rn(a, b);
    const double pe = __fma_rn(a, b, -p);  // exact product error
    const double t = __dadd_rn(s, p);
    const double bp = __dsub_rn(t, s);
    const double se = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(p, bp));  // two_sum error
    s = t;
    c = __dadd_rn(c, __dadd_rn(se, pe));
  }
  __device__ __forceinline__ void merge(const DDAcc& o) {
    const double t = __dadd_rn(s, o.s);
    const double bp = __dsub_rn(t, s);
    const double se = __dadd_rn(__dsub_rn(s, __dsub_rn(t, bp)), __dsub_rn(o.s, bp));
    s = t;
    c = __dadd_rn(c, __dadd_rn(se, o.c));
  }
  __device__ __forceinline__ double value() const { return __dadd_rn(s, c); }
};

__device__ __forceinline__ DDAcc warp_dd_reduce(DDAcc a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    DDAcc b;
    b.s = __shfl_xor_sync(FULL, a.s, o);
    b.c = __shfl_xor_sync(FULL, a.c, o);
    a.merge(b);
  }
  return a;
}

// unsigned code u of dim j of row r from the rcodes layout (include/ivrq_b200.h)
__device__ __forceinline__ int rcode_at(const uint8_t* rc, int64_t rb, int64_t r, int j, bool nib) {
  const uint8_t* row = rc + r * rb;
  return nib ? (row[j >> 1] >> (4 * (j & 1))) & 15 : row[j];
}

// ------------------------------------------------------------ ip_bitwise
// words (g, n) interleaved, planes (qb, g): sum_j w_j sum_gi popc(word & plane_j),
// w_j = 2^j except the sign plane -2^(qb-1)  (search.py:176-183).
__global__ void ip_bitwise_kernel(const uint32_t* __restrict__ words, int g, int64_t n,
                                  const uint32_t* __restrict__ planes, int qb, int64_t* __restrict__ out) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  long long acc = 0;
  for (int gi = 0; gi < g; ++gi) {
    const uint32_t w = words[(int64_t)gi * n + v];
    for (int j = 0; j < qb; ++j) {
      const long long c = __popc(w & planes[j * g + gi]);
      acc += (j == qb - 1) ? -(c << j) : (c << j);
    }
  }
  out[v] = acc;
}

// ------------------------------------------------------------ ip_lut
// out[v] = sum_b luts[b][nib[v][b]]: float32 entries accumulated in float64 in
// block order (the reference's sum is exact for these operands, so any order
// that does not round gives its value).
__global__ void ip_lut_kernel(const uint8_t* __restrict__ nib, int64_t n, int blocks, const float* __restrict__ luts,
                              double* __restrict__ out) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  double acc = 0.0;
  for (int b = 0; b < blocks; ++b) acc = dadd(acc, (double)luts[b * 16 + (nib[v * blocks + b] & 15)]);
  out[v] = acc;
}

// ------------------------------------------------------------ estimate_stage1
struct Stage1 {
  double est2, lb2;
};

// search.py:281-287 in the reference's operand order
__device__ __forceinline__ Stage1 stage1(double ip, double add, double scale, double err, double half_code,
                                         double ip_margin, double d_qc2) {
  const double ip_signed = dsub(ip, half_code);
  const double est2 = dmax(dsub(dadd(add, d_qc2), dmul(scale, ip_signed)), 0.0);
  double margin = dmul(err, dsqrt(d_qc2));
  if (ip_margin != 0.0) {
    const double sm = dmul(scale, ip_margin);
    margin = dsqrt(dadd(dmul(margin, margin), dmul(sm, sm)));
  }
  return {est2, dmax(dsub(est2, margin), 0.0)};
}

__global__ void estimate_stage1_kernel(const double* __restrict__ ip, const double* __restrict__ sf, int64_t n,
                                       const double* __restrict__ d_qc2, double half_code, double ip_margin,
                                       double* __restrict__ est2, double* __restrict__ lb2) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n) return;
  const Stage1 r = stage1(ip[v], sf[3 * v], sf[3 * v + 1], sf[3 * v + 2], half_code, ip_margin, d_qc2[v]);
  est2[v] = r.est2;
  lb2[v] = r.lb2;
}

// ------------------------------------------------------------ refine_stage2
// One warp per row: ip_u = 2^(bits-1) * ip_binary + <ex, q_rot>;
// est2 = max(add + d_qc2 - scale * (ip_u - k_b * sum_q), 0)   (search.py:304-310)
__global__ void refine_stage2_kernel(const double* __restrict__ ex, int64_t n, int d, const double* __restrict__ ip,
                                     const double* __restrict__ lf, const double* __restrict__ q_rot, double sum_q,
                                     const double* __restrict__ d_qc2, int bits, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  DDAcc acc;
  for (int j = lane; j < d; j += 32) acc.add_prod(ex[r * d + j], q_rot[j]);
  acc = warp_dd_reduce(acc);
  if (lane == 0) {
    const double k_b = ((double)((1 << bits) - 1)) / 2.0;
    const double ip_u = dadd(dmul((double)(1 << (bits - 1)), ip[r]), acc.value());
    out[r] = dmax(dsub(dadd(lf[2 * r], d_qc2[r]), dmul(lf[2 * r + 1], dsub(ip_u, dmul(k_b, sum_q)))), 0.0);
  }
}

// ------------------------------------------------------------ cluster_local_search
struct ClsArgs {
  ivrq_index_view ix;
  int64_t cluster;
  const double* q_rot;    // [dims]
  const uint32_t* planes; // [qb * g] (bitwise)
  const float* luts;      // [8g * 16] (lut)
  int mode, qb, refine, k;
  double sum_q, delta, code_sum, ip_margin, threshold, d_qc2;
  int have_d_qc2;
  int64_t cap;  // power of two >= list size
  double* keys;
  int64_t* ids;
  int32_t* rows;
  double* est;
  int64_t* out_ids;
  double* out_dists;
  int32_t* out_count;
};

constexpr int CLS_THREADS = 1024;

__global__ void __launch_bounds__(CLS_THREADS) cluster_local_search_kernel(const ClsArgs a) {
  __shared__ int s_cnt;
  __shared__ double s_dqc2;
  __shared__ double s_red[2][CLS_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int d = a.ix.dims, g = words_per_vector(d);
  const int64_t lo = a.ix.offsets[a.cluster], n_c = a.ix.offsets[a.cluster + 1] - lo;
  if (tid == 0) s_cnt = 0;
  // d_qc2 = (q_rot - c) @ (q_rot - c) when not given (search.py:350-352)
  if (!a.have_d_qc2) {
    DDAcc acc;
    for (int j = tid; j < d; j += CLS_THREADS) {
      const double df = dsub(a.q_rot[j], (double)a.ix.centroids[a.cluster * d + j]);
      acc.add_prod(df, df);
    }
    acc = warp_dd_reduce(acc);
    if (lane == 0) {
      s_red[0][wid] = acc.s;
      s_red[1][wid] = acc.c;
    }
    __syncthreads();
    if (tid == 0) {
      DDAcc t;
      for (int w = 0; w < CLS_THREADS / 32; ++w) t.merge(DDAcc{s_red[0][w], s_red[1][w]});
      s_dqc2 = t.value();
    }
  } else if (tid == 0) {
    s_dqc2 = a.d_qc2;
  }
  __syncthreads();
  const double d_qc2 = s_dqc2;
  const double half_code = dmul(0.5, a.code_sum);
  // stage 1 + prune (search.py:354-359)
  for (int64_t v = tid; v < n_c; v += CLS_THREADS) {
    double ip;
    if (a.mode == IVRQ_IP_BITWISE) {
      long long acc = 0;
      for (int gi = 0; gi < g; ++gi) {
        const uint32_t w = a.ix.packed_msb[g * lo + (int64_t)gi * n_c + v];
        for (int j = 0; j < a.qb; ++j) {
          const long long c = __popc(w & a.planes[j * g + gi]);
          acc += (j == a.qb - 1) ? -(c << j) : (c << j);
        }
      }
      ip = dmul(a.delta, (double)acc);
    } else {
      double acc = 0.0;
      for (int gi = 0; gi < g; ++gi) {
        const uint32_t w = a.ix.packed_msb[g * lo + (int64_t)gi * n_c + v];
        for (int s = 0; s < 8; ++s) acc = dadd(acc, (double)a.luts[(gi * 8 + s) * 16 + ((w >> (4 * s)) & 15u)]);
      }
      ip = acc;
    }
    const int64_t row = lo + v;
    const Stage1 st = stage1(ip, (double)a.ix.short_add[row], (double)a.ix.short_scale[row],
                             (double)a.ix.short_err[row], half_code, a.ip_margin, d_qc2);
    if (st.lb2 <= a.threshold) {
      const int p = atomicAdd(&s_cnt, 1);
      a.rows[p] = (int32_t)v;
      a.est[p] = st.est2;
    }
  }
  __syncthreads();
  const int m = s_cnt;
  const bool refine = a.refine && a.ix.bits >= 2;
  const bool nib = rcode_nibbles(a.ix.bits);
  const double k_b = ((double)((1 << a.ix.bits) - 1)) / 2.0;
  // refine survivors, one warp each (_refine_from_codes, search.py:313-323)
  for (int p = wid; p < m; p += CLS_THREADS / 32) {
    const int64_t row = lo + a.rows[p];
    double dist = a.est[p];
    if (refine) {
      DDAcc acc;
      for (int j = lane; j < d; j += 32)
        acc.add_prod((double)rcode_at(a.ix.rcodes, a.ix.rcode_bytes, row, j, nib), a.q_rot[j]);
      acc = warp_dd_reduce(acc);
      const double ip_u = acc.value();
      const float2 lf = reinterpret_cast<const float2*>(a.ix.long_factors)[row];
      dist = dmax(dsub(dadd((double)lf.x, d_qc2), dmul((double)lf.y, dsub(ip_u, dmul(k_b, a.sum_q)))), 0.0);
    }
    if (lane == 0) {
      a.keys[p] = dist;
      a.ids[p] = a.ix.pids[row];
    }
  }
  for (int64_t i = m + tid; i < a.cap; i += CLS_THREADS) {
    a.keys[i] = dinf();
    a.ids[i] = NO_ID;
  }
  __syncthreads();
  // bitonic sort of (dist, pid) over the power-of-two padded buffer (np.lexsort((pids, dists)))
  int64_t n2 = 1;
  while (n2 < m) n2 <<= 1;
  for (int64_t size = 2; size <= n2; size <<= 1) {
    for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int64_t i = tid; i < n2; i += CLS_THREADS) {
        const int64_t j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const double di = a.keys[i], dj = a.keys[j];
          const int64_t ii = a.ids[i], ij = a.ids[j];
          const bool swap = up ? key_less(dj, ij, di, ii) : key_less(di, ii, dj, ij);
          if (swap) {
            a.keys[i] = dj;
            a.keys[j] = di;
            a.ids[i] = ij;
            a.ids[j] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  const int kk = m < a.k ? m : a.k;
  for (int i = tid; i < kk; i += CLS_THREADS) {
    a.out_ids[i] = a.ids[i];
    a.out_dists[i] = a.keys[i];
  }
  if (tid == 0) *a.out_count = kk;
}

// ------------------------------------------------------------ compute_factors_batch
// One warp per row; lanes 2e / 2e+1 hold the two accumulators of einsum e
// (codec.py:355-379): <xb,o>, <x,x>, <x,o>, <xb,c'>, <x,c'>.
__global__ void compute_factors_kernel(const uint8_t* __restrict__ u, const double* __restrict__ o,
                                       const double* __restrict__ dist, const double* __restrict__ c, int64_t n, int d,
                                       int bits, double eps, double* __restrict__ short_f, double* __restrict__ long_f,
                                       uint8_t* __restrict__ low_quality) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  const int eb = bits - 1;
  const double k_b = ((double)((1 << bits) - 1)) / 2.0;
  const int e = lane >> 1, l = lane & 1;
  const uint8_t* ur = u + r * d;
  const double* orow = o + r * d;
  const double* crow = c + r * d;
  auto term = [&](int dim) -> double {
    const double uv = (double)ur[dim];
    const double xb = dsub((double)(ur[dim] >> eb), 0.5);
    const double x = dsub(uv, k_b);
    switch (e) {
      case 0: return dmul(xb, orow[dim]);
      case 1: return dmul(x, x);
      case 2: return dmul(x, orow[dim]);
      case 3: return dmul(xb, crow[dim]);
      default: return dmul(x, crow[dim]);
    }
  };
  double acc = 0.0;
  if (e < 5) {
    int i = 0;
    for (; i + 8 <= d; i += 8)
#pragma unroll
      for (int blk = 3; blk >= 0; --blk) acc = dadd(term(i + 2 * blk + l), acc);
    for (; i < d; i += 2) acc = dadd((i + l) < d ? term(i + l) : 0.0, acc);
  }
  double res[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    const double a0 = __shfl_sync(FULL, acc, 2 * q);
    const double a1 = __shfl_sync(FULL, acc, 2 * q + 1);
    res[q] = dadd(0.0, dadd(a0, a1));
  }
  if (lane != 0) return;
  const double dd = dist[r];
  const double norm_b = dmul(0.5, dsqrt((double)d));
  double cos_b = ddiv(res[0], norm_b);
  const double norm_x = dsqrt(res[1]);
  double cos_x = ddiv(res[2], norm_x);
  const bool live = dd > 0.0;
  low_quality[r] = (live && cos_b <= 0.0) ? 1 : 0;
  double s_add = 0.0, s_scale = 0.0, s_err = 0.0, l_add = 0.0, l_scale = 0.0;
  if (live) {
    cos_b = dmax(cos_b, 1e-6);
    cos_x = dmax(cos_x, 1e-6);
    const double two_d = dmul(2.0, dd);
    const double dsq = dmul(dd, dd);
    s_scale = ddiv(two_d, dmul(norm_b, cos_b));
    s_add = dadd(dsq, dmul(s_scale, res[3]));
    const double cb2 = dmul(cos_b, cos_b);
    const double var = ddiv(dmax(dsub(1.0, cb2), 0.0), dmul(cb2, (double)(d - 1 > 1 ? d - 1 : 1)));
    s_err = dmul(dmul(two_d, eps), dsqrt(var));
    l_scale = ddiv(two_d, dmul(norm_x, cos_x));
    l_add = dadd(dsq, dmul(l_scale, res[4]));
  }
  short_f[3 * r] = s_add;
  short_f[3 * r + 1] = s_scale;
  short_f[3 * r + 2] = s_err;
  long_f[2 * r] = l_add;
  long_f[2 * r + 1] = l_scale;
}

// ------------------------------------------------------------ normalize_residuals
// diff = x - c; d = sqrt(einsum(diff, diff)) (einsum order, codec.py:147) or the
// double-double norm (np.linalg.norm, codec.py:129); o = diff / d, zero rows -> 0.
__global__ void normalize_residuals_kernel(const double* __restrict__ x, const double* __restrict__ c, int64_t n,
                                           int d, int dd_norm, double* __restrict__ o, double* __restrict__ dist) {
  const int lane = threadIdx.x & 31;
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= n) return;
  const double* xr = x + r * d;
  const double* cr = c + r * d;
  double nrm;
  if (dd_norm) {
    DDAcc acc;
    for (int j = lane; j < d; j += 32) {
      const double df = dsub(xr[j], cr[j]);
      acc.add_prod(df, df);
    }
    acc = warp_dd_reduce(acc);
    nrm = dsqrt(acc.value());
  } else {
    double acc = 0.0;
    if (lane < 2) {
      int i = 0;
      for (; i + 8 <= d; i += 8)
#pragma unroll
        for (int blk = 3; blk >= 0; --blk) {
          const double df = dsub(xr[i + 2 * blk + lane], cr[i + 2 * blk + lane]);
          acc = dadd(dmul(df, df), acc);
        }
      for (; i < d; i += 2) {
        double p = 0.0;
        if (i + lane < d) {
          const double df = dsub(xr[i + lane], cr[i + lane]);
          p = dmul(df, df);
        }
        acc = dadd(p, acc);
      }
    }
    const double a1 = __shfl_sync(FULL, acc, 1);
    nrm = dsqrt(dadd(0.0, dadd(__shfl_sync(FULL, acc, 0), a1)));
  }
  for (int j = lane; j < d; j += 32) o[r * d + j] = nrm == 0.0 ? 0.0 : ddiv(dsub(xr[j], cr[j]), nrm);
  if (lane == 0) dist[r] = nrm;
}

// ------------------------------------------------------------ quantize_oracle
// Exhaustive critical-factor quantizer for one vector (codec.py:262-303), one CTA:
// crit = unique(level / |o_i|) (bitonic sort + compaction), evaluation points
// crit[0]/2, midpoints, crit[-1]+1; per point the rounded code, its cosine with
// einsum-order num / sqrt(den); the first maximum, exact ties to the
// lexicographically smallest code.
constexpr int QO_THREADS = 1024;

struct QoArgs {
  const double* o;
  int d, bits;
  int64_t cap;  // power of two >= number of critical values
  double* crit;
  double* cosv;
  uint8_t* out;
};

__device__ __forceinline__ double qo_code(double t, double ov, int bits, double k_b) {
  // _round_codes: floor(t*o + (k_b + 0.5)), clipped to [0, 2^bits - 1]
  double x = dadd(dmul(t, ov), dadd(k_b, 0.5));
  x = floor(x);
  const double top = (double)((1 << bits) - 1);
  return x < 0.0 ? 0.0 : (x > top ? top : x);
}

__global__ void __launch_bounds__(QO_THREADS) quantize_oracle_kernel(const QoArgs a) {
  __shared__ int s_m;
  __shared__ int s_u;
  __shared__ double s_best;
  __shared__ int s_bidx;
  const int tid = threadIdx.x;
  const int d = a.d, bits = a.bits;
  const int L = (1 << (bits - 1)) - 1;  // levels 1 .. 2^(bits-1)-1
  const double k_b = ((double)((1 << bits) - 1)) / 2.0;
  const int u_zero = (1 << (bits - 1)) - 1;
  if (tid == 0) s_m = 0;
  __syncthreads();
  // critical values level / |o_i| of the nonzero coordinates
  for (int i = tid; i < d; i += QO_THREADS) {
    const double ov = a.o[i];
    if (ov != 0.0) {
      const double az = fabs(ov);
      const int base = atomicAdd(&s_m, L);
      for (int l = 1; l <= L; ++l) a.crit[base + l - 1] = ddiv((double)l, az);
    }
  }
  __syncthreads();
  const int m = s_m;
  if (m == 0) {
    // no critical value: every coordinate is zero (the all-midpoint code, codec.py:283-284)
    // or bits == 1 (the sign pattern, codec.py:285-286; all-zero again gives the midpoint 1)
    __shared__ int s_nz;
    if (tid == 0) s_nz = 0;
    __syncthreads();
    for (int j = tid; j < d; j += QO_THREADS)
      if (a.o[j] != 0.0) atomicOr(&s_nz, 1);
    __syncthreads();
    for (int j = tid; j < d; j += QO_THREADS)
      a.out[j] = (uint8_t)(s_nz ? (a.o[j] > 0.0 ? 1 : 0) : (1 << (bits - 1)));
    return;
  }
  for (int64_t i = m + tid; i < a.cap; i += QO_THREADS) a.crit[i] = dinf();
  __syncthreads();
  int64_t n2 = 1;
  while (n2 < m) n2 <<= 1;
  for (int64_t size = 2; size <= n2; size <<= 1)
    for (int64_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (int64_t i = tid; i < n2; i += QO_THREADS) {
        const int64_t j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const double x = a.crit[i], y = a.crit[j];
          if (up ? (y < x) : (x < y)) {
            a.crit[i] = y;
            a.crit[j] = x;
          }
        }
      }
      __syncthreads();
    }
  if (tid == 0) {  // np.unique: drop exact duplicates (sorted)
    int u = 0;
    for (int i = 0; i < m; ++i)
      if (u == 0 || a.crit[i] != a.crit[u - 1]) a.crit[u++] = a.crit[i];
    s_u = u;
  }
  __syncthreads();
  const int U = s_u;
  // evaluation points: [crit0/2, mids..., crit[-1]+1], or [1.0] when crit is empty
  const int E = U > 0 ? U + 1 : 1;
  for (int e = tid; e < E; e += QO_THREADS) {
    double t;
    if (U == 0) t = 1.0;
    else if (e == 0) t = ddiv(a.crit[0], 2.0);
    else if (e == U) t = dadd(a.crit[U - 1], 1.0);
    else t = ddiv(dadd(a.crit[e - 1], a.crit[e]), 2.0);
    EinsumAcc num, den;
    auto sv = [&](int j) -> double {
      const double ov = a.o[j];
      const double code = ov == 0.0 ? (double)u_zero : qo_code(t, ov, bits, k_b);
      return dsub(code, k_b);
    };
    int i = 0;
    for (; i + 8 <= d; i += 8) {
      double pn[8], pd[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const double s = sv(i + k);
        pn[k] = dmul(s, a.o[i + k]);
        pd[k] = dmul(s, s);
      }
      num.block8(pn);
      den.block8(pd);
    }
    for (; i < d; i += 2) {
      const bool has1 = (i + 1) < d;
      const double s0 = sv(i), s1 = has1 ? sv(i + 1) : 0.0;
      num.pair(dmul(s0, a.o[i]), has1 ? dmul(s1, a.o[i + 1]) : 0.0, has1);
      den.pair(dmul(s0, s0), has1 ? dmul(s1, s1) : 0.0, has1);
    }
    a.cosv[e] = ddiv(num.result(), dsqrt(den.result()));
  }
  __syncthreads();
  if (tid == 0) {  // argmax (first), then the lexicographically smallest code among exact ties
    int best = 0;
    for (int e = 1; e < E; ++e)
      if (a.cosv[e] > a.cosv[best]) best = e;
    s_best = a.cosv[best];
    s_bidx = best;
  }
  __syncthreads();
  if (tid == 0) {
    auto tval = [&](int e) -> double {
      if (U == 0) return 1.0;
      if (e == 0) return ddiv(a.crit[0], 2.0);
      if (e == U) return dadd(a.crit[U - 1], 1.0);
      return ddiv(dadd(a.crit[e - 1], a.crit[e]), 2.0);
    };
    int best = s_bidx;
    for (int e = best + 1; e < E; ++e) {
      if (!(a.cosv[e] == s_best)) continue;
      const double te = tval(e), tb = tval(best);
      for (int j = 0; j < d; ++j) {
        const double ov = a.o[j];
        const double ce = ov == 0.0 ? (double)u_zero : qo_code(te, ov, bits, k_b);
        const double cb = ov == 0.0 ? (double)u_zero : qo_code(tb, ov, bits, k_b);
        if (ce != cb) {
          if (ce < cb) best = e;
          break;
        }
      }
    }
    s_bidx = best;
  }
  __syncthreads();
  const double tb = [&]() {
    const int e = s_bidx;
    if (U == 0) return 1.0;
    if (e == 0) return ddiv(a.crit[0], 2.0);
    if (e == U) return dadd(a.crit[U - 1], 1.0);
    return ddiv(dadd(a.crit[e - 1], a.crit[e]), 2.0);
  }();
  for (int j = tid; j < d; j += QO_THREADS) {
    const double ov = a.o[j];
    a.out[j] = (uint8_t)(ov == 0.0 ? u_zero : (int)qo_code(tb, ov, bits, k_b));
  }
}

}  // namespace ops
}  // namespace ivrq

using namespace ivrq;

extern "C" int ivrq_ip_bitwise(const uint32_t* words, int32_t groups, int64_t n, const uint32_t* planes,
                               int32_t query_bits, int64_t* out, void* stream) {
  if (n < 0 || groups < 0 || query_bits < 1 || query_bits > 32) return fail(IVRQ_EINVAL, "ivrq_ip_bitwise: bad sizes");
  if (n == 0) return IVRQ_OK;
  if (!words || !planes || !out) return fail(IVRQ_EINVAL, "ivrq_ip_bitwise: null pointer");
  ops::ip_bitwise_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(words, groups, n, planes,
                                                                                    query_bits, out);
  return check_launch("ivrq_ip_bitwise");
}

extern "C" int ivrq_ip_lut(const uint8_t* nibbles, int64_t n, int32_t blocks, const float* luts, double* out,
                           void* stream) {
  if (n < 0 || blocks < 0) return fail(IVRQ_EINVAL, "ivrq_ip_lut: bad sizes");
  if (n == 0) return IVRQ_OK;
  if (!nibbles || !luts || !out) return fail(IVRQ_EINVAL, "ivrq_ip_lut: null pointer");
  ops::ip_lut_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(nibbles, n, blocks, luts, out);
  return check_launch("ivrq_ip_lut");
}

extern "C" int ivrq_estimate_stage1(const double* ip, const double* short_factors, int64_t n, const double* d_qc2,
                                    double code_sum_q, double ip_margin, double* est2, double* lb2, void* stream) {
  if (n < 0) return fail(IVRQ_EINVAL, "ivrq_estimate_stage1: bad size");
  if (n == 0) return IVRQ_OK;
  if (!ip || !short_factors || !d_qc2 || !est2 || !lb2) return fail(IVRQ_EINVAL, "ivrq_estimate_stage1: null pointer");
  ops::estimate_stage1_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, as_stream(stream)>>>(
      ip, short_factors, n, d_qc2, 0.5 * code_sum_q, ip_margin, est2, lb2);
  return check_launch("ivrq_estimate_stage1");
}

extern "C" int ivrq_refine_stage2(const double* ex, int64_t n, int32_t dims, const double* ip_binary,
                                  const double* long_factors, const double* q_rot, double sum_q, const double* d_qc2,
                                  int32_t bits, double* out, void* stream) {
  if (bits < 2 || bits > 8) return fail(IVRQ_EINVAL, "refinement requires bits >= 2 (no ex-code exists for 1-bit indexes)");
  if (n < 0 || dims < 0) return fail(IVRQ_EINVAL, "ivrq_refine_stage2: bad sizes");
  if (n == 0) return IVRQ_OK;
  if (!ex || !ip_binary || !long_factors || !q_rot || !d_qc2 || !out)
    return fail(IVRQ_EINVAL, "ivrq_refine_stage2: null pointer");
  ops::refine_stage2_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, as_stream(stream)>>>(
      ex, n, dims, ip_binary, long_factors, q_rot, sum_q, d_qc2, bits, out);
  return check_launch("ivrq_refine_stage2");
}

extern "C" size_t ivrq_cluster_local_search_workspace(int64_t list_size) {
  int64_t cap = 1;
  while (cap < list_size) cap <<= 1;
  return (size_t)cap * (sizeof(double) + sizeof(int64_t) + sizeof(int32_t) + sizeof(double)) + 64;
}

extern "C" int ivrq_cluster_local_search(const ivrq_index_view* index, int64_t cluster, const double* q_rot,
                                         const uint32_t* planes, const float* luts, const double* qstate,
                                         const ivrq_search_params* params, double threshold, const double* d_qc2,
                                         int64_t* out_ids, double* out_dists, int32_t* out_count, void* workspace,
                                         size_t workspace_bytes, int64_t list_size, void* stream) {
  if (!index || !params || !qstate || !q_rot || !out_ids || !out_dists || !out_count)
    return fail(IVRQ_EINVAL, "ivrq_cluster_local_search: null argument");
  if (cluster < 0 || cluster >= index->n_clusters) return fail(IVRQ_EINVAL, "cluster id out of range");
  if (params->k < 1) return fail(IVRQ_EINVAL, "k must be >= 1");
  if (params->ip_mode == IVRQ_IP_BITWISE ? !planes : !luts)
    return fail(IVRQ_EINVAL, "ivrq_cluster_local_search: the query state lacks planes / tables for this ip_mode");
  if (params->refine && index->bits >= 2 && !index->rcodes) return fail(IVRQ_EINVAL, "refine needs rcodes");
  if (workspace_bytes < ivrq_cluster_local_search_workspace(list_size))
    return fail(IVRQ_ENOMEM, "ivrq_cluster_local_search: workspace too small");
  ops::ClsArgs a{};
  a.ix = *index;
  a.cluster = cluster;
  a.q_rot = q_rot;
  a.planes = planes;
  a.luts = luts;
  a.mode = params->ip_mode;
  a.qb = params->query_bits;
  a.refine = params->refine;
  a.k = params->k;
  a.sum_q = qstate[IVRQ_QS_SUM_Q];
  a.delta = qstate[IVRQ_QS_DELTA];
  a.code_sum = qstate[IVRQ_QS_CODE_SUM];
  a.ip_margin = qstate[IVRQ_QS_IP_MARGIN];
  a.threshold = threshold;
  a.have_d_qc2 = d_qc2 != nullptr;
  a.d_qc2 = d_qc2 ? *d_qc2 : 0.0;
  int64_t cap = 1;
  while (cap < list_size) cap <<= 1;
  a.cap = cap;
  unsigned char* p = static_cast<unsigned char*>(workspace);
  a.keys = reinterpret_cast<double*>(p);
  a.est = reinterpret_cast<double*>(p + cap * 8);
  a.ids = reinterpret_cast<int64_t*>(p + cap * 16);
  a.rows = reinterpret_cast<int32_t*>(p + cap * 24);
  a.out_ids = out_ids;
  a.out_dists = out_dists;
  a.out_count = out_count;
  ops::cluster_local_search_kernel<<<1, ops::CLS_THREADS, 0, as_stream(stream)>>>(a);
  return check_launch("ivrq_cluster_local_search");
}

extern "C" int ivrq_compute_factors(const uint8_t* u, const double* o, const double* dist, const double* c_rot,
                                    int64_t n, int32_t dims, int32_t bits, double eps_bound, double* short_factors,
                                    double* long_factors, uint8_t* low_quality, void* stream) {
  if (bits < 1 || bits > 8 || n < 0 || dims < 1) return fail(IVRQ_EINVAL, "ivrq_compute_factors: bad arguments");
  if (n == 0) return IVRQ_OK;
  if (!u || !o || !dist || !c_rot || !short_factors || !long_factors || !low_quality)
    return fail(IVRQ_EINVAL, "ivrq_compute_factors: null pointer");
  ops::compute_factors_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, as_stream(stream)>>>(
      u, o, dist, c_rot, n, dims, bits, eps_bound, short_factors, long_factors, low_quality);
  return check_launch("ivrq_compute_factors");
}

extern "C" int ivrq_normalize_residuals(const double* x, const double* c, int64_t n, int32_t dims, int32_t dd_norm,
                                        double* o, double* dist, void* stream) {
  if (n < 0 || dims < 0) return fail(IVRQ_EINVAL, "ivrq_normalize_residuals: bad sizes");
  if (n == 0) return IVRQ_OK;
  if (!x || !c || !o || !dist) return fail(IVRQ_EINVAL, "ivrq_normalize_residuals: null pointer");
  ops::normalize_residuals_kernel<<<(unsigned)ceil_div(n * 32, 256), 256, 0, as_stream(stream)>>>(x, c, n, dims,
                                                                                                dd_norm, o, dist);
  return check_launch("ivrq_normalize_residuals");
}

extern "C" size_t ivrq_quantize_oracle_workspace(int32_t dims, int32_t bits) {
  const int64_t m = (int64_t)dims * ((1 << (bits - 1)) - 1);
  int64_t cap = 1;
  while (cap < m) cap <<= 1;
  return (size_t)cap * 8 + (size_t)(m + 2) * 8 + 64;
}

extern "C" int ivrq_quantize_oracle(const double* o, int32_t dims, int32_t bits, uint8_t* out, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  if (bits < 1 || bits > 8 || dims < 1) return fail(IVRQ_EINVAL, "ivrq_quantize_oracle: bits must be in [1, 8]");
  if (!o || !out) return fail(IVRQ_EINVAL, "ivrq_quantize_oracle: null pointer");
  if (workspace_bytes < ivrq_quantize_oracle_workspace(dims, bits))
    return fail(IVRQ_ENOMEM, "ivrq_quantize_oracle: workspace too small");
  const int64_t m = (int64_t)dims * ((1 << (bits - 1)) - 1);
  int64_t cap = 1;
  while (cap < m) cap <<= 1;
  ops::QoArgs a{};
  a.o = o;
  a.d = dims;
  a.bits = bits;
  a.cap = cap;
  a.crit = static_cast<double*>(workspace);
  a.cosv = a.crit + cap;
  a.out = out;
  ops::quantize_oracle_kernel<<<1, ops::QO_THREADS, 0, as_stream(stream)>>>(a);
  return check_launch("ivrq_quantize_oracle");
}
