// Search path: query rotation, coarse probe, query preparation and the fused
// two-stage list scan.  Reference: search.py (search_batch 390-454).
#include <algorithm>

#include "ivrq_common.cuh"
#include "ivrq_gemm.cuh"

namespace ivrq {

// ============================================================ query rotation
// q_rot[i][j] = sum_k q[i][k] * R[j][k]   (search.py:422: q @ rotation.T)
struct StoreF64 {
  double* out;
  int64_t ld;
  __device__ __forceinline__ void operator()(int64_t r, int64_t c, double v) const { out[r * ld + c] = v; }
};

// ============================================================ probe distances
// d = max((q_sq + c_sq) - 2 * <q, c>, 0)  (search.py:240-242)
struct ProbeDistEpi {
  const double* q_sq;
  const double* c_sq;
  double* out;
  int64_t ld;
  __device__ __forceinline__ void operator()(int64_t r, int64_t c, double dot) const {
    double d = dsub(dadd(q_sq[r], c_sq[c]), dmul(2.0, dot));
    out[r * ld + c] = dmax(d, 0.0);
  }
};

// Per-query exact top-n_probe selection by (distance, id) over one row of the
// distance matrix: an MSB-first 8-bit radix select on the (non-negative)
// float64 bit patterns, then an id-ordered compaction.  order_by_id=0 also
// ranks the selected set by (distance, id) like np.argsort(kind="stable").
__global__ void __launch_bounds__(256) probe_select_kernel(const double* __restrict__ dist, int64_t row_base,
                                                           int32_t nlist, int32_t nprobe, int32_t order_by_id,
                                                           int64_t* __restrict__ ids_out,
                                                           double* __restrict__ d2_out) {
  __shared__ int32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int32_t s_need;
  __shared__ int32_t warp_tot[8];
  __shared__ int32_t s_base;
  __shared__ int32_t s_eq_base;
  const int64_t q = row_base + blockIdx.x;
  const double* row = dist + (int64_t)blockIdx.x * nlist;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  uint64_t prefix = 0, mask = 0;
  int need = nprobe;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < nlist; i += blockDim.x) {
      uint64_t key = (uint64_t)__double_as_longlong(row[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255], 1);
    }
    __syncthreads();
    if (tid == 0) {
      int cum = 0, digit = 255;
      for (int b = 0; b < 256; ++b) {
        if (cum + hist[b] >= need) {
          digit = b;
          break;
        }
        cum += hist[b];
      }
      s_prefix = prefix | ((uint64_t)digit << shift);
      s_need = need - cum;
    }
    __syncthreads();
    prefix = s_prefix;
    need = s_need;
    mask |= (uint64_t)255 << shift;
    __syncthreads();
  }
  const uint64_t kth = prefix;  // key of the n_probe-th smallest
  // `need` = how many elements equal to kth are taken (the lowest ids)
  // ordered compaction, ascending cluster id
  int64_t* out_i = ids_out + q * nprobe;
  double* out_d = d2_out + q * nprobe;
  if (tid == 0) {
    s_base = 0;
    s_eq_base = 0;
  }
  __syncthreads();
  for (int c0 = 0; c0 < nlist; c0 += blockDim.x) {
    int i = c0 + tid;
    uint64_t key = 0;
    bool lt = false, eq = false;
    if (i < nlist) {
      key = (uint64_t)__double_as_longlong(row[i]);
      lt = key < kth;
      eq = key == kth;
    }
    // rank of equal keys in id order
    unsigned eqb = __ballot_sync(0xffffffffu, eq);
    unsigned ltb = __ballot_sync(0xffffffffu, lt);
    __shared__ int32_t weq[8], wlt[8];
    if (lane == 0) {
      weq[wid] = __popc(eqb);
      wlt[wid] = __popc(ltb);
    }
    __syncthreads();
    int eq_before = s_eq_base, lt_before = 0;
    for (int w = 0; w < wid; ++w) eq_before += weq[w];
    eq_before += __popc(eqb & ((1u << lane) - 1));
    bool take = lt || (eq && eq_before < need);
    unsigned tb = __ballot_sync(0xffffffffu, take);
    if (lane == 0) warp_tot[wid] = __popc(tb);
    __syncthreads();
    int pos = s_base;
    for (int w = 0; w < wid; ++w) pos += warp_tot[w];
    pos += __popc(tb & ((1u << lane) - 1));
    if (take) {
      out_i[pos] = i;
      out_d[pos] = row[i];
    }
    (void)lt_before;
    __syncthreads();
    if (tid == 0) {
      int tot = 0, te = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        tot += warp_tot[w];
        te += weq[w];
      }
      s_base += tot;
      s_eq_base += te;
    }
    __syncthreads();
  }
  if (!order_by_id) {
    // rank the selected set by (distance, id); n_probe is modest for this API path
    __syncthreads();
    extern __shared__ unsigned char sel_smem[];
    double* sd = reinterpret_cast<double*>(sel_smem);
    int64_t* si = reinterpret_cast<int64_t*>(sd + nprobe);
    for (int e = tid; e < nprobe; e += blockDim.x) {
      sd[e] = out_d[e];
      si[e] = out_i[e];
    }
    __syncthreads();
    for (int e = tid; e < nprobe; e += blockDim.x) {
      double de = sd[e];
      int64_t ie = si[e];
      int rank = 0;
      for (int f = 0; f < nprobe; ++f) rank += key_less(sd[f], si[f], de, ie) ? 1 : 0;
      out_i[rank] = ie;
      out_d[rank] = de;
    }
  }
}

// ============================================================ query prep
// One warp per query: QueryState of _prepare_from_rotated (search.py:186-214)
// and build_luts (search.py:115-132).
__global__ void prepare_kernel(const double* __restrict__ q_rot, int64_t nq, int d, int mode, int qbits,
                               int index_bits, double eps_bound, double* __restrict__ scalars,
                               uint32_t* __restrict__ planes, float* __restrict__ luts) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const double* x = q_rot + q * d;
  const int g = words_per_vector(d);
  double sum_q = 0.0;
  if (lane == 0) sum_q = pairwise_sum_seq(x, d);
  sum_q = __shfl_sync(0xffffffffu, sum_q, 0);
  const double k_b = ((double)((1 << index_bits) - 1)) / 2.0;
  double* sc = scalars + q * IVRQ_QS_COUNT;
  if (mode == IVRQ_IP_LUT) {
    // L[j][key] = float32(sum over set bits i of key of q[4j+i]), dims padded with 0
    const int nblk = 8 * g;
    for (int e = lane; e < nblk * 16; e += 32) {
      int j = e / 16, key = e % 16;
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int dim = 4 * j + i;
        double v = dim < d ? x[dim] : 0.0;
        acc = dadd(acc, dmul(v, (double)((key >> i) & 1)));
      }
      luts[q * nblk * 16 + e] = (float)acc;
    }
    if (lane == 0) {
      sc[IVRQ_QS_SUM_Q] = sum_q;
      sc[IVRQ_QS_DELTA] = 1.0;
      sc[IVRQ_QS_CODE_SUM] = sum_q;  // QueryState.__post_init__ (search.py:102-104)
      sc[IVRQ_QS_IP_MARGIN] = 0.0;
      sc[IVRQ_QS_KB_SUM] = dmul(k_b, sum_q);
      sc[IVRQ_QS_HALF_CODE] = dmul(0.5, sum_q);
    }
    return;
  }
  // bitwise: delta, q_hat = clip(rint(q/delta)), two's-complement planes
  double mx = 0.0;
  for (int i = lane; i < d; i += 32) mx = dmax(mx, fabs(x[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = dmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int half = 1 << (qbits - 1);
  const double delta = mx > 0.0 ? ddiv(mx, (double)(half - 1)) : 1.0;
  long long qsum = 0;
  for (int gi = 0; gi < g; ++gi) {
    int dim = gi * 32 + lane;
    int qh = 0;
    if (dim < d) {
      double r = rint(ddiv(x[dim], delta));
      r = r < (double)(-half) ? (double)(-half) : r;
      r = r > (double)(half - 1) ? (double)(half - 1) : r;
      qh = (int)r;
    }
    qsum += qh;
    unsigned twos = (unsigned)qh & ((1u << qbits) - 1u);
    for (int j = 0; j < qbits; ++j) {
      unsigned w = __ballot_sync(0xffffffffu, (twos >> j) & 1u);
      if (lane == 0) planes[(q * qbits + j) * g + gi] = w;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) qsum += __shfl_xor_sync(0xffffffffu, qsum, o);
  if (lane == 0) {
    double code_sum = dmul(delta, (double)qsum);
    double ipm = dmul(dmul(eps_bound, delta), dsqrt(ddiv((double)d, 24.0)));
    sc[IVRQ_QS_SUM_Q] = sum_q;
    sc[IVRQ_QS_DELTA] = delta;
    sc[IVRQ_QS_CODE_SUM] = code_sum;
    sc[IVRQ_QS_IP_MARGIN] = ipm;
    sc[IVRQ_QS_KB_SUM] = dmul(k_b, sum_q);
    sc[IVRQ_QS_HALF_CODE] = dmul(0.5, code_sum);
  }
}

// ============================================================ fused scan
namespace scan {

constexpr int THREADS = 256;
constexpr int CHUNK = 1024;  // vectors of one list handled per stage-1 pass

struct Args {
  ivrq_index_view ix;
  const double* q_rot;
  const int64_t* probe_ids;
  const double* probe_d2;
  const double* scalars;
  const uint32_t* planes;
  const float* luts;
  int64_t nq;
  int k, nprobe, qbits, prune;
  int g, eb, exw;
  int sort_n;  // power of two >= CHUNK + k
  int64_t* out_ids;
  double* out_dists;
  int32_t* out_counts;
  int64_t* stats;
};

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

// block-wide bitonic sort (ascending (key, id)) of n (power of two) entries
__device__ void bitonic_sort(double* key, int64_t* id, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        int lo = 2 * t - (t & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        double kl = key[lo], kh = key[hi];
        int64_t il = id[lo], ih = id[hi];
        bool swap = up ? key_less(kh, ih, kl, il) : key_less(kl, il, kh, ih);
        if (swap) {
          key[lo] = kh;
          key[hi] = kl;
          id[lo] = ih;
          id[hi] = il;
        }
      }
    }
  }
  __syncthreads();
}

// Extract the 32 ex-code fields (eb bits each, LSB-first) of one 32-dim group
// and accumulate sum_i u_i * q_i with u_i = msb_i << eb | ex_i.
template <int EB>
__device__ __forceinline__ double group_dot(const uint32_t* __restrict__ exg, uint32_t msb, const double* q) {
  double acc = 0.0;
  if constexpr (EB == 0) {
#pragma unroll
    for (int i = 0; i < 32; ++i) acc = fma((double)((msb >> i) & 1u), q[i], acc);
  } else {
    uint32_t w[EB + 1];
#pragma unroll
    for (int i = 0; i < EB; ++i) w[i] = exg[i];
    w[EB] = 0u;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      constexpr uint32_t mask = (1u << EB) - 1u;
      const int bit = i * EB;
      const int wi = bit >> 5, off = bit & 31;
      const uint64_t win = ((uint64_t)w[wi + 1] << 32) | (uint64_t)w[wi];
      const uint32_t field = (uint32_t)(win >> off) & mask;
      const uint32_t u = ((((msb >> i) & 1u)) << EB) | field;
      acc = fma((double)u, q[i], acc);
    }
  }
  return acc;
}

template <int MODE, int EB, bool REFINE>
__global__ void __launch_bounds__(THREADS) scan_kernel(Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int64_t q = blockIdx.x;
  if (q >= a.nq) return;
  const int d = a.ix.dims, g = a.g, k = a.k;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // ---- shared memory carve-up
  double* s_q = reinterpret_cast<double*>(smem);                 // [32*g] rotated query (refine)
  double* s_sortk = s_q + 32 * g;                                  // [sort_n]
  int64_t* s_sorti = reinterpret_cast<int64_t*>(s_sortk + a.sort_n);  // [sort_n]
  double* s_pool_d = reinterpret_cast<double*>(s_sorti + a.sort_n);   // [k]
  int64_t* s_pool_i = reinterpret_cast<int64_t*>(s_pool_d + k);       // [k]
  double* s_cd = reinterpret_cast<double*>(s_pool_i + k);             // [CHUNK] candidate dist
  int32_t* s_cv = reinterpret_cast<int32_t*>(s_cd + CHUNK);          // [CHUNK] candidate row
  uint32_t* s_planes = reinterpret_cast<uint32_t*>(s_cv + CHUNK);    // [qbits*g]
  float* s_lut = reinterpret_cast<float*>(s_planes + (MODE == IVRQ_IP_BITWISE ? a.qbits * g : 0));  // [8g*16]
  __shared__ int s_ncand, s_nfilt, s_pool_n;
  __shared__ double s_T;
  __shared__ long long s_probed, s_surv;

  if (REFINE) {
    for (int i = tid; i < 32 * g; i += THREADS) s_q[i] = i < d ? a.q_rot[q * d + i] : 0.0;
  }
  if (MODE == IVRQ_IP_BITWISE) {
    for (int i = tid; i < a.qbits * g; i += THREADS) s_planes[i] = a.planes[q * a.qbits * g + i];
  } else {
    for (int i = tid; i < 8 * g * 16; i += THREADS) s_lut[i] = a.luts[q * 8 * g * 16 + i];
  }
  const double* sc = a.scalars + q * IVRQ_QS_COUNT;
  const double delta = sc[IVRQ_QS_DELTA];
  const double half_code = sc[IVRQ_QS_HALF_CODE];
  const double ipm = sc[IVRQ_QS_IP_MARGIN];
  const double kb_sum = sc[IVRQ_QS_KB_SUM];
  if (tid == 0) {
    s_pool_n = 0;
    s_T = dinf();
    s_probed = 0;
    s_surv = 0;
  }
  __syncthreads();

  const int64_t* pid_list = a.probe_ids + q * a.nprobe;
  const double* pd2_list = a.probe_d2 + q * a.nprobe;
  for (int p = 0; p < a.nprobe; ++p) {  // ascending cluster id (search.py:429)
    const int64_t c = pid_list[p];
    const double d_qc2 = pd2_list[p];
    const int64_t lo = a.ix.offsets[c], hi = a.ix.offsets[c + 1];
    const int64_t n_c = hi - lo;
    if (n_c == 0) continue;
    const double T_list = a.prune ? s_T : dinf();
    const double sq = dsqrt(d_qc2);
    const uint32_t* words = a.ix.packed_msb + (int64_t)g * lo;
    for (int64_t c0 = 0; c0 < n_c; c0 += CHUNK) {
      const int cn = (int)min((int64_t)CHUNK, n_c - c0);
      if (tid == 0) s_ncand = 0;
      __syncthreads();
      // ---------------- stage 1: binary estimate + lower bound, prune
      for (int vb = 0; vb < cn; vb += THREADS) {
        const int vi = vb + tid;
        bool keep = false;
        double est2 = 0.0;
        if (vi < cn) {
          const int64_t v = c0 + vi;
          double ipb;
          if (MODE == IVRQ_IP_BITWISE) {
            int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int gi = 0; gi < g; ++gi) {
              uint32_t w = words[(int64_t)gi * n_c + v];
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (j < a.qbits) cnt[j] += __popc(w & s_planes[j * g + gi]);
            }
            long long raw = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (j < a.qbits - 1) raw += (long long)cnt[j] << j;
              else if (j == a.qbits - 1) raw -= (long long)cnt[j] << j;
            }
            ipb = dmul(delta, (double)raw);
          } else {
            double acc = 0.0;
            for (int gi = 0; gi < g; ++gi) {
              uint32_t w = words[(int64_t)gi * n_c + v];
#pragma unroll
              for (int s = 0; s < 8; ++s) acc = dadd(acc, (double)s_lut[(gi * 8 + s) * 16 + ((w >> (4 * s)) & 15u)]);
            }
            ipb = acc;
          }
          const double add = (double)a.ix.short_add[lo + v];
          const double scale = (double)a.ix.short_scale[lo + v];
          const double err = (double)a.ix.short_err[lo + v];
          const double ip_signed = dsub(ipb, half_code);
          est2 = dmax(dsub(dadd(add, d_qc2), dmul(scale, ip_signed)), 0.0);
          if (est2 <= T_list) {
            keep = true;  // lb2 <= est2 <= T
          } else {
            double margin = dmul(err, sq);
            if (ipm != 0.0) {
              double sm = dmul(scale, ipm);
              margin = dsqrt(dadd(dmul(margin, margin), dmul(sm, sm)));
            }
            double lb2 = dmax(dsub(est2, margin), 0.0);
            keep = lb2 <= T_list;
          }
        }
        unsigned kb = __ballot_sync(0xffffffffu, keep);
        int base = 0;
        if (lane == 0 && kb) base = atomicAdd(&s_ncand, __popc(kb));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) {
          int pos = base + __popc(kb & ((1u << lane) - 1u));
          s_cv[pos] = vi;
          s_cd[pos] = est2;
        }
      }
      __syncthreads();
      const int ncand = s_ncand;
      if (tid == 0) {
        s_probed += cn;
        s_surv += ncand;
      }
      // ---------------- stage 2: refine survivors with the full code
      if (REFINE && ncand > 0) {
        // lanes per candidate: power of two >= g, capped at 32
        int lpc = 1;
        while (lpc < g && lpc < 32) lpc <<= 1;
        const int cpw = 32 / lpc;  // candidates per warp per step
        const int sub = lane / lpc, sl = lane % lpc;
        for (int cb = wid * cpw; cb < ncand; cb += (THREADS / 32) * cpw) {
          const int ci = cb + sub;
          double acc = 0.0;
          int64_t row = 0;
          if (ci < ncand) {
            const int64_t v = c0 + s_cv[ci];
            row = lo + v;
            const uint32_t* exrow = a.ix.excodes + row * a.exw;
            for (int gi = sl; gi < g; gi += lpc) {
              uint32_t msb = words[(int64_t)gi * n_c + v];
              acc += group_dot<EB>(exrow + gi * EB, msb, s_q + gi * 32);
            }
          }
          for (int o = lpc >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          if (ci < ncand && sl == 0) {
            const float2 lf = reinterpret_cast<const float2*>(a.ix.long_factors)[row];
            double dist = dmax(dsub(dadd((double)lf.x, d_qc2), dmul((double)lf.y, dsub(acc, kb_sum))), 0.0);
            s_cd[ci] = dist;
          }
        }
        __syncthreads();
      }
      // ---------------- merge survivors into the running pool
      if (ncand > 0) {
        if (tid == 0) s_nfilt = 0;
        __syncthreads();
        const int pn = s_pool_n;
        const bool full = pn >= k;
        const double kd = full ? s_pool_d[k - 1] : 0.0;
        const int64_t kid = full ? s_pool_i[k - 1] : 0;
        for (int cb = 0; cb < ncand; cb += THREADS) {
          const int ci = cb + tid;
          bool pass = false;
          double dist = 0.0;
          int64_t pid = 0;
          if (ci < ncand) {
            dist = s_cd[ci];
            pid = a.ix.pids[lo + c0 + s_cv[ci]];
            pass = !full || key_less(dist, pid, kd, kid);
          }
          unsigned pb = __ballot_sync(0xffffffffu, pass);
          int base = 0;
          if (lane == 0 && pb) base = atomicAdd(&s_nfilt, __popc(pb));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (pass) {
            int pos = pn + base + __popc(pb & ((1u << lane) - 1u));
            s_sortk[pos] = dist;
            s_sorti[pos] = pid;
          }
        }
        __syncthreads();
        const int m = s_nfilt;
        if (m > 0) {
          for (int i = tid; i < pn; i += THREADS) {
            s_sortk[i] = s_pool_d[i];
            s_sorti[i] = s_pool_i[i];
          }
          int tot = pn + m;
          int n2 = 1;
          while (n2 < tot) n2 <<= 1;
          for (int i = tot + tid; i < n2; i += THREADS) {
            s_sortk[i] = dinf();
            s_sorti[i] = 0x7fffffffffffffffLL;
          }
          bitonic_sort(s_sortk, s_sorti, n2);
          const int newn = min(tot, k);
          for (int i = tid; i < newn; i += THREADS) {
            s_pool_d[i] = s_sortk[i];
            s_pool_i[i] = s_sorti[i];
          }
          __syncthreads();
          if (tid == 0) s_pool_n = newn;
        }
        __syncthreads();
      }
    }
    // threshold update after the whole list (search.py:444-447)
    if (tid == 0 && s_pool_n >= k) s_T = s_pool_d[k - 1];
    __syncthreads();
  }
  const int pn = s_pool_n;
  for (int i = tid; i < k; i += THREADS) {
    a.out_ids[q * k + i] = i < pn ? s_pool_i[i] : -1;
    a.out_dists[q * k + i] = i < pn ? s_pool_d[i] : dinf();
  }
  if (tid == 0) {
    a.out_counts[q] = pn;
    if (a.stats) {
      a.stats[2 * q] = s_probed;
      a.stats[2 * q + 1] = s_surv;
    }
  }
}

size_t smem_bytes(const Args& a, int mode) {
  size_t b = 0;
  b += sizeof(double) * 32 * a.g;
  b += (sizeof(double) + sizeof(int64_t)) * a.sort_n;
  b += (sizeof(double) + sizeof(int64_t)) * a.k;
  b += (sizeof(double) + sizeof(int32_t)) * CHUNK;
  b += mode == IVRQ_IP_BITWISE ? sizeof(uint32_t) * a.qbits * a.g : sizeof(float) * 8 * a.g * 16;
  return b + 64;
}

template <int MODE, int EB, bool REFINE>
int launch_t(const Args& a, cudaStream_t s) {
  size_t sm = smem_bytes(a, MODE);
  auto kern = scan_kernel<MODE, EB, REFINE>;
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return fail(IVRQ_EUNSUP, "ivrq_search_scan: shared memory request too large");
  }
  kern<<<(unsigned)a.nq, THREADS, sm, s>>>(a);
  return check_launch("ivrq_search_scan");
}

template <int MODE>
int launch_mode(const Args& a, bool refine, cudaStream_t s) {
  if (!refine) return launch_t<MODE, 0, false>(a, s);
  switch (a.eb) {
    case 1: return launch_t<MODE, 1, true>(a, s);
    case 2: return launch_t<MODE, 2, true>(a, s);
    case 3: return launch_t<MODE, 3, true>(a, s);
    case 4: return launch_t<MODE, 4, true>(a, s);
    case 5: return launch_t<MODE, 5, true>(a, s);
    case 6: return launch_t<MODE, 6, true>(a, s);
    case 7: return launch_t<MODE, 7, true>(a, s);
    default: return fail(IVRQ_EUNSUP, "ivrq_search_scan: bits out of range");
  }
}

}  // namespace scan
}  // namespace ivrq

using namespace ivrq;

extern "C" int ivrq_rotate_queries(const void* q, int q_is_f64, int64_t nq, int32_t dims,
                                   const float* rotation, double* q_rot, void* stream) {
  if (nq < 0 || dims <= 0) return fail(IVRQ_EINVAL, "ivrq_rotate_queries: bad sizes");
  gemm::RowMajor<float> lb{rotation, dims, dims};
  StoreF64 epi{q_rot, dims};
  if (q_is_f64) {
    gemm::RowMajor<double> la{(const double*)q, nq, dims};
    return gemm::launch_gemm(la, nq, lb, dims, dims, epi, as_stream(stream), "ivrq_rotate_queries");
  }
  gemm::RowMajor<float> la{(const float*)q, nq, dims};
  return gemm::launch_gemm(la, nq, lb, dims, dims, epi, as_stream(stream), "ivrq_rotate_queries");
}

static int64_t probe_chunk_rows(int64_t nq, int32_t n_clusters) {
  // bytes of distance matrix per pass: enough for >= 256 query rows so the
  // GEMM tiles stay full even when "clusters" are a whole base set (exact k-NN)
  const int64_t budget = std::max<int64_t>((int64_t)256 << 20, (int64_t)256 * n_clusters * 8);
  int64_t rows = budget / ((int64_t)n_clusters * 8);
  rows = std::max<int64_t>(rows, 1);
  return std::min<int64_t>(rows, std::max<int64_t>(nq, 1));
}

extern "C" size_t ivrq_select_clusters_workspace(int64_t nq, int32_t n_clusters) {
  int64_t rows = probe_chunk_rows(nq, n_clusters);
  return (size_t)(rows * n_clusters * 8 + nq * 8 + 256);
}

extern "C" int ivrq_select_clusters(const double* q_rot, int64_t nq, int32_t dims, const float* centroids,
                                    const double* centroid_sqnorms, int32_t n_clusters, int32_t n_probe,
                                    int64_t* ids, double* d2, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  return ivrq_select_clusters_ordered(q_rot, nq, dims, centroids, centroid_sqnorms, n_clusters, n_probe, 0, ids,
                                      d2, workspace, workspace_bytes, stream);
}

extern "C" int ivrq_select_clusters_ordered(const double* q_rot, int64_t nq, int32_t dims,
                                            const float* centroids, const double* centroid_sqnorms,
                                            int32_t n_clusters, int32_t n_probe, int32_t order_by_id,
                                            int64_t* ids, double* d2, void* workspace, size_t workspace_bytes,
                                            void* stream) {
  if (n_probe < 1 || n_probe > n_clusters)
    return fail(IVRQ_EINVAL, "n_probe=" + std::to_string(n_probe) + " exceeds " + std::to_string(n_clusters) +
                                 " clusters");
  if (nq == 0) return IVRQ_OK;
  if (workspace_bytes < ivrq_select_clusters_workspace(nq, n_clusters))
    return fail(IVRQ_ENOMEM, "ivrq_select_clusters: workspace too small");
  cudaStream_t s = as_stream(stream);
  const int64_t rows = probe_chunk_rows(nq, n_clusters);
  double* dist = reinterpret_cast<double*>(workspace);
  double* q_sq = dist + rows * n_clusters;
  IVRQ_TRY(ivrq_row_sqnorms(q_rot, 1, nq, dims, q_sq, stream));
  gemm::RowMajor<float> lb{centroids, n_clusters, dims};
  size_t sel_smem = order_by_id ? 0 : (size_t)n_probe * 16;
  if (sel_smem > 48 * 1024) {
    if (cudaFuncSetAttribute(probe_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sel_smem) !=
        cudaSuccess)
      return fail(IVRQ_EUNSUP, "ivrq_select_clusters: n_probe too large for distance ordering");
  }
  for (int64_t r0 = 0; r0 < nq; r0 += rows) {
    const int64_t rn = std::min(rows, nq - r0);
    gemm::RowMajor<double> la{q_rot + r0 * dims, rn, dims};
    ProbeDistEpi epi{q_sq + r0, centroid_sqnorms, dist, n_clusters};
    IVRQ_TRY(gemm::launch_gemm(la, rn, lb, n_clusters, dims, epi, s, "ivrq_select_clusters(gemm)"));
    probe_select_kernel<<<(unsigned)rn, 256, sel_smem, s>>>(dist, r0, n_clusters, n_probe, order_by_id, ids, d2);
    IVRQ_TRY(check_launch("ivrq_select_clusters(select)"));
  }
  return IVRQ_OK;
}

extern "C" int ivrq_prepare_queries(const double* q_rot, int64_t nq, int32_t dims,
                                    const ivrq_search_params* params, int32_t index_bits, double eps_bound,
                                    double* scalars, uint32_t* planes, float* luts, void* stream) {
  if (!params) return fail(IVRQ_EINVAL, "ivrq_prepare_queries: null params");
  if (params->ip_mode == IVRQ_IP_BITWISE && (params->query_bits < 2 || params->query_bits > 8))
    return fail(IVRQ_EINVAL, "query_bits must be in [2, 8]");
  if (params->ip_mode == IVRQ_IP_BITWISE && !planes) return fail(IVRQ_EINVAL, "bitwise mode needs planes");
  if (params->ip_mode == IVRQ_IP_LUT && !luts) return fail(IVRQ_EINVAL, "lut mode needs luts");
  if (nq == 0) return IVRQ_OK;
  const int wpb = 4;
  prepare_kernel<<<(unsigned)ceil_div(nq, wpb), wpb * 32, 0, as_stream(stream)>>>(
      q_rot, nq, dims, params->ip_mode, params->query_bits, index_bits, eps_bound, scalars, planes, luts);
  return check_launch("ivrq_prepare_queries");
}

extern "C" int ivrq_search_scan(const ivrq_index_view* index, const double* q_rot, const int64_t* probe_ids,
                                const double* probe_d2, const double* scalars, const uint32_t* planes,
                                const float* luts, int64_t nq, const ivrq_search_params* params,
                                int64_t* out_ids, double* out_dists, int32_t* out_counts, int64_t* stats,
                                void* stream) {
  if (!index || !params) return fail(IVRQ_EINVAL, "ivrq_search_scan: null argument");
  if (params->k < 1) return fail(IVRQ_EINVAL, "k must be >= 1");
  if (params->k > 4096) return fail(IVRQ_EUNSUP, "ivrq_search_scan: k > 4096 not supported");
  if (index->bits < 1 || index->bits > 8) return fail(IVRQ_EINVAL, "index bits out of range");
  if (nq == 0) return IVRQ_OK;
  scan::Args a{};
  a.ix = *index;
  a.q_rot = q_rot;
  a.probe_ids = probe_ids;
  a.probe_d2 = probe_d2;
  a.scalars = scalars;
  a.planes = planes;
  a.luts = luts;
  a.nq = nq;
  a.k = params->k;
  a.nprobe = params->n_probe;
  a.qbits = params->query_bits;
  a.prune = params->prune;
  a.g = words_per_vector(index->dims);
  a.eb = index->bits - 1;
  a.exw = a.eb * a.g;
  int n2 = 1;
  while (n2 < scan::CHUNK + a.k) n2 <<= 1;
  a.sort_n = n2;
  a.out_ids = out_ids;
  a.out_dists = out_dists;
  a.out_counts = out_counts;
  a.stats = stats;
  const bool refine = params->refine && index->bits >= 2;
  cudaStream_t s = as_stream(stream);
  if (params->ip_mode == IVRQ_IP_BITWISE) return scan::launch_mode<IVRQ_IP_BITWISE>(a, refine, s);
  return scan::launch_mode<IVRQ_IP_LUT>(a, refine, s);
}
