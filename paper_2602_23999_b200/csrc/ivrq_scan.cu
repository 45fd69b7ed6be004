// The fused two-stage list scan + top-k (search.py:326-387 inside the
// per-query loop 425-448).  One CTA per query visits the query's probed
// lists in ascending cluster id; within a list:
//   stage 1  every vector: binary inner product (AND+POPC against the query's
//            bit planes, or 4-bit LUT lookups), float64 estimate + lower bound,
//            prune lb2 <= T with T the K-th best distance before this list;
//   stage 2  survivors: full-code inner product <u, q_rot> on the int8 tensor
//            cores (mma.sync m16n8k32: 16 survivors x 8 digit slices of the
//            query), combined exactly in integers and rounded once to float64;
//            then the refined estimate;
//   merge    survivors into the running (dist, pid) top-k; after the list
//            T := pool[k-1] once the pool holds k entries.
// The threshold trajectory, and therefore every prune decision, is the
// reference's.  k <= 32 keeps per-warp top-32 queues in registers (bitonic
// shuffle networks); larger k falls back to a block-wide bitonic sort.
#include <cstdlib>
#include <functional>
#include <type_traits>
#include <vector>

#include "ivrq_common.cuh"
#include "ivrq_tc.cuh"

namespace ivrq {
namespace scan {

constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int CHUNK = 512;             // vectors of one list per stage-1 pass
constexpr int VPT = CHUNK / THREADS;   // vectors per thread per pass
constexpr int SLICES = 8;              // base-128 digits of the query (refine)
constexpr int SPAD = 16;               // slice row padding (bank spread)
constexpr unsigned FULL = 0xffffffffu;
constexpr int64_t NO_ID = 0x7fffffffffffffffLL;
// list-major stage-1 inner products (ip_list_kernel)
constexpr int TQ = 64;   // queries per tile: 4 m16 tiles, every warp
constexpr int TV = 256;  // vectors per tile: 8 warps x 4 n8 tiles
constexpr int TQ_PAD = 16;

// ip row of a (list, query) pair: n_c rounded up to 8 elements
__host__ __device__ inline int64_t ip_row_stride(int64_t n_c) { return (n_c + 7) & ~int64_t(7); }

struct Args {
  ivrq_index_view ix;
  const int64_t* probe_ids;
  const double* probe_d2;
  const double* scalars;
  const uint32_t* planes;
  const float* luts;
  const int8_t* qslices;
  const int64_t* qorder;  // CTA -> query (queries grouped by first probed list)
  int skip_first;         // the first in-range probe was handled by first_list_kernel
  int64_t nq;
  int k, nprobe, qbits, prune;
  int64_t list_lo, list_hi;  // global cluster ids held by this (shard of the) index
  const int64_t* init_ids;   // optional pool carried in (exact ascending-id chain)
  const double* init_dists;
  const int32_t* init_counts;
  int g, kpad;
  int sort_n;  // big-k path: power of two >= CHUNK + k
  int64_t* out_ids;
  double* out_dists;
  int32_t* out_counts;
  int64_t* stats;
  // stage-1 inner products precomputed list-major (ip_list_kernel), or null
  const void* ipbuf;
  const int32_t* pslot;      // [nq * nprobe] slot of (q, p) in its list's bucket
  const int64_t* pair_base;  // [nlist + 1]
  // refined distances of every vector of each query's first list (first_dist_kernel), or null:
  // row of qorder slot i (bucket c) at fdist + fbase[c] + (i - qoff[c]) * ip_row_stride(n_c)
  const double* fdist;
  const int64_t* fbase;
  const int64_t* qoff;
  int l2_prefetch;  // warp kernel: L2 prefetch of survivor rcode rows
  // per (query, probe) list metadata (probe_meta_kernel), so the warp kernels prefetch the next
  // list's CSR bounds and row base one list ahead instead of chaining dependent loads per list
  const int64_t* m_lo;      // [nq * nprobe] first row of the probed list
  const int32_t* m_nc;      // [nq * nprobe] its size, -1 = another shard's list
  const int64_t* m_base;    // [nq * nprobe] (list, query) pair row base in ipbuf / rdist
  // approximate refined distance of every probed (pair, vector) (tc_refine_kernel), or null, and
  // the per-query radius bounding its distance to the exact value (rd_radius_kernel)
  const float* rdist;
  const double* rrad;
  int32_t* fix_count;        // queries the approximate pass could not certify (rerun exactly), and
  int32_t* fix_list;         // their ids
  const float4* sf4;         // (add, scale, err, 0) per vector: one 16-byte load (pack_short_kernel), or null
  double* fin_d;             // [nq][32] the approximate pass's queue, for rda_final_kernel
  int64_t* fin_e;
  const int32_t* fix_only;   // scan_warp_kernel as the rerun: process only slots < *fix_only_count ...
  const int32_t* fix_only_count;  // ... of fix_only
  int32_t* rda_next;         // scan_rda_kernel's query-slot counter (zeroed), or null: one slot per warp
};

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7ff0000000000000LL); }

struct QueryCtx {
  double delta, half_code, ipm, kb_sum;
  int sexp;
};

// ------------------------------------------------------------ stage 1
// Fills s_cv (row within list) / s_cd (stage-1 estimate) with the survivors of
// vectors [c0, c0+cn) of the list; returns the count via s_ncand.
template <int MODE, int QB, int IPB>
__device__ __forceinline__ void stage1_chunk(const Args& a, const QueryCtx& qc, const uint32_t* __restrict__ words,
                                             int64_t lo, int64_t n_c, int64_t c0, int cn, double d_qc2, double sq,
                                             double T_list, const uint32_t* s_planes8, const float* s_lut,
                                             int32_t* s_cv, double* s_cd, int* s_ncand, const void* iprow) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int g = a.g;
  double ipb[VPT];
  if (IPB) {  // integer inner products from ip_list_kernel (same integer as the popcount sum below)
    using IPT = typename std::conditional<IPB == 2, int16_t, int32_t>::type;
    const IPT* r = reinterpret_cast<const IPT*>(iprow) + c0;
#pragma unroll
    for (int u = 0; u < VPT; ++u) {
      const int vi = tid + u * THREADS;
      ipb[u] = dmul(qc.delta, (double)(vi < cn ? (int)__ldg(r + vi) : 0));
    }
  } else if (MODE == IVRQ_IP_BITWISE) {
    int pos[VPT], last[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) pos[u] = last[u] = 0;
    const int qb = QB ? QB : a.qbits;
    constexpr int GB = 8;  // 32-dim groups whose words are in flight together
    for (int g0 = 0; g0 < g; g0 += GB) {
      uint32_t wv[GB][VPT];
#pragma unroll
      for (int j = 0; j < GB; ++j)
#pragma unroll
        for (int u = 0; u < VPT; ++u) {
          const int vi = tid + u * THREADS;
          wv[j][u] = (g0 + j < g && vi < cn) ? __ldg(words + (int64_t)(g0 + j) * n_c + c0 + vi) : 0u;
        }
#pragma unroll
      for (int j = 0; j < GB; ++j) {
      const int gi = g0 + j;
      if (gi >= g) break;
      const uint4 pa = *reinterpret_cast<const uint4*>(s_planes8 + gi * 8);
      uint4 pb = make_uint4(0u, 0u, 0u, 0u);
      if (QB == 0 || QB > 4) pb = *reinterpret_cast<const uint4*>(s_planes8 + gi * 8 + 4);
      const uint32_t pl[8] = {pa.x, pa.y, pa.z, pa.w, pb.x, pb.y, pb.z, pb.w};
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const uint32_t w = wv[j][u];
        if (QB) {
#pragma unroll
          for (int b = 0; b < QB; ++b) pos[u] += __popc(w & pl[b]) << b;
          last[u] += __popc(w & pl[QB - 1]);
        } else {
#pragma unroll
          for (int b = 0; b < 8; ++b) {
            if (b < qb) {
              const int c = __popc(w & pl[b]);
              pos[u] += c << b;
              if (b == qb - 1) last[u] += c;
            }
          }
        }
      }
      }
    }
#pragma unroll
    for (int u = 0; u < VPT; ++u) ipb[u] = dmul(qc.delta, (double)(pos[u] - (last[u] << qb)));
  } else {
    double acc[VPT];
#pragma unroll
    for (int u = 0; u < VPT; ++u) acc[u] = 0.0;
    for (int gi = 0; gi < g; ++gi) {
      const uint32_t* wrow = words + (int64_t)gi * n_c + c0;
      const float* lrow = s_lut + gi * 8 * 16;
#pragma unroll
      for (int u = 0; u < VPT; ++u) {
        const int vi = tid + u * THREADS;
        const uint32_t w = vi < cn ? __ldg(wrow + vi) : 0u;
#pragma unroll
        for (int s = 0; s < 8; ++s) acc[u] = dadd(acc[u], (double)lrow[s * 16 + ((w >> (4 * s)) & 15u)]);
      }
    }
#pragma unroll
    for (int u = 0; u < VPT; ++u) ipb[u] = acc[u];
  }
#pragma unroll
  for (int u = 0; u < VPT; ++u) {
    const int vi = tid + u * THREADS;
    bool keep = false;
    double est2 = 0.0;
    if (vi < cn) {
      const int64_t row = lo + c0 + vi;
      const double add = (double)__ldg(a.ix.short_add + row);
      const double scale = (double)__ldg(a.ix.short_scale + row);
      const double ip_signed = dsub(ipb[u], qc.half_code);
      est2 = dmax(dsub(dadd(add, d_qc2), dmul(scale, ip_signed)), 0.0);
      if (est2 <= T_list) {
        keep = true;  // lb2 <= est2 <= T
      } else {
        const double err = (double)__ldg(a.ix.short_err + row);
        double margin = dmul(err, sq);
        if (qc.ipm != 0.0) {
          // margin = sqrt(margin^2 + (scale*ipm)^2); decide lb2 <= T from the
          // squares when the answer is unambiguous by a wide (2^-38) margin,
          // otherwise evaluate the reference expression exactly.
          const double sm = dmul(scale, qc.ipm);
          const double S = dadd(dmul(margin, margin), dmul(sm, sm));
          const double gap = dsub(est2, T_list);
          const double g2 = dmul(gap, gap);
          if (S >= g2 * (1.0 + 0x1p-38)) {
            keep = true;
          } else if (S <= g2 * (1.0 - 0x1p-38) && gap > T_list * 0x1p-12) {
            keep = false;
          } else {
            keep = dmax(dsub(est2, dsqrt(S)), 0.0) <= T_list;
          }
        } else {
          keep = dmax(dsub(est2, margin), 0.0) <= T_list;
        }
      }
    }
    const unsigned kb = __ballot_sync(FULL, keep);
    int base = 0;
    if (lane == 0 && kb) base = atomicAdd(s_ncand, __popc(kb));
    base = __shfl_sync(FULL, base, 0);
    if (keep) {
      const int p = base + __popc(kb & ((1u << lane) - 1u));
      s_cv[p] = vi;
      s_cd[p] = est2;
    }
  }
}

// ------------------------------------------------------------ stage 2
__device__ __forceinline__ void mma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Refined distance of every candidate, in place in s_cd (search.py:313-323):
//   ip_u = <u, q_rot> = 2^(e-54) * sum_s 128^(7-s) * <u, D_s>
// with the int32 dot products <u, D_s> from the tensor cores (exact), the
// digit sum assembled in int64 (exact) and rounded once to float64.
template <bool NIB>
__device__ __forceinline__ void refine_chunk(const Args& a, const QueryCtx& qc, int64_t lo, int64_t c0, double d_qc2,
                                             const int8_t* s_slices, const int32_t* s_cv, double* s_cd, int ncand) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gid = lane >> 2, t4 = lane & 3;
  const int kp = a.kpad, ss = kp + SPAD;
  const int64_t rb = a.ix.rcode_bytes;
  const uint8_t* __restrict__ rc = a.ix.rcodes;
  const int8_t* sl = s_slices + gid * ss + 4 * t4;  // this lane's B column (slice gid)
  for (int cb = wid * 16; cb < ncand; cb += WARPS * 16) {
    const int i0 = cb + gid, i1 = cb + gid + 8;
    const int64_t r0 = lo + c0 + s_cv[min(i0, ncand - 1)];
    const int64_t r1 = lo + c0 + s_cv[min(i1, ncand - 1)];
    const uint8_t* row0 = rc + r0 * rb;
    const uint8_t* row1 = rc + r1 * rb;
    int c[4] = {0, 0, 0, 0};
    for (int p = 0; p < kp / 64; ++p) {
      uint32_t a0s0, a2s0, a0s1, a2s1, a1s0, a3s0, a1s1, a3s1;
      if (NIB) {
        const uint2 x0 = __ldg(reinterpret_cast<const uint2*>(row0 + 8 * (4 * p + t4)));
        const uint2 x1 = __ldg(reinterpret_cast<const uint2*>(row1 + 8 * (4 * p + t4)));
        a0s0 = x0.x & 0x0F0F0F0Fu;
        a2s0 = (x0.x >> 4) & 0x0F0F0F0Fu;
        a0s1 = x0.y & 0x0F0F0F0Fu;
        a2s1 = (x0.y >> 4) & 0x0F0F0F0Fu;
        a1s0 = x1.x & 0x0F0F0F0Fu;
        a3s0 = (x1.x >> 4) & 0x0F0F0F0Fu;
        a1s1 = x1.y & 0x0F0F0F0Fu;
        a3s1 = (x1.y >> 4) & 0x0F0F0F0Fu;
      } else {
        const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(row0 + 16 * (4 * p + t4)));
        const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(row1 + 16 * (4 * p + t4)));
        a0s0 = x0.x;
        a2s0 = x0.y;
        a0s1 = x0.z;
        a2s1 = x0.w;
        a1s0 = x1.x;
        a3s0 = x1.y;
        a1s1 = x1.z;
        a3s1 = x1.w;
      }
      const int kb0 = 64 * p, kb1 = 64 * p + 32;
      const uint32_t b00 = *reinterpret_cast<const uint32_t*>(sl + kb0);
      const uint32_t b10 = *reinterpret_cast<const uint32_t*>(sl + kb0 + 16);
      const uint32_t b01 = *reinterpret_cast<const uint32_t*>(sl + kb1);
      const uint32_t b11 = *reinterpret_cast<const uint32_t*>(sl + kb1 + 16);
      mma_u8s8(c, a0s0, a1s0, a2s0, a3s0, b00, b10);
      mma_u8s8(c, a0s1, a1s1, a2s1, a3s1, b01, b11);
    }
    // c0,c1: row gid, slices 2t4, 2t4+1; c2,c3: row gid+8.  Slices 0-3 form
    // the high int64 half (weights 128^3..1), slices 4-7 the low half.
    const long long w0 = (t4 & 1) ? 128LL : 2097152LL;  // 128^3 or 128 (first slice of the pair)
    const long long w1 = (t4 & 1) ? 1LL : 16384LL;
    long long p0 = (long long)c[0] * w0 + (long long)c[1] * w1;
    long long p1 = (long long)c[2] * w0 + (long long)c[3] * w1;
    p0 += __shfl_xor_sync(FULL, p0, 1);
    p1 += __shfl_xor_sync(FULL, p1, 1);
    const long long q0 = __shfl_xor_sync(FULL, p0, 2);  // lane t4=0 receives the low half
    const long long q1 = __shfl_xor_sync(FULL, p1, 2);
    if (t4 == 0) {
      const double hi_s = ldexp(1.0, qc.sexp - 26), lo_s = ldexp(1.0, qc.sexp - 54);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int ci = h ? i1 : i0;
        if (ci >= ncand) continue;
        const long long hi = h ? p1 : p0, lw = h ? q1 : q0;
        const double ip = dadd(dmul((double)hi, hi_s), dmul((double)lw, lo_s));
        const float2 lf = __ldg(reinterpret_cast<const float2*>(a.ix.long_factors) + (h ? r1 : r0));
        s_cd[ci] = dmax(dsub(dadd((double)lf.x, d_qc2), dmul((double)lf.y, dsub(ip, qc.kb_sum))), 0.0);
      }
    }
  }
}

// ------------------------------------------------------------ warp top-32 queues
// (dist, id) queues in the 32 lanes of a warp.  `Less` orders two (dist, id) keys: key_less on
// pids for the exact passes, the row-entry order (EntryLess) for the approximate pass.
struct PidLess {
  __device__ __forceinline__ bool operator()(double da, int64_t ia, double db, int64_t ib) const {
    return key_less(da, ia, db, ib);
  }
};

template <class Less>
__device__ __forceinline__ void cmpx(double& d, int64_t& id, int stride, bool take_min, const Less& lt) {
  const double od = __shfl_xor_sync(FULL, d, stride);
  const int64_t oi = __shfl_xor_sync(FULL, id, stride);
  const bool other_less = lt(od, oi, d, id);
  if (take_min ? other_less : lt(d, id, od, oi)) {
    d = od;
    id = oi;
  }
}

template <class Less = PidLess>
__device__ __forceinline__ void warp_sort32(double& d, int64_t& id, const Less& lt = Less()) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const bool up = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      cmpx(d, id, stride, lower == up, lt);
    }
  }
}

// q (sorted ascending) := 32 smallest of q ∪ b (b sorted ascending), sorted.
template <class Less = PidLess>
__device__ __forceinline__ void warp_merge32(double& qd, int64_t& qi, double bd, int64_t bi, const Less& lt = Less()) {
  const int lane = threadIdx.x & 31;
  const double rd = __shfl_sync(FULL, bd, 31 - lane);
  const int64_t ri = __shfl_sync(FULL, bi, 31 - lane);
  if (lt(rd, ri, qd, qi)) {
    qd = rd;
    qi = ri;
  }
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) cmpx(qd, qi, stride, (lane & stride) == 0, lt);
}

// Fold this warp's candidates (d, id) where `pass` into the sorted queue.
// Few passers: insert one at a time (position by ballot, shift by shfl_up);
// many (a filling queue): sort the batch and merge.  An insertion past the
// k-th entry is skipped (the exact passes keep only the top k); the
// approximate pass folds with k = 32 to keep the 32 smallest.
template <class Less = PidLess>
__device__ __forceinline__ void warp_fold(double& qd, int64_t& qi, double d, int64_t id, bool pass, int k,
                                          const Less& lt = Less()) {
  const int lane = threadIdx.x & 31;
  unsigned m = __ballot_sync(FULL, pass);
  if (__popc(m) > 6) {
    if (!pass) {
      d = dinf();
      id = NO_ID;
    }
    warp_sort32(d, id, lt);
    warp_merge32(qd, qi, d, id, lt);
    return;
  }
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const double xd = __shfl_sync(FULL, d, src);
    const int64_t xi = __shfl_sync(FULL, id, src);
    const double kd = __shfl_sync(FULL, qd, k - 1);
    const int64_t ki = __shfl_sync(FULL, qi, k - 1);
    if (!lt(xd, xi, kd, ki)) continue;  // the queue moved on
    const int pos = __popc(__ballot_sync(FULL, lt(qd, qi, xd, xi)));
    const double ud = __shfl_up_sync(FULL, qd, 1);
    const int64_t ui = __shfl_up_sync(FULL, qi, 1);
    if (lane > pos) {
      qd = ud;
      qi = ui;
    } else if (lane == pos) {
      qd = xd;
      qi = xi;
    }
  }
}

// ------------------------------------------------------------ common prologue
struct Smem {
  int8_t* s_slices;
  uint32_t* s_planes8;
  float* s_lut;
  double* s_cd;
  int32_t* s_cv;
  double* s_pool_d;
  int64_t* s_pool_i;
  double* s_sortk;
  int64_t* s_sorti;
};

template <int MODE, bool REFINE>
__device__ __forceinline__ Smem carve(const Args& a, unsigned char* smem, bool bigk) {
  Smem s{};
  const int g = a.g;
  unsigned char* p = smem;
  s.s_cd = reinterpret_cast<double*>(p);
  p += sizeof(double) * CHUNK;
  s.s_pool_d = reinterpret_cast<double*>(p);
  p += sizeof(double) * (bigk ? a.k : 32);
  s.s_pool_i = reinterpret_cast<int64_t*>(p);
  p += sizeof(int64_t) * (bigk ? a.k : 32);
  s.s_sortk = reinterpret_cast<double*>(p);  // big k: sort buffer; small k: per-warp queues
  p += sizeof(double) * (bigk ? a.sort_n : WARPS * 32);
  s.s_sorti = reinterpret_cast<int64_t*>(p);
  p += sizeof(int64_t) * (bigk ? a.sort_n : WARPS * 32);
  s.s_cv = reinterpret_cast<int32_t*>(p);
  p += sizeof(int32_t) * CHUNK;
  s.s_planes8 = reinterpret_cast<uint32_t*>(p);
  p += MODE == IVRQ_IP_BITWISE ? sizeof(uint32_t) * 8 * g : 0;
  s.s_lut = reinterpret_cast<float*>(p);
  p += MODE == IVRQ_IP_LUT ? sizeof(float) * 8 * g * 16 : 0;
  s.s_slices = reinterpret_cast<int8_t*>(p);
  return s;
}

size_t smem_bytes(const Args& a, int mode, bool refine, bool bigk) {
  size_t b = 0;
  b += sizeof(double) * CHUNK;
  b += (sizeof(double) + sizeof(int64_t)) * (bigk ? a.k : 32);
  b += (sizeof(double) + sizeof(int64_t)) * (bigk ? a.sort_n : WARPS * 32);
  b += sizeof(int32_t) * CHUNK;
  b += mode == IVRQ_IP_BITWISE ? sizeof(uint32_t) * 8 * a.g : sizeof(float) * 8 * a.g * 16;
  b += refine ? (size_t)SLICES * (a.kpad + SPAD) : 0;
  return b + 16;
}

template <int MODE, bool REFINE>
__device__ __forceinline__ QueryCtx load_query(const Args& a, const Smem& s, int64_t q) {
  const int g = a.g, tid = threadIdx.x;
  if (REFINE) {
    const int kp = a.kpad, ss = kp + SPAD;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.qslices + q * SLICES * (int64_t)kp);
    for (int i = tid; i < SLICES * kp / 4; i += THREADS) {
      const int sidx = (4 * i) / kp, k = (4 * i) % kp;
      *reinterpret_cast<uint32_t*>(s.s_slices + sidx * ss + k) = src[i];
    }
  }
  if (MODE == IVRQ_IP_BITWISE) {
    for (int i = tid; i < 8 * g; i += THREADS) {
      const int gi = i / 8, j = i % 8;
      s.s_planes8[i] = j < a.qbits ? a.planes[(q * a.qbits + j) * g + gi] : 0u;
    }
  } else {
    for (int i = tid; i < 8 * g * 16; i += THREADS) s.s_lut[i] = a.luts[q * 8 * g * 16 + i];
  }
  const double* sc = a.scalars + q * IVRQ_QS_COUNT;
  QueryCtx qc;
  qc.delta = sc[IVRQ_QS_DELTA];
  qc.half_code = sc[IVRQ_QS_HALF_CODE];
  qc.ipm = sc[IVRQ_QS_IP_MARGIN];
  qc.kb_sum = sc[IVRQ_QS_KB_SUM];
  qc.sexp = REFINE ? (int)sc[IVRQ_QS_SLICE_EXP] : 0;
  return qc;
}

// ------------------------------------------------------------ kernel, k <= 32
template <int MODE, bool REFINE, bool NIB, int QB, int IPB>
__global__ void __launch_bounds__(THREADS, 4) scan_kernel(Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_ncand;
  __shared__ double s_T;
  __shared__ int s_pool_n;
  __shared__ long long s_probed, s_surv;
  // one query per CTA; as the exact rerun of listed queries (fix_only) a small grid strides the list
  const int64_t nslot = a.fix_only ? (int64_t)*a.fix_only_count : a.nq;
  for (int64_t slot = blockIdx.x; slot < nslot; slot += gridDim.x) {
  const int64_t q = a.fix_only ? (int64_t)a.fix_only[slot] : a.qorder ? a.qorder[slot] : slot;
  const int k = a.k;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const Smem s = carve<MODE, REFINE>(a, smem, false);
  const QueryCtx qc = load_query<MODE, REFINE>(a, s, q);
  const int init_n = a.init_counts ? a.init_counts[q] : 0;  // pool carried in from the previous shard
  if (tid < 32) {
    s.s_pool_d[tid] = tid < init_n ? a.init_dists[q * k + tid] : dinf();
    s.s_pool_i[tid] = tid < init_n ? a.init_ids[q * k + tid] : NO_ID;
  }
  if (tid == 0) {
    s_T = init_n >= k ? a.init_dists[q * k + k - 1] : dinf();
    s_pool_n = init_n;
    // after the first-list phase the first list's counts are already in stats
    s_probed = (a.skip_first && a.stats) ? a.stats[2 * q] : 0;
    s_surv = (a.skip_first && a.stats) ? a.stats[2 * q + 1] : 0;
  }
  __syncthreads();
  const int64_t* pid_list = a.probe_ids + q * a.nprobe;
  const double* pd2_list = a.probe_d2 + q * a.nprobe;
  bool first_pending = a.skip_first != 0;
  for (int p = 0; p < a.nprobe; ++p) {  // ascending cluster id (search.py:429)
    const int64_t cg = pid_list[p];
    if (cg < a.list_lo || cg >= a.list_hi) continue;  // another shard's list
    if (first_pending) {  // scanned by first_list_kernel
      first_pending = false;
      continue;
    }
    const int64_t c = cg - a.list_lo;
    const double d_qc2 = pd2_list[p];
    const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
    if (n_c == 0) continue;
    const double T_list = a.prune ? s_T : dinf();
    const bool pool_full = s_pool_n >= k;
    const double pk_d = pool_full ? s.s_pool_d[k - 1] : dinf();
    const int64_t pk_i = pool_full ? s.s_pool_i[k - 1] : NO_ID;
    const double sq = dsqrt(d_qc2);
    const uint32_t* words = a.ix.packed_msb + (int64_t)a.g * lo;
    const void* iprow = nullptr;
    if (IPB) {
      const int64_t slot = a.pslot[q * a.nprobe + p];
      iprow = reinterpret_cast<const char*>(a.ipbuf) + IPB * (a.pair_base[c] + slot * ip_row_stride(n_c));
    }
    double qd = dinf();  // this warp's top-32 queue (lane i = i-th smallest)
    int64_t qi = NO_ID;
    bool any_cand = false;
    for (int64_t c0 = 0; c0 < n_c; c0 += CHUNK) {
      const int cn = (int)min((int64_t)CHUNK, n_c - c0);
      if (tid == 0) s_ncand = 0;
      __syncthreads();
      stage1_chunk<MODE, QB, IPB>(a, qc, words, lo, n_c, c0, cn, d_qc2, sq, T_list, s.s_planes8, s.s_lut, s.s_cv,
                                  s.s_cd, &s_ncand, iprow);
      __syncthreads();
      const int ncand = s_ncand;
      if (tid == 0) {
        s_probed += cn;
        s_surv += ncand;
      }
      if (ncand == 0) continue;
      any_cand = true;
      if (REFINE) {
        refine_chunk<NIB>(a, qc, lo, c0, d_qc2, s.s_slices, s.s_cv, s.s_cd, ncand);
        __syncthreads();
      }
      // each warp folds its share of the candidates into its queue
      for (int cb = wid * 32; cb < ncand; cb += THREADS) {
        const int ci = cb + lane;
        const double d0 = ci < ncand ? s.s_cd[ci] : dinf();
        const double wk_d = __shfl_sync(FULL, qd, k - 1);
        const int64_t wk_i = __shfl_sync(FULL, qi, k - 1);
        // the pid is only needed when the distance can enter the queue
        const bool maybe = d0 <= wk_d && d0 <= pk_d && ci < ncand;
        if (!__any_sync(FULL, maybe)) continue;
        double d = d0;
        int64_t id = maybe ? (int64_t)__ldg(a.ix.pids + lo + c0 + s.s_cv[ci]) : NO_ID;
        const bool pass = maybe && key_less(d, id, wk_d, wk_i) && key_less(d, id, pk_d, pk_i);
        if (!__any_sync(FULL, pass)) continue;
        warp_fold(qd, qi, d, id, pass, k);
      }
    }
    if (!__syncthreads_or(any_cand)) continue;
    // fold the warp queues into the pool (warp 0), then move the threshold
    s.s_sortk[wid * 32 + lane] = qd;
    s.s_sorti[wid * 32 + lane] = qi;
    __syncthreads();
    if (wid == 0) {
      double pd = s.s_pool_d[lane];
      int64_t pi = s.s_pool_i[lane];
      for (int w = 0; w < WARPS; ++w) {
        if (s.s_sorti[w * 32] == NO_ID) continue;
        warp_merge32(pd, pi, s.s_sortk[w * 32 + lane], s.s_sorti[w * 32 + lane]);
      }
      s.s_pool_d[lane] = pd;
      s.s_pool_i[lane] = pi;
      const int cnt = __popc(__ballot_sync(FULL, lane < k && pi != NO_ID));
      const double kd = __shfl_sync(FULL, pd, k - 1);
      if (lane == 0) {
        s_pool_n = cnt;
        if (cnt >= k) s_T = kd;  // search.py:444-447
      }
    }
    __syncthreads();
  }
  const int pn = s_pool_n;
  for (int i = tid; i < k; i += THREADS) {
    a.out_ids[q * k + i] = i < pn ? s.s_pool_i[i] : -1;
    a.out_dists[q * k + i] = i < pn ? s.s_pool_d[i] : dinf();
  }
  if (tid == 0) {
    a.out_counts[q] = pn;
    if (a.stats) {
      a.stats[2 * q] = s_probed;
      a.stats[2 * q + 1] = s_surv;
    }
  }
  __syncthreads();  // the CTA's shared state is reused by the next slot
  }
}

// ------------------------------------------------------------ per-probe metadata
__global__ void probe_meta_kernel(Args a, int64_t* __restrict__ m_lo, int32_t* __restrict__ m_nc,
                                  int64_t* __restrict__ m_base) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.nq * a.nprobe) return;
  const int64_t cg = a.probe_ids[i];
  if (cg < a.list_lo || cg >= a.list_hi) {
    m_nc[i] = -1;
    m_lo[i] = 0;
    m_base[i] = 0;
    return;
  }
  const int64_t c = cg - a.list_lo;
  const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
  m_lo[i] = lo;
  m_nc[i] = (int32_t)n_c;
  m_base[i] = a.pslot ? a.pair_base[c] + (int64_t)a.pslot[i] * ip_row_stride(n_c) : 0;
}

struct ListMeta {
  int64_t lo, base;
  int32_t nc;
  double d2;
};

__device__ __forceinline__ ListMeta list_meta(const Args& a, int64_t qp) {
  ListMeta m;
  m.lo = __ldg(a.m_lo + qp);
  m.nc = __ldg(a.m_nc + qp);
  m.base = __ldg(a.m_base + qp);
  m.d2 = __ldg(a.probe_d2 + qp);
  return m;
}

// ------------------------------------------------------------ float32 stage-1 decision
// The prune test keeps a vector iff max(est2 - sqrt(S), 0) <= T (search.py:360-366 with the
// stage1_chunk shortcuts), est2 = max((add + d_qc2) - scale (delta ip - half_code), 0) and
// S = (err sqrt(d_qc2))^2 + (scale ip_margin)^2, all in float64.  Evaluated in float32, est2 is
// within E = 2^-19 M of the float64 value (M = |add| + d_qc2 + |scale| (|delta ip| + |half_code|):
// about ten float32 roundings of at most 2^-24 M each, input conversions included) and S within
// 2^-19 relative.  Outside those bands the float32 answer is the float64 one; inside (about 1e-5 of
// the vectors) the caller runs the float64 test.  Returns 1 keep, 0 prune, -1 undecided.
struct Stage1F32 {
  float delta, half, ahalf, dqc, sq, ipm, T_lo, T_hi;
};

__device__ __forceinline__ Stage1F32 stage1_f32(double delta, double half_code, double ipm, double d_qc2, double sq,
                                                double T) {
  Stage1F32 f;
  f.delta = (float)delta;
  f.half = (float)half_code;
  f.ahalf = fabsf(f.half);
  f.dqc = (float)d_qc2;
  f.sq = (float)sq;
  f.ipm = (float)ipm;
  f.T_lo = __double2float_rd(T);
  f.T_hi = __double2float_ru(T);
  return f;
}

__device__ __forceinline__ int stage1_decide_f32x(float t1, float add, float scale, float err, const Stage1F32& f,
                                                  float extra);

__device__ __forceinline__ int stage1_decide_f32(int ip, float add, float scale, float err, const Stage1F32& f) {
  return stage1_decide_f32x(f.delta * (float)ip, add, scale, err, f, 0.f);
}

// The same test from t1 = delta * ip given directly, with `extra` (>= 0) added to the inner product's
// error (the certified LUT estimate's bound, scan_rda_kernel<LUT>).
__device__ __forceinline__ int stage1_decide_f32x(float t1, float add, float scale, float err, const Stage1F32& f,
                                                  float extra) {
  const float e = (add + f.dqc) - scale * (t1 - f.half);
  const float M = fabsf(add) + f.dqc + fabsf(scale) * (fabsf(t1) + f.ahalf);
  const float E = M * 0x1p-19f + fabsf(scale) * extra;
  const float dk = (e + E) - f.T_lo;  // >= est2 - T
  if (dk <= 0.f) return 1;
  const float mg = err * f.sq, sm = scale * f.ipm;
  const float S = mg * mg + sm * sm;
  if (dk * dk < S * (1.f - 0x1p-19f)) return 1;
  const float dr = (e - E) - f.T_hi;  // <= est2 - T
  if (dr > 0.f && dr * dr > S * (1.f + 0x1p-19f)) return 0;
  return -1;
}

// ------------------------------------------------------------ warp-per-query kernel (precomputed inner products)
// With the stage-1 inner products already in HBM (ip_list_kernel) a query's
// remaining work is a light stream (2-byte ip + 8-byte factors per vector)
// plus the refine of its survivors, so one warp owns one query and nothing
// synchronises beyond the warp: survivors queue in a per-warp ring in shared
// memory, every 16 of them go through one m16n8k32 refine group, and the
// warp's register top-32 queue IS the query's pool.  Same prune test, refine
// arithmetic and (dist, id) order as scan_kernel, so results are identical.
constexpr int WQ = 2;      // queries (warps) per CTA
constexpr int WQ_MINB = 8;  // resident CTAs per SM the register budget is sized for (B200 A/B, scan ms:
                            // C2 2.93 vs 3.01 at 12, C4 8.6 vs 9.06, C5 16.6 vs 18.3)
constexpr int SUB = 4;     // 32-vector sub-chunks loaded together (memory-level parallelism)
constexpr int RING = 256;  // survivor ring per warp (holds < 32 + 32 * SUB)

size_t warp_smem_bytes(int kpad, bool refine) {
  const size_t per = (refine ? (size_t)SLICES * (kpad + SPAD) : 0) + RING * sizeof(int32_t);
  return WQ * ((per + 15) & ~size_t(15));
}

__device__ __forceinline__ void load_a_frag(const uint8_t* row0, const uint8_t* row1, int p, int t4, bool nib,
                                            uint32_t (&s0)[4], uint32_t (&s1)[4]) {
  if (nib) {
    const uint2 x0 = __ldg(reinterpret_cast<const uint2*>(row0 + 8 * (4 * p + t4)));
    const uint2 x1 = __ldg(reinterpret_cast<const uint2*>(row1 + 8 * (4 * p + t4)));
    s0[0] = x0.x & 0x0F0F0F0Fu;
    s0[2] = (x0.x >> 4) & 0x0F0F0F0Fu;
    s1[0] = x0.y & 0x0F0F0F0Fu;
    s1[2] = (x0.y >> 4) & 0x0F0F0F0Fu;
    s0[1] = x1.x & 0x0F0F0F0Fu;
    s0[3] = (x1.x >> 4) & 0x0F0F0F0Fu;
    s1[1] = x1.y & 0x0F0F0F0Fu;
    s1[3] = (x1.y >> 4) & 0x0F0F0F0Fu;
  } else {
    const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(row0 + 16 * (4 * p + t4)));
    const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(row1 + 16 * (4 * p + t4)));
    s0[0] = x0.x;
    s0[2] = x0.y;
    s1[0] = x0.z;
    s1[2] = x0.w;
    s0[1] = x1.x;
    s0[3] = x1.y;
    s1[1] = x1.z;
    s1[3] = x1.w;
  }
}

// Refined distances of up to 32 candidates: entries head..head+m-1 of the
// ring rv (mod RING), or rows head..head+m-1 directly when rv is null.  Two
// m16 tiles share the query's B fragments; lane L < m receives candidate L.
template <bool NIB>
__device__ __forceinline__ void warp_refine32(const Args& a, const QueryCtx& qc, int64_t lo, double d_qc2,
                                              const int8_t* sl_base, const int32_t* rv, int head, int m,
                                              double& dist, int& vrow) {
  const int lane = threadIdx.x & 31, gid = lane >> 2, t4 = lane & 3;
  const int kp = a.kpad;
  const int64_t rb = a.ix.rcode_bytes;
  int vr[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {  // rows gid, gid+8, gid+16, gid+24
    const int e = min(gid + 8 * t, m - 1);
    vr[t] = rv ? rv[(head + e) & (RING - 1)] : head + e;
  }
  const uint8_t* ra0 = a.ix.rcodes + (lo + vr[0]) * rb;
  const uint8_t* ra1 = a.ix.rcodes + (lo + vr[1]) * rb;
  const uint8_t* rb0 = a.ix.rcodes + (lo + vr[2]) * rb;
  const uint8_t* rb1 = a.ix.rcodes + (lo + vr[3]) * rb;
  const int8_t* sl = sl_base + gid * (kp + SPAD) + 4 * t4;
  const bool two = m > 16;  // warp-uniform
  int ca[4] = {0, 0, 0, 0}, cb[4] = {0, 0, 0, 0};
#pragma unroll 3
  for (int p = 0; p < kp / 64; ++p) {
    uint32_t as0[4], as1[4], bs0[4], bs1[4];
    load_a_frag(ra0, ra1, p, t4, NIB, as0, as1);
    if (two) load_a_frag(rb0, rb1, p, t4, NIB, bs0, bs1);
    const uint32_t b00 = *reinterpret_cast<const uint32_t*>(sl + 64 * p);
    const uint32_t b10 = *reinterpret_cast<const uint32_t*>(sl + 64 * p + 16);
    const uint32_t b01 = *reinterpret_cast<const uint32_t*>(sl + 64 * p + 32);
    const uint32_t b11 = *reinterpret_cast<const uint32_t*>(sl + 64 * p + 48);
    mma_u8s8(ca, as0[0], as0[1], as0[2], as0[3], b00, b10);
    if (two) mma_u8s8(cb, bs0[0], bs0[1], bs0[2], bs0[3], b00, b10);
    mma_u8s8(ca, as1[0], as1[1], as1[2], as1[3], b01, b11);
    if (two) mma_u8s8(cb, bs1[0], bs1[1], bs1[2], bs1[3], b01, b11);
  }
  const long long w0 = (t4 & 1) ? 128LL : 2097152LL;
  const long long w1 = (t4 & 1) ? 1LL : 16384LL;
  const int L = lane & 15, src = (L & 7) * 4;  // lane t4 == 0 of group (L & 7) holds the sums
  const bool hi8 = L >= 8, tb = lane >= 16;
  // one tile at a time (register pressure): lanes 0-15 take tile a's rows, 16-31 tile b's
  long long hsel = 0, lsel = 0;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int* cc = t ? cb : ca;
    long long p0 = (long long)cc[0] * w0 + (long long)cc[1] * w1;
    long long p1 = (long long)cc[2] * w0 + (long long)cc[3] * w1;
    p0 += __shfl_xor_sync(FULL, p0, 1);
    p1 += __shfl_xor_sync(FULL, p1, 1);
    const long long l0 = __shfl_xor_sync(FULL, p0, 2), l1 = __shfl_xor_sync(FULL, p1, 2);
    // the source lane supplies both row halves; the receiver picks
    const long long h0 = __shfl_sync(FULL, p0, src), h1 = __shfl_sync(FULL, p1, src);
    const long long g0 = __shfl_sync(FULL, l0, src), g1 = __shfl_sync(FULL, l1, src);
    if (tb == (t == 1)) {
      hsel = hi8 ? h1 : h0;
      lsel = hi8 ? g1 : g0;
    }
  }
  dist = dinf();
  vrow = -1;
  if (lane < m) {
    vrow = rv ? rv[(head + lane) & (RING - 1)] : head + lane;
    const long long hi = hsel, lw = lsel;
    const double hi_s = ldexp(1.0, qc.sexp - 26), lo_s = ldexp(1.0, qc.sexp - 54);
    const double ip = dadd(dmul((double)hi, hi_s), dmul((double)lw, lo_s));
    const float2 lf = __ldg(reinterpret_cast<const float2*>(a.ix.long_factors) + lo + vrow);
    dist = dmax(dsub(dadd((double)lf.x, d_qc2), dmul((double)lf.y, dsub(ip, qc.kb_sum))), 0.0);
  }
}

// offer (d, row) on each lane to the warp queue (pid loaded only when it can enter)
__device__ __forceinline__ void warp_offer(const Args& a, double& qd, int64_t& qi, double d, int vrow, int64_t lo,
                                           int k) {
  const double kd = __shfl_sync(FULL, qd, k - 1);
  const int64_t ki = __shfl_sync(FULL, qi, k - 1);
  const bool maybe = vrow >= 0 && d <= kd;
  if (!__any_sync(FULL, maybe)) return;
  const int64_t id = maybe ? (int64_t)__ldg(a.ix.pids + lo + vrow) : NO_ID;
  const bool pass = maybe && key_less(d, id, kd, ki);
  if (!__any_sync(FULL, pass)) return;
  warp_fold(qd, qi, d, id, pass, k);
}

template <bool REFINE, bool NIB, int IPB, int MINB>
__global__ void __launch_bounds__(WQ * 32, MINB) scan_warp_kernel(Args a) {
  using IPT = typename std::conditional<IPB == 2, int16_t, int32_t>::type;
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t slot_q = (int64_t)blockIdx.x * WQ + wid;
  if (slot_q >= a.nq) return;  // whole warps only: nothing below synchronises the block
  // as the exact rerun of queries the approximate pass listed: only slots < *fix_only_count
  if (a.fix_only && slot_q >= *a.fix_only_count) return;
  const int64_t q = a.fix_only ? (int64_t)a.fix_only[slot_q] : a.qorder ? a.qorder[slot_q] : slot_q;
  const int k = a.k, kp = a.kpad;
  const size_t per = ((REFINE ? (size_t)SLICES * (kp + SPAD) : 0) + RING * sizeof(int32_t) + 15) & ~size_t(15);
  unsigned char* wbase = smem + wid * per;
  int8_t* s_sl = reinterpret_cast<int8_t*>(wbase);
  int32_t* r_v = reinterpret_cast<int32_t*>(wbase + (REFINE ? (size_t)SLICES * (kp + SPAD) : 0));
  if (REFINE) {
    const uint32_t* src = reinterpret_cast<const uint32_t*>(a.qslices + q * SLICES * (int64_t)kp);
    for (int i = lane; i < SLICES * kp / 4; i += 32) {
      const int sidx = (4 * i) / kp, kk = (4 * i) % kp;
      *reinterpret_cast<uint32_t*>(s_sl + sidx * (kp + SPAD) + kk) = src[i];
    }
  }
  const double* sc = a.scalars + q * IVRQ_QS_COUNT;
  QueryCtx qc;
  qc.delta = sc[IVRQ_QS_DELTA];
  qc.half_code = sc[IVRQ_QS_HALF_CODE];
  qc.ipm = sc[IVRQ_QS_IP_MARGIN];
  qc.kb_sum = sc[IVRQ_QS_KB_SUM];
  qc.sexp = REFINE ? (int)sc[IVRQ_QS_SLICE_EXP] : 0;
  const int init_n = a.init_counts ? a.init_counts[q] : 0;
  double qd = lane < init_n ? a.init_dists[q * k + lane] : dinf();
  int64_t qi = lane < init_n ? a.init_ids[q * k + lane] : NO_ID;
  double T = init_n >= k ? __shfl_sync(FULL, qd, k - 1) : dinf();
  long long probed = (a.skip_first && a.stats) ? a.stats[2 * q] : 0;
  long long surv = (a.skip_first && a.stats) ? a.stats[2 * q + 1] : 0;
  __syncwarp();
  bool first_pending = true;  // the first in-range probe is still ahead
  ListMeta nxt = list_meta(a, q * a.nprobe);
  for (int p = 0; p < a.nprobe; ++p) {  // ascending cluster id (search.py:429)
    const ListMeta cur = nxt;
    if (p + 1 < a.nprobe) nxt = list_meta(a, q * a.nprobe + p + 1);  // prefetched one list ahead
    if (cur.nc < 0) continue;  // another shard's list
    const bool is_first = first_pending;
    first_pending = false;
    const int64_t c = a.probe_ids[q * a.nprobe + p] - a.list_lo;
    const double d_qc2 = cur.d2;
    const int64_t lo = cur.lo, n_c = cur.nc;
    if (n_c == 0) continue;
    const double T_list = a.prune ? T : dinf();
    probed += n_c;
    if (REFINE && T_list == dinf()) {  // nothing can be pruned (lb2 <= +inf): refine the whole list
      surv += n_c;
      if (a.fdist && is_first) {  // the query's first list: refined on the tensor cores list-major
        const double* frow = a.fdist + a.fbase[c] + (slot_q - a.qoff[c]) * ip_row_stride(n_c);
        for (int64_t c0 = 0; c0 < n_c; c0 += 32) {
          const int64_t vi = c0 + lane;
          warp_offer(a, qd, qi, vi < n_c ? __ldg(frow + vi) : dinf(), vi < n_c ? (int)vi : -1, lo, k);
        }
        const int cnt = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
        if (cnt >= k) T = __shfl_sync(FULL, qd, k - 1);
        continue;
      }
      for (int64_t c0 = 0; c0 < n_c; c0 += 32) {
        double d;
        int vr;
        warp_refine32<NIB>(a, qc, lo, d_qc2, s_sl, nullptr, (int)c0, (int)min((int64_t)32, n_c - c0), d, vr);
        warp_offer(a, qd, qi, d, vr, lo, k);
      }
      const int cnt = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
      if (cnt >= k) T = __shfl_sync(FULL, qd, k - 1);
      continue;
    }
    const double sq = dsqrt(d_qc2);
    const IPT* iprow = reinterpret_cast<const IPT*>(a.ipbuf) + cur.base;
    int head = 0, nb = 0;  // ring of pending survivors (warp-uniform)
    for (int64_t c0 = 0; c0 < n_c; c0 += 32 * SUB) {
      // loads of SUB sub-chunks first (ip, add, scale, err), then the tests
      int ipv[SUB];
      float fa[SUB], fs[SUB], fe[SUB];
#pragma unroll
      for (int u = 0; u < SUB; ++u) {
        const int64_t vi = c0 + u * 32 + lane;
        const bool in = vi < n_c;
        ipv[u] = in ? (int)__ldg(iprow + vi) : 0;
        fa[u] = in ? __ldg(a.ix.short_add + lo + vi) : 0.f;
        fs[u] = in ? __ldg(a.ix.short_scale + lo + vi) : 0.f;
        fe[u] = in ? __ldg(a.ix.short_err + lo + vi) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < SUB; ++u) {
        const int64_t vi = c0 + u * 32 + lane;
        if (c0 + u * 32 >= n_c) break;  // warp-uniform
        bool keep = false;
        double est2 = 0.0;
        // (the float32 pre-decision of scan_rd_kernel measured no faster here: this kernel is
        // latency-bound on its survivor refine, not on the float64 test)
        if (vi < n_c) {
          const double ipb = dmul(qc.delta, (double)ipv[u]);
          const double add = (double)fa[u];
          const double scale = (double)fs[u];
          const double ip_signed = dsub(ipb, qc.half_code);
          est2 = dmax(dsub(dadd(add, d_qc2), dmul(scale, ip_signed)), 0.0);
          if (est2 <= T_list) {
            keep = true;  // lb2 <= est2 <= T
          } else {
            double margin = dmul((double)fe[u], sq);
            if (qc.ipm != 0.0) {
              // same decision as stage1_chunk: squares when unambiguous, else the reference expression
              const double sm = dmul(scale, qc.ipm);
              const double S = dadd(dmul(margin, margin), dmul(sm, sm));
              const double gap = dsub(est2, T_list);
              const double g2 = dmul(gap, gap);
              if (S >= g2 * (1.0 + 0x1p-38)) {
                keep = true;
              } else if (S <= g2 * (1.0 - 0x1p-38) && gap > T_list * 0x1p-12) {
                keep = false;
              } else {
                keep = dmax(dsub(est2, dsqrt(S)), 0.0) <= T_list;
              }
            } else {
              keep = dmax(dsub(est2, margin), 0.0) <= T_list;
            }
          }
        }
        const unsigned kb = __ballot_sync(FULL, keep);
        if (!kb) continue;
        surv += __popc(kb);
        if (!REFINE) {  // 1-bit index: the stage-1 estimate is the distance (search.py:362-366)
          warp_offer(a, qd, qi, keep ? est2 : dinf(), keep ? (int)vi : -1, lo, k);
          continue;
        }
        if (keep) {
          r_v[(head + nb + __popc(kb & ((1u << lane) - 1u))) & (RING - 1)] = (int)vi;
          if (a.l2_prefetch) {  // the survivor's rcode row is read by a refine group a few batches later
            const uint8_t* row = a.ix.rcodes + (lo + vi) * a.ix.rcode_bytes;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(row), "r"((unsigned)a.ix.rcode_bytes));
          }
        }
        nb += __popc(kb);
      }
      if (REFINE) {
        __syncwarp();
        while (nb >= 32) {
          double d;
          int vr;
          warp_refine32<NIB>(a, qc, lo, d_qc2, s_sl, r_v, head, 32, d, vr);
          warp_offer(a, qd, qi, d, vr, lo, k);
          head = (head + 32) & (RING - 1);
          nb -= 32;
        }
        __syncwarp();  // consumed ring slots may be rewritten
      }
    }
    if (REFINE && nb > 0) {
      double d;
      int vr;
      warp_refine32<NIB>(a, qc, lo, d_qc2, s_sl, r_v, head, nb, d, vr);
      warp_offer(a, qd, qi, d, vr, lo, k);
    }
    __syncwarp();
    const int cnt = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
    if (cnt >= k) T = __shfl_sync(FULL, qd, k - 1);  // search.py:444-447
  }
  const int pn = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
  if (lane < k) {
    a.out_ids[q * k + lane] = lane < pn ? qi : -1;
    a.out_dists[q * k + lane] = lane < pn ? qd : dinf();
  }
  if (lane == 0) {
    a.out_counts[q] = pn;
    if (a.stats) {
      a.stats[2 * q] = probed;
      a.stats[2 * q + 1] = surv;
    }
  }
}

// ------------------------------------------------------------ per-query passes over precomputed stage-1 inputs
// With the stage-1 inner products of every probed (pair, vector) in ipbuf
// (tc_ip_kernel / ip_list_kernel), a query's pass is a stream: per list in
// ascending id, the stage-1 estimate and prune (same test as stage1_chunk),
// then its survivors offered to the warp's register queue (the pool).
constexpr int RDW = 4;    // queries (warps) per CTA

// The float64 prune test lb2 <= T of stage1_chunk for one vector (est2 already computed).
__device__ __forceinline__ bool stage1_keep64(double est2, double err, double scale, double sq, double ipm, double T) {
  if (est2 <= T) return true;  // lb2 <= est2 <= T
  const double margin = dmul(err, sq);
  if (ipm != 0.0) {  // same decision as stage1_chunk
    const double sm = dmul(scale, ipm);
    const double S = dadd(dmul(margin, margin), dmul(sm, sm));
    const double gap = dsub(est2, T);
    const double g2 = dmul(gap, gap);
    if (S >= g2 * (1.0 + 0x1p-38)) return true;
    if (S <= g2 * (1.0 - 0x1p-38) && gap > T * 0x1p-12) return false;
    return dmax(dsub(est2, dsqrt(S)), 0.0) <= T;
  }
  return dmax(dsub(est2, margin), 0.0) <= T;
}

// 1-bit indexes: the stage-1 estimate is the distance (search.py:362-366); no refine.
template <int IPB, int RSUB, int MINB = 1>
__global__ void __launch_bounds__(RDW * 32, MINB) scan_rd_kernel(Args a) {
  using IPT = typename std::conditional<IPB == 2, int16_t, int32_t>::type;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t slot_q = (int64_t)blockIdx.x * RDW + wid;
  if (slot_q >= a.nq) return;  // whole warps only
  const int64_t q = a.qorder ? a.qorder[slot_q] : slot_q;
  const int k = a.k;
  const double* sc = a.scalars + q * IVRQ_QS_COUNT;
  const double delta = sc[IVRQ_QS_DELTA], half_code = sc[IVRQ_QS_HALF_CODE], ipm = sc[IVRQ_QS_IP_MARGIN];
  const int init_n = a.init_counts ? a.init_counts[q] : 0;
  double qd = lane < init_n ? a.init_dists[q * k + lane] : dinf();
  int64_t qi = lane < init_n ? a.init_ids[q * k + lane] : NO_ID;
  double T = init_n >= k ? __shfl_sync(FULL, qd, k - 1) : dinf();
  long long probed = 0, surv = 0;
  ListMeta nxt = list_meta(a, q * a.nprobe);
  for (int p = 0; p < a.nprobe; ++p) {  // ascending cluster id (search.py:429)
    const ListMeta cur = nxt;
    if (p + 1 < a.nprobe) nxt = list_meta(a, q * a.nprobe + p + 1);  // prefetched one list ahead
    if (cur.nc <= 0) continue;  // another shard's list, or empty
    const int64_t lo = cur.lo, n_c = cur.nc;
    const double d_qc2 = cur.d2;
    const double T_list = a.prune ? T : dinf();
    probed += n_c;
    const IPT* iprow = reinterpret_cast<const IPT*>(a.ipbuf) + cur.base;
    const double sq = dsqrt(d_qc2);
    for (int64_t c0 = 0; c0 < n_c; c0 += 32 * RSUB) {
      int ipv[RSUB];
      float fa[RSUB], fs[RSUB], fe[RSUB];
#pragma unroll
      for (int u = 0; u < RSUB; ++u) {
        const int64_t vi = c0 + u * 32 + lane;
        const bool in = vi < n_c;
        ipv[u] = in ? (int)__ldg(iprow + vi) : 0;
        fa[u] = in ? __ldg(a.ix.short_add + lo + vi) : 0.f;
        fs[u] = in ? __ldg(a.ix.short_scale + lo + vi) : 0.f;
        fe[u] = in ? __ldg(a.ix.short_err + lo + vi) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < RSUB; ++u) {
        const int64_t vi = c0 + u * 32 + lane;
        if (c0 + u * 32 >= n_c) break;  // warp-uniform
        bool keep = false;
        double est2 = 0.0;
        if (vi < n_c) {
          const double scale = (double)fs[u];
          est2 = dmax(dsub(dadd((double)fa[u], d_qc2), dmul(scale, dsub(dmul(delta, (double)ipv[u]), half_code))), 0.0);
          keep = stage1_keep64(est2, (double)fe[u], scale, sq, ipm, T_list);
        }
        const unsigned kb = __ballot_sync(FULL, keep);
        if (!kb) continue;
        surv += __popc(kb);
        warp_offer(a, qd, qi, keep ? est2 : dinf(), keep ? (int)vi : -1, lo, k);
      }
    }
    const int cnt = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
    if (cnt >= k) T = __shfl_sync(FULL, qd, k - 1);  // search.py:444-447
  }
  const int pn = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
  if (lane < k) {
    a.out_ids[q * k + lane] = lane < pn ? qi : -1;
    a.out_dists[q * k + lane] = lane < pn ? qd : dinf();
  }
  if (lane == 0) {
    a.out_counts[q] = pn;
    if (a.stats) {
      a.stats[2 * q] = probed;
      a.stats[2 * q + 1] = surv;
    }
  }
}

// ------------------------------------------------------------ approximate refined distances, certified
// The refine pass over tc_refine_kernel's approximate distances.  Every stored
// value s is within rad(s) = rrad[q] + s 2^-23 of the exact refined distance x
// (refine_chunk's value).  The pass replays the reference's threshold chain
// with intervals and obtains exact values only where an interval leaves a
// decision open:
//  * the queue keeps every candidate that could still be among the k nearest
//    (s - rad(s) <= s_k + rad(s_k), s_k the queue's k-th value), the 32
//    smallest by value, so the k-th order statistic of the queue is within
//    rad(s_k) of the exact threshold T (both are 1-Lipschitz);
//  * a prune test lb2 <= T is decided by lb2 <= s_k - rad(s_k) (keep) or
//    lb2 > s_k + rad(s_k) (prune); otherwise the list-start queue (kept in
//    shared memory) gets exact values for its possible members and T is exact
//    for the rest of the list;
//  * at the end the possible members of the top k get exact values and the
//    queue is re-sorted, so ids, order and distances are the exact pass's.
// A queue entry is a shard row (bits 0-39) with its probe index (40-59) for the
// list's d_qc2, EXACT once its value is exact, or a carried-in pool's pid
// (PIDE).  Should the 32 slots ever fill with possible members (near-ties
// across > 32 - k vectors), the query is listed for an exact rerun
// (scan_warp_kernel with fix_only).
constexpr int64_t E_ROW = (1LL << 40) - 1;
constexpr int E_PSH = 40;
constexpr int64_t E_EXACT = 1LL << 60;
constexpr int64_t E_PIDE = 1LL << 61;  // pid entry (carried-in pool), always exact

__device__ __forceinline__ int64_t entry_pid(const int64_t* pids, int64_t e) {
  return e == NO_ID ? NO_ID : (e & E_PIDE) ? (e & E_ROW) : pids[e & E_ROW];
}

// tie of two values: the pids decide (rare; kept out of line so the sort networks stay small)
__device__ __noinline__ bool entry_tie_less(const int64_t* pids, int64_t ea, int64_t eb) {
  return entry_pid(pids, ea) < entry_pid(pids, eb);
}

struct EntryLess {  // (value, pid) order of queue entries
  const int64_t* pids;
  __device__ __forceinline__ int64_t pid(int64_t e) const { return entry_pid(pids, e); }
  __device__ __forceinline__ bool operator()(double da, int64_t ea, double db, int64_t eb) const {
    return da < db || (da == db && ea != eb && entry_tie_less(pids, ea, eb));
  }
};

__device__ __forceinline__ double entry_rad(double d, int64_t e, double rq) {
  return (e == NO_ID || (e & (E_EXACT | E_PIDE))) ? 0.0 : rq + d * 0x1p-23;
}

// P <-> K position of the query digit slices (bits 2-3 and 4-5 swapped; see tc_bpairs_kernel)
__device__ __forceinline__ int slice_pos(int P) { return (P & ~0x3C) | ((P & 0x0C) << 2) | ((P & 0x30) >> 2); }

// What the exact refine of a queue entry needs (kept in local memory by the out-of-line helpers
// below, which run a few times per query: the hot loop stays small enough for the instruction cache)
struct ExactCtx {
  const uint8_t* rcodes;
  const float2* lf;
  const double* pd2;     // this query's probe distances
  const int8_t* qs;      // this query's digit slices
  int64_t rb;
  int kp, sexp;
  double kb, rq;
  bool nib;
};

// The query's digits as per-position (high, low) halves in shared memory: position P of an rcode
// row pairs with hl[P] = (sum_{s<4} D_s 128^(3-s), sum_{s>=4} D_s 128^(7-s)) at slice index slice_pos(P).
__device__ __noinline__ void load_hl(const ExactCtx& c, int2* hl) {
  const int kp = c.kp, lane = threadIdx.x & 31;
  // four consecutive slice positions per lane and load: the eight digit words are independent loads
  for (int k0 = 4 * lane; k0 < kp; k0 += 128) {
    uint32_t w[SLICES];
#pragma unroll
    for (int s2 = 0; s2 < SLICES; ++s2) w[s2] = __ldg(reinterpret_cast<const uint32_t*>(c.qs + s2 * kp + k0));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int h = 0, l = 0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        h = h * 128 + (int)(int8_t)(w[s2] >> (8 * j));
        l = l * 128 + (int)(int8_t)(w[s2 + 4] >> (8 * j));
      }
      hl[slice_pos(k0 + j)] = make_int2(h, l);
    }
  }
  __syncwarp();
}

// Exact refined distance of queue entry e (refine_chunk's arithmetic), warp-collective.
__device__ __forceinline__ double exact_value(const ExactCtx& c, const int2* hl, int64_t e) {
  const int lane = threadIdx.x & 31, kp = c.kp;
  const int64_t row = e & E_ROW;
  const int p = (int)((e >> E_PSH) & 0xFFFFF);
  const uint8_t* rc = c.rcodes + row * c.rb;
  long long H = 0, L = 0;
  // lane-strided positions (coalesced row bytes), eight loads in flight
#pragma unroll 8
  for (int P = lane; P < kp; P += 32) {
    int u;
    if (c.nib) {
      const uint8_t by = __ldg(rc + (P >> 4) * 8 + ((P >> 3) & 1) * 4 + (P & 3));
      u = ((P >> 2) & 1) ? (by >> 4) : (by & 15);
    } else {
      u = __ldg(rc + P);
    }
    const int2 w = hl[P];
    H += (long long)u * w.x;
    L += (long long)u * w.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    H += __shfl_xor_sync(FULL, H, o);
    L += __shfl_xor_sync(FULL, L, o);
  }
  const double ip = dadd(dmul((double)H, ldexp(1.0, c.sexp - 26)), dmul((double)L, ldexp(1.0, c.sexp - 54)));
  const float2 lf = __ldg(c.lf + row);
  return dmax(dsub(dadd((double)lf.x, __ldg(c.pd2 + p)), dmul((double)lf.y, dsub(ip, c.kb))), 0.0);
}

// Exact values for the queue's possible members of the top k (value - rad <= s_k + rad(s_k)),
// then the queue re-sorted: its first k entries are then the exact top k, exact.
__device__ __noinline__ void exactify_top(const ExactCtx& c, const int2* hl, const int64_t* pids, double& qd,
                                          int64_t& qi, int k) {
  const double kd = __shfl_sync(FULL, qd, k - 1);
  const int64_t ke = __shfl_sync(FULL, qi, k - 1);
  const double lim = kd + entry_rad(kd, ke, c.rq);
  const bool need = qi != NO_ID && !(qi & (E_EXACT | E_PIDE)) && dsub(qd, entry_rad(qd, qi, c.rq)) <= lim;
  unsigned m = __ballot_sync(FULL, need);
  if (!m) return;
  while (m) {
    const int src = __ffs(m) - 1;
    m &= m - 1;
    const int64_t e = __shfl_sync(FULL, qi, src);
    const double x = exact_value(c, hl, e);
    if ((threadIdx.x & 31) == src) {
      qd = x;
      qi = e | E_EXACT;
    }
  }
  warp_sort32(qd, qi, EntryLess{pids});
}

// The float64 prune test (stage1_keep64) against an interval [T_lo, T_hi] of the threshold: 1 keep
// for every T in it, 0 prune for every T in it, -1 open.
__device__ __noinline__ int decide64(int ipv, float fa, float fs, float fe, double d_qc2, const double* sc,
                                     double T_lo, double T_hi) {
  const double delta = sc[IVRQ_QS_DELTA], half_code = sc[IVRQ_QS_HALF_CODE], ipm = sc[IVRQ_QS_IP_MARGIN];
  const double sq = dsqrt(d_qc2);
  const double scale = (double)fs;
  const double est2 = dmax(dsub(dadd((double)fa, d_qc2), dmul(scale, dsub(dmul(delta, (double)ipv), half_code))), 0.0);
  if (stage1_keep64(est2, (double)fe, scale, sq, ipm, T_lo)) return 1;
  if (!stage1_keep64(est2, (double)fe, scale, sq, ipm, T_hi)) return 0;
  return -1;
}

// LUT mode: the exact stage-1 inner product (the reference's table sum, scan_kernel's order) of row
// vi of a list, then the float64 test against [T_lo, T_hi] as decide64.  Out of line: it runs only where
// the certified estimate leaves the float32 test open.
__device__ __noinline__ int decide64_lut(const uint32_t* words, int64_t n_c, int64_t vi, int g, const float* lut,
                                         float fa, float fs, float fe, double d_qc2, const double* sc, double T_lo,
                                         double T_hi) {
  double acc = 0.0;
  for (int gi = 0; gi < g; ++gi) {
    const uint32_t w = __ldg(words + (int64_t)gi * n_c + vi);
    const float* lrow = lut + gi * 8 * 16;
#pragma unroll
    for (int s2 = 0; s2 < 8; ++s2) acc = dadd(acc, (double)lrow[s2 * 16 + ((w >> (4 * s2)) & 15u)]);
  }
  const double half_code = sc[IVRQ_QS_HALF_CODE], ipm = sc[IVRQ_QS_IP_MARGIN];
  const double sq = dsqrt(d_qc2), scale = (double)fs;
  const double est2 = dmax(dsub(dadd((double)fa, d_qc2), dmul(scale, dsub(acc, half_code))), 0.0);
  if (stage1_keep64(est2, (double)fe, scale, sq, ipm, T_lo)) return 1;
  if (!stage1_keep64(est2, (double)fe, scale, sq, ipm, T_hi)) return 0;
  return -1;
}

// The exact threshold of a list: exact values for the list-start queue's possible members
// (snap_d / snap_e, shared memory), its k-th value after the re-sort.  Warp-collective, out of line.
__device__ __noinline__ double resolve_threshold(const uint8_t* rcodes, const float* lfac, const double* pd2,
                                                 const int8_t* qs, const int64_t* pids, int64_t rb, int kp, int sexp,
                                                 double kb, double rq, bool nib, int2* hl, double* snap_d,
                                                 int64_t* snap_e, int k) {
  ExactCtx ec;
  ec.rcodes = rcodes;
  ec.lf = reinterpret_cast<const float2*>(lfac);
  ec.pd2 = pd2;
  ec.qs = qs;
  ec.rb = rb;
  ec.kp = kp;
  ec.sexp = sexp;
  ec.kb = kb;
  ec.rq = rq;
  ec.nib = nib;
  load_hl(ec, hl);
  const int lane = threadIdx.x & 31;
  double sd = snap_d[lane];
  int64_t se = snap_e[lane];
  exactify_top(ec, hl, pids, sd, se, k);
  snap_d[lane] = sd;  // the list-start queue, now exact where it matters (a second open test reuses it)
  snap_e[lane] = se;
  __syncwarp();
  return __shfl_sync(FULL, sd, k - 1);
}

#ifdef IVRQ_RDA_STATS  // development builds only: how often the intervals leave decisions open
__device__ unsigned long long g_rda_stats[6];  // prune resolutions, exact values, queries, sum rq/T (1e-12), reruns
#define RDA_STAT(i, v) (((threadIdx.x & 31) == 0) ? (void)atomicAdd(&g_rda_stats[i], (unsigned long long)(v)) : (void)0)
#else
#define RDA_STAT(i, v) ((void)0)
#endif

template <int IPB, int RSUB, int MINB = 1>
__global__ void __launch_bounds__(RDW * 32, MINB) scan_rda_kernel(Args a) {
  // IPB 2 / 4: exact integer stage-1 inner products in ipbuf (int16 / int32) beside float32 distances;
  // 1 / 0: (distance, stage-1 value) float pairs from the fused refine, the value an exact integer (1)
  // or the certified LUT estimate (0), with the short factors packed as float4
  constexpr bool LUT = IPB == 0;
  constexpr bool PK = IPB < 2;
  using IPT = typename std::conditional<IPB == 2, int16_t, int32_t>::type;
  extern __shared__ __align__(16) unsigned char rda_smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int it = 0;; ++it) {  // persistent warps: one query slot per iteration
  int64_t slot_q;
  if (a.rda_next) {  // the next slot from a counter (no tail of partial waves, uneven queries balance)
    int v = 0;
    if (lane == 0) v = atomicAdd(a.rda_next, 1);
    slot_q = __shfl_sync(FULL, v, 0);
  } else {
    if (it) return;
    slot_q = (int64_t)blockIdx.x * RDW + wid;
  }
  if (slot_q >= a.nq) return;  // whole warps only
  const int64_t q = a.qorder ? a.qorder[slot_q] : slot_q;
  const int k = a.k, kp = a.kpad;
  unsigned char* wbase = rda_smem + (size_t)wid * ((size_t)kp * sizeof(int2) + 32 * 16);
  int2* hl = reinterpret_cast<int2*>(wbase);
  double* snap_d = reinterpret_cast<double*>(wbase + (size_t)kp * sizeof(int2));
  int64_t* snap_e = reinterpret_cast<int64_t*>(snap_d + 32);
  // The queue is ordered by (value, entry bits): the order of tied approximate values never decides
  // anything (the threshold is a value; a tie at the 32nd slot is a saturation); the exact top k is
  // re-sorted by (value, pid) in exactify_top.
  const PidLess lt;
  const double* sc = a.scalars + q * IVRQ_QS_COUNT;
  const double rq = a.rrad[q];
  // LUT: |estimate - table sum| <= eq + |estimate| 2^-23: the tables' float32 rounding (2^-24 sum|q|),
  // their float64 sums, and the neglected query digits (kpad 135274560 2^(e-54)); float, rounded up
  float eq = 0.f;
  if (LUT)
    eq = __double2float_ru((sc[IVRQ_QS_L1] * (0x1p-24 + 0x1p-44) +
                            (double)kp * ldexp(135274560.0, (int)sc[IVRQ_QS_SLICE_EXP] - 54)) * (1.0 + 0x1p-20));
  const int init_n = a.init_counts ? a.init_counts[q] : 0;
  double qd = lane < init_n ? a.init_dists[q * k + lane] : dinf();
  int64_t qi = lane < init_n ? (a.init_ids[q * k + lane] | E_PIDE) : NO_ID;
  bool unsafe = false;
  int probed = 0, surv = 0;
  // Offer survivors (float32 value d, entry e; e = NO_ID: none) to the queue.  A new entry is a
  // possible member iff d - rad(d) <= s_k + rad(s_k), i.e. d <= (s_k + rad(s_k) + rq) / (1 - 2^-23):
  // that bound is kept as a float rounded up (a looser filter only lets more candidates into the
  // fold) and recomputed when the queue changes.
  auto member_bound = [&]() {
    const double kd = __shfl_sync(FULL, qd, k - 1);
    const int64_t ke = __shfl_sync(FULL, qi, k - 1);
    return kd == dinf() ? __int_as_float(0x7f800000)
                        : __double2float_ru((kd + entry_rad(kd, ke, rq) + rq) * (1.0 + 0x1p-22));
  };
  float lim = member_bound();
  auto offer = [&](float d, int64_t e) {
    const bool maybe = e != NO_ID && d <= lim;
    if (!__any_sync(FULL, maybe)) return;
    warp_fold(qd, qi, maybe ? (double)d : dinf(), maybe ? e : NO_ID, maybe, 32, lt);
    lim = member_bound();
  };
  // The 32nd slot a possible member: a candidate pushed out of the queue may have been one.  Checked
  // once per list: pushed-out values are >= the final 32nd value, s - rad(s) increases with s and
  // the k-th value only decreases, so a 32nd slot that is not a possible member now never was.
  auto check_saturation = [&]() {
    const double nk = __shfl_sync(FULL, qd, k - 1);
    const int64_t nke = __shfl_sync(FULL, qi, k - 1);
    const double d31 = __shfl_sync(FULL, qd, 31);
    const int64_t e31 = __shfl_sync(FULL, qi, 31);
    if (e31 != NO_ID && dsub(d31, entry_rad(d31, e31, rq)) <= nk + entry_rad(nk, nke, rq)) unsafe = true;
  };
  ListMeta nxt = list_meta(a, q * a.nprobe);
  for (int p = 0; p < a.nprobe; ++p) {  // ascending cluster id (search.py:429)
    const ListMeta cur = nxt;
    if (p + 1 < a.nprobe) nxt = list_meta(a, q * a.nprobe + p + 1);  // prefetched one list ahead
    if (cur.nc <= 0) continue;  // another shard's list, or empty
    const int64_t lo = cur.lo, n_c = cur.nc;
    const double d_qc2 = cur.d2;
    // the threshold before this list (search.py:444-447) as an interval: the queue's k-th value
    // and its radius (the threshold state lives in the queue, not in registers across lists)
    double T_list = dinf(), rT = 0.0;
    if (a.prune && __popc(__ballot_sync(FULL, lane < k && qi != NO_ID)) >= k) {
      T_list = __shfl_sync(FULL, qd, k - 1);
      rT = entry_rad(T_list, __shfl_sync(FULL, qi, k - 1), rq);
    }
    probed += (int)n_c;
    const float* rrow = a.rdist + (PK ? 2 : 1) * cur.base;
    if (T_list == dinf()) {  // nothing can be pruned (lb2 <= +inf): every vector's refined distance
      surv += (int)n_c;
      for (int64_t c0 = 0; c0 < n_c; c0 += 32 * RSUB) {
        float dv[RSUB];
#pragma unroll
        for (int u = 0; u < RSUB; ++u) {
          const int64_t vi = c0 + u * 32 + lane;
          dv[u] = vi < n_c ? __ldg(rrow + (PK ? 2 : 1) * vi) : 0.f;
        }
#pragma unroll 1
        for (int u = 0; u < RSUB; ++u) {  // one copy of the queue code (instruction cache); the values
          const float d0 = dv[0];         // rotate through dv[0] so every index stays static (registers)
#pragma unroll
          for (int j = 0; j + 1 < RSUB; ++j) dv[j] = dv[j + 1];
          const int64_t vi = c0 + u * 32 + lane;
          if (c0 + u * 32 >= n_c) break;  // warp-uniform
          offer(d0, vi < n_c ? ((lo + vi) | ((int64_t)p << E_PSH)) : NO_ID);
        }
      }
    } else {
      // the list-start queue, for an exact threshold should an interval leave a test open
      snap_d[lane] = qd;
      snap_e[lane] = qi;
      __syncwarp();
      const IPT* iprow = PK ? nullptr : reinterpret_cast<const IPT*>(a.ipbuf) + cur.base;
      Stage1F32 f32 = stage1_f32(sc[IVRQ_QS_DELTA], sc[IVRQ_QS_HALF_CODE], sc[IVRQ_QS_IP_MARGIN], d_qc2, dsqrt(d_qc2),
                                 T_list);
      f32.T_lo = __double2float_rd(T_list - rT * (1.0 + 0x1p-40));
      f32.T_hi = __double2float_ru(T_list + rT * (1.0 + 0x1p-40));
      for (int64_t c0 = 0; c0 < n_c; c0 += 32 * RSUB) {
        int ipv[RSUB];
        float fa[RSUB], fs[RSUB], fe[RSUB], pre[RSUB];
#pragma unroll
        for (int u = 0; u < RSUB; ++u) {
          const int64_t vi = c0 + u * 32 + lane;
          const bool in = vi < n_c;
          if (PK) {
            const float2 r = in ? __ldg(reinterpret_cast<const float2*>(rrow) + vi) : make_float2(0.f, 0.f);
            pre[u] = r.x;
            ipv[u] = LUT ? __float_as_int(r.y) : (int)r.y;
            const float4 f = in ? __ldg(a.sf4 + lo + vi) : make_float4(0.f, 0.f, 0.f, 0.f);
            fa[u] = f.x;
            fs[u] = f.y;
            fe[u] = f.z;
          } else {
            pre[u] = in ? __ldg(rrow + vi) : 0.f;
            ipv[u] = in ? (int)__ldg(iprow + vi) : 0;
            fa[u] = in ? __ldg(a.ix.short_add + lo + vi) : 0.f;
            fs[u] = in ? __ldg(a.ix.short_scale + lo + vi) : 0.f;
            fe[u] = in ? __ldg(a.ix.short_err + lo + vi) : 0.f;
          }
        }
        int dec[RSUB];
        bool open = false;
#pragma unroll
        for (int u = 0; u < RSUB; ++u) {
          const int64_t vi = c0 + u * 32 + lane;
          if (LUT) {
            const float t1 = __int_as_float(ipv[u]);
            dec[u] = vi < n_c ? stage1_decide_f32x(t1, fa[u], fs[u], fe[u], f32, eq + fabsf(t1) * 0x1p-23f) : 0;
            if (dec[u] < 0)  // the exact table sum, out of line
              dec[u] = decide64_lut(a.ix.packed_msb + (int64_t)a.g * lo, n_c, vi, a.g, a.luts + q * 8 * a.g * 16,
                                    fa[u], fs[u], fe[u], d_qc2, sc, T_list - rT, T_list + rT);
          } else {
            dec[u] = vi < n_c ? stage1_decide_f32(ipv[u], fa[u], fs[u], fe[u], f32) : 0;
            // the float64 test inside the float32 band (about 1e-5 of the vectors), out of line
            if (dec[u] < 0)
              dec[u] = decide64(ipv[u], fa[u], fs[u], fe[u], d_qc2, sc, T_list - rT, T_list + rT);
          }
          open |= dec[u] < 0;
        }
        if (__any_sync(FULL, open)) {
          // the threshold's interval leaves a test open: exact values for the list-start
          // queue's possible members give the exact T for the rest of this list
          T_list = resolve_threshold(a.ix.rcodes, a.ix.long_factors, a.probe_d2 + q * a.nprobe,
                                     a.qslices + q * SLICES * (int64_t)kp, a.ix.pids, a.ix.rcode_bytes, kp,
                                     (int)sc[IVRQ_QS_SLICE_EXP], sc[IVRQ_QS_KB_SUM], rq, rcode_nibbles(a.ix.bits), hl,
                                     snap_d, snap_e, k);
          rT = 0.0;
          f32.T_lo = __double2float_rd(T_list);
          f32.T_hi = __double2float_ru(T_list);
#pragma unroll
          for (int u = 0; u < RSUB; ++u)
            if (dec[u] < 0)
              dec[u] = LUT ? decide64_lut(a.ix.packed_msb + (int64_t)a.g * lo, n_c, c0 + u * 32 + lane, a.g,
                                          a.luts + q * 8 * a.g * 16, fa[u], fs[u], fe[u], d_qc2, sc, T_list, T_list)
                           : decide64(ipv[u], fa[u], fs[u], fe[u], d_qc2, sc, T_list, T_list);
        }
        bool keep[RSUB];
#pragma unroll
        for (int u = 0; u < RSUB; ++u) keep[u] = dec[u] > 0;
#pragma unroll 1
        for (int u = 0; u < RSUB; ++u) {  // one copy of the queue code (instruction cache); values
          const float d0 = pre[0];        // rotate through slot 0 so every index stays static
          const bool k0 = keep[0];
#pragma unroll
          for (int j = 0; j + 1 < RSUB; ++j) {
            pre[j] = pre[j + 1];
            keep[j] = keep[j + 1];
          }
          const unsigned kbits = __ballot_sync(FULL, k0);
          if (!kbits) continue;
          surv += __popc(kbits);
          offer(d0, k0 ? ((lo + c0 + u * 32 + lane) | ((int64_t)p << E_PSH)) : NO_ID);
        }
      }
    }
    check_saturation();
  }
  // the queue (values, entries) for rda_final_kernel, which makes the top k exact
  a.fin_d[q * 32 + lane] = qd;
  a.fin_e[q * 32 + lane] = qi;
  if (lane == 0) {
    if (a.stats) {
      a.stats[2 * q] = probed;
      a.stats[2 * q + 1] = surv;
    }
    if (unsafe) a.fix_list[atomicAdd(a.fix_count, 1)] = (int32_t)q;
  }
  }  // query slots
}

// The end of the approximate pass, one CTA (4 warps) per query: exact values for the queue's
// possible members of the top k (the warps share the query's digit table in shared memory and
// split the entries), the queue re-sorted by (value, pid), the first k written out.
constexpr int FIN_W = 4;

#ifndef FIN_MINB
#define FIN_MINB 10  // 48 registers: 10 CTAs per SM (C3 step 3.26 -> 3.24 ms; 12 CTAs at 40 registers: 3.29)
#endif
__global__ void __launch_bounds__(FIN_W * 32, FIN_MINB) rda_final_kernel(Args a) {
  extern __shared__ __align__(16) unsigned char fin_smem[];
  int2* hl = reinterpret_cast<int2*>(fin_smem);
  double* sd = reinterpret_cast<double*>(fin_smem + (size_t)a.kpad * sizeof(int2));
  int64_t* se = reinterpret_cast<int64_t*>(sd + 32);
  __shared__ int s_need[32];
  __shared__ int s_nneed;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t q = blockIdx.x;
  const int k = a.k, kp = a.kpad;
  const double* sc = a.scalars + q * IVRQ_QS_COUNT;
  ExactCtx ec;
  ec.rcodes = a.ix.rcodes;
  ec.lf = reinterpret_cast<const float2*>(a.ix.long_factors);
  ec.pd2 = a.probe_d2 + q * a.nprobe;
  ec.qs = a.qslices + q * SLICES * (int64_t)kp;
  ec.rb = a.ix.rcode_bytes;
  ec.kp = kp;
  ec.sexp = (int)sc[IVRQ_QS_SLICE_EXP];
  ec.kb = sc[IVRQ_QS_KB_SUM];
  ec.rq = a.rrad[q];
  ec.nib = rcode_nibbles(a.ix.bits);
  // the digit table, all threads: four slice positions per thread and pass
  for (int k0 = 4 * (int)threadIdx.x; k0 < kp; k0 += 4 * FIN_W * 32) {
    uint32_t w[SLICES];
#pragma unroll
    for (int s2 = 0; s2 < SLICES; ++s2) w[s2] = __ldg(reinterpret_cast<const uint32_t*>(ec.qs + s2 * kp + k0));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int h = 0, l = 0;
#pragma unroll
      for (int s2 = 0; s2 < 4; ++s2) {
        h = h * 128 + (int)(int8_t)(w[s2] >> (8 * j));
        l = l * 128 + (int)(int8_t)(w[s2 + 4] >> (8 * j));
      }
      hl[slice_pos(k0 + j)] = make_int2(h, l);
    }
  }
  if (wid == 0) {
    const double qd = a.fin_d[q * 32 + lane];
    const int64_t qi = a.fin_e[q * 32 + lane];
    sd[lane] = qd;
    se[lane] = qi;
    const double kd = __shfl_sync(FULL, qd, k - 1);
    const int64_t ke = __shfl_sync(FULL, qi, k - 1);
    const double lim = kd + entry_rad(kd, ke, ec.rq);
    const bool need = qi != NO_ID && !(qi & (E_EXACT | E_PIDE)) && dsub(qd, entry_rad(qd, qi, ec.rq)) <= lim;
    const unsigned m = __ballot_sync(FULL, need);
    if (need) s_need[__popc(m & ((1u << lane) - 1u))] = lane;
    if (lane == 0) s_nneed = __popc(m);
  }
  __syncthreads();
  for (int i = wid; i < s_nneed; i += FIN_W) {
    const int slot = s_need[i];
    const double x = exact_value(ec, hl, se[slot]);
    if (lane == 0) {
      sd[slot] = x;
      se[slot] |= E_EXACT;
    }
  }
  __syncthreads();
  if (wid == 0) {
    double qd = sd[lane];
    int64_t qi = se[lane];
    warp_sort32(qd, qi, EntryLess{a.ix.pids});
    const int pn = __popc(__ballot_sync(FULL, lane < k && qi != NO_ID));
    if (lane < k) {
      a.out_ids[q * k + lane] = lane < pn ? entry_pid(a.ix.pids, qi) : -1;
      a.out_dists[q * k + lane] = lane < pn ? qd : dinf();
    }
    if (lane == 0) a.out_counts[q] = pn;
  }
}

// ------------------------------------------------------------ kernel, k > 32
// block-wide bitonic sort (ascending (key, id)) of n (power of two) entries
__device__ void bitonic_sort(double* key, int64_t* id, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < (n >> 1); t += blockDim.x) {
        const int lo = 2 * t - (t & (stride - 1));
        const int hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const double kl = key[lo], kh = key[hi];
        const int64_t il = id[lo], ih = id[hi];
        const bool swap = up ? key_less(kh, ih, kl, il) : key_less(kl, il, kh, ih);
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

template <int MODE, bool REFINE, bool NIB, int QB>
__global__ void __launch_bounds__(THREADS) scan_kernel_bigk(Args a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_ncand, s_nfilt, s_pool_n;
  __shared__ double s_T;
  __shared__ long long s_probed, s_surv;
  if (blockIdx.x >= a.nq) return;
  const int64_t q = a.qorder ? a.qorder[blockIdx.x] : (int64_t)blockIdx.x;
  const int k = a.k;
  const int tid = threadIdx.x, lane = tid & 31;
  const Smem s = carve<MODE, REFINE>(a, smem, true);
  const QueryCtx qc = load_query<MODE, REFINE>(a, s, q);
  const int init_n = a.init_counts ? a.init_counts[q] : 0;
  for (int i = tid; i < init_n; i += THREADS) {
    s.s_pool_d[i] = a.init_dists[q * k + i];
    s.s_pool_i[i] = a.init_ids[q * k + i];
  }
  if (tid == 0) {
    s_pool_n = init_n;
    s_T = init_n >= k ? a.init_dists[q * k + k - 1] : dinf();
    s_probed = 0;
    s_surv = 0;
  }
  __syncthreads();
  const int64_t* pid_list = a.probe_ids + q * a.nprobe;
  const double* pd2_list = a.probe_d2 + q * a.nprobe;
  for (int p = 0; p < a.nprobe; ++p) {
    const int64_t cg = pid_list[p];
    if (cg < a.list_lo || cg >= a.list_hi) continue;  // another shard's list
    const int64_t c = cg - a.list_lo;
    const double d_qc2 = pd2_list[p];
    const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
    if (n_c == 0) continue;
    const double T_list = a.prune ? s_T : dinf();
    const double sq = dsqrt(d_qc2);
    const uint32_t* words = a.ix.packed_msb + (int64_t)a.g * lo;
    for (int64_t c0 = 0; c0 < n_c; c0 += CHUNK) {
      const int cn = (int)min((int64_t)CHUNK, n_c - c0);
      if (tid == 0) s_ncand = 0;
      __syncthreads();
      stage1_chunk<MODE, QB, 0>(a, qc, words, lo, n_c, c0, cn, d_qc2, sq, T_list, s.s_planes8, s.s_lut, s.s_cv,
                                s.s_cd, &s_ncand, nullptr);
      __syncthreads();
      const int ncand = s_ncand;
      if (tid == 0) {
        s_probed += cn;
        s_surv += ncand;
      }
      if (ncand == 0) continue;
      if (REFINE) {
        refine_chunk<NIB>(a, qc, lo, c0, d_qc2, s.s_slices, s.s_cv, s.s_cd, ncand);
        __syncthreads();
      }
      if (tid == 0) s_nfilt = 0;
      __syncthreads();
      const int pn = s_pool_n;
      const bool full = pn >= k;
      const double kd = full ? s.s_pool_d[k - 1] : 0.0;
      const int64_t kid = full ? s.s_pool_i[k - 1] : 0;
      for (int cb = 0; cb < ncand; cb += THREADS) {
        const int ci = cb + tid;
        bool pass = false;
        double dist = 0.0;
        int64_t pid = 0;
        if (ci < ncand) {
          dist = s.s_cd[ci];
          pid = (int64_t)__ldg(a.ix.pids + lo + c0 + s.s_cv[ci]);
          pass = !full || key_less(dist, pid, kd, kid);
        }
        const unsigned pb = __ballot_sync(FULL, pass);
        int base = 0;
        if (lane == 0 && pb) base = atomicAdd(&s_nfilt, __popc(pb));
        base = __shfl_sync(FULL, base, 0);
        if (pass) {
          const int pos = pn + base + __popc(pb & ((1u << lane) - 1u));
          s.s_sortk[pos] = dist;
          s.s_sorti[pos] = pid;
        }
      }
      __syncthreads();
      const int m = s_nfilt;
      if (m > 0) {
        for (int i = tid; i < pn; i += THREADS) {
          s.s_sortk[i] = s.s_pool_d[i];
          s.s_sorti[i] = s.s_pool_i[i];
        }
        const int tot = pn + m;
        int n2 = 1;
        while (n2 < tot) n2 <<= 1;
        for (int i = tot + tid; i < n2; i += THREADS) {
          s.s_sortk[i] = dinf();
          s.s_sorti[i] = NO_ID;
        }
        bitonic_sort(s.s_sortk, s.s_sorti, n2);
        const int newn = min(tot, k);
        for (int i = tid; i < newn; i += THREADS) {
          s.s_pool_d[i] = s.s_sortk[i];
          s.s_pool_i[i] = s.s_sorti[i];
        }
        __syncthreads();
        if (tid == 0) s_pool_n = newn;
      }
      __syncthreads();
    }
    if (tid == 0 && s_pool_n >= k) s_T = s.s_pool_d[k - 1];
    __syncthreads();
  }
  const int pn = s_pool_n;
  for (int i = tid; i < k; i += THREADS) {
    a.out_ids[q * k + i] = i < pn ? s.s_pool_i[i] : -1;
    a.out_dists[q * k + i] = i < pn ? s.s_pool_d[i] : dinf();
  }
  if (tid == 0) {
    a.out_counts[q] = pn;
    if (a.stats) {
      a.stats[2 * q] = s_probed;
      a.stats[2 * q + 1] = s_surv;
    }
  }
}

// ------------------------------------------------------------ first-list phase
// Each query's first (lowest-id) probed list is scanned with the threshold at
// +inf (search.py:435 before any merge): every vector survives and is refined.
// That is the bulk of all refines, and queries sharing a first list can share
// one pass over its codes: one CTA takes a list and up to QG of the queries
// whose first list it is, streams the list's rcodes once through the int8
// tensor cores against all their digit slices, and leaves each query's pool
// after that list.  scan_kernel then continues from those pools.
constexpr int QG = 8;

struct FArgs {
  ivrq_index_view ix;
  int64_t list_lo, list_hi;
  const int64_t* probe_ids;
  const double* probe_d2;
  int nprobe;
  const double* scalars;
  const int8_t* qslices;
  int kpad;
  const int64_t* qorder;  // queries sorted by first list (local id), bucket nlist = none
  const int64_t* qoff;    // [nlist + 2] start of each bucket in qorder
  const int32_t* gpre;    // [nlist + 1] prefix sum of ceil(bucket size / QG)
  int nlist, k;
  int64_t* pool_ids;
  double* pool_d;
  int32_t* pool_n;
  int64_t* stats;
};

__global__ void group_prefix_kernel(const int64_t* __restrict__ qoff, int nlist, int32_t* __restrict__ gpre) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int32_t s = 0;
  gpre[0] = 0;
  for (int c = 0; c < nlist; ++c) {
    s += (int32_t)((qoff[c + 1] - qoff[c] + QG - 1) / QG);
    gpre[c + 1] = s;
  }
}

template <bool NIB>
__global__ void __launch_bounds__(THREADS) first_list_kernel(FArgs a) {
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ double s_qd[WARPS][32];
  __shared__ int64_t s_qi[WARPS][32];
  __shared__ int64_t s_q[QG];
  __shared__ double s_dq[QG], s_kb[QG], s_hs[QG], s_ls[QG];
  __shared__ int s_e[QG];
  __shared__ unsigned long long s_bnd[QG];  // bits of a bound on each query's k-th distance
  const int b = blockIdx.x;
  if (b >= a.gpre[a.nlist]) return;
  int lo_c = 0, hi_c = a.nlist;  // gpre[lo_c] <= b < gpre[hi_c]
  while (hi_c - lo_c > 1) {
    const int mid = (lo_c + hi_c) >> 1;
    if (a.gpre[mid] <= b) lo_c = mid; else hi_c = mid;
  }
  const int c = lo_c;
  const int64_t qs = a.qoff[c] + (int64_t)(b - a.gpre[c]) * QG;
  const int nqg = (int)min((int64_t)QG, a.qoff[c + 1] - qs);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gid = lane >> 2, t4 = lane & 3;
  const int kp = a.kpad, ss = kp + SPAD, k = a.k;
  int8_t* s_sl = reinterpret_cast<int8_t*>(fsm);  // [QG][SLICES][ss]
  if (tid < QG) {
    int64_t q = -1;
    double dq = 0.0;
    if (tid < nqg) {
      q = a.qorder[qs + tid];
      for (int p = 0; p < a.nprobe; ++p) {  // the first in-range probe is list c
        if (a.probe_ids[q * a.nprobe + p] == c + a.list_lo) {
          dq = a.probe_d2[q * a.nprobe + p];
          break;
        }
      }
      s_kb[tid] = a.scalars[q * IVRQ_QS_COUNT + IVRQ_QS_KB_SUM];
      s_e[tid] = (int)a.scalars[q * IVRQ_QS_COUNT + IVRQ_QS_SLICE_EXP];
      s_hs[tid] = ldexp(1.0, s_e[tid] - 26);
      s_ls[tid] = ldexp(1.0, s_e[tid] - 54);
    }
    s_q[tid] = q;
    s_dq[tid] = dq;
    s_bnd[tid] = 0x7ff0000000000000ULL;  // +inf
  }
  __syncthreads();
  for (int i = tid; i < nqg * SLICES * kp / 4; i += THREADS) {
    const int j = (4 * i) / (SLICES * kp), rem = (4 * i) % (SLICES * kp);
    const int sidx = rem / kp, kk = rem % kp;
    *reinterpret_cast<uint32_t*>(s_sl + (j * SLICES + sidx) * ss + kk) =
        reinterpret_cast<const uint32_t*>(a.qslices + s_q[j] * SLICES * (int64_t)kp)[rem / 4];
  }
  __syncthreads();
  const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
  const int64_t rb = a.ix.rcode_bytes;
  double qd[QG];
  int64_t qi[QG];
#pragma unroll
  for (int j = 0; j < QG; ++j) {
    qd[j] = dinf();
    qi[j] = NO_ID;
  }
  for (int64_t t0 = (int64_t)wid * 16; t0 < n_c; t0 += WARPS * 16) {
    const int64_t v0 = min(t0 + gid, n_c - 1), v1 = min(t0 + gid + 8, n_c - 1);
    const uint8_t* row0 = a.ix.rcodes + (lo + v0) * rb;
    const uint8_t* row1 = a.ix.rcodes + (lo + v1) * rb;
    int acc[QG][4];
#pragma unroll
    for (int j = 0; j < QG; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
    for (int p = 0; p < kp / 64; ++p) {
      uint32_t a0s0, a2s0, a0s1, a2s1, a1s0, a3s0, a1s1, a3s1;
      if (NIB) {
        const uint2 x0 = __ldg(reinterpret_cast<const uint2*>(row0 + 8 * (4 * p + t4)));
        const uint2 x1 = __ldg(reinterpret_cast<const uint2*>(row1 + 8 * (4 * p + t4)));
        a0s0 = x0.x & 0x0F0F0F0Fu;
        a2s0 = (x0.x >> 4) & 0x0F0F0F0Fu;
        a0s1 = x0.y & 0x0F0F0F0Fu;
        a2s1 = (x0.y >> 4) & 0x0F0F0F0Fu;
        a1s0 = x1.x & 0x0F0F0F0Fu;
        a3s0 = (x1.x >> 4) & 0x0F0F0F0Fu;
        a1s1 = x1.y & 0x0F0F0F0Fu;
        a3s1 = (x1.y >> 4) & 0x0F0F0F0Fu;
      } else {
        const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(row0 + 16 * (4 * p + t4)));
        const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(row1 + 16 * (4 * p + t4)));
        a0s0 = x0.x;
        a2s0 = x0.y;
        a0s1 = x0.z;
        a2s1 = x0.w;
        a1s0 = x1.x;
        a3s0 = x1.y;
        a1s1 = x1.z;
        a3s1 = x1.w;
      }
#pragma unroll
      for (int j = 0; j < QG; ++j) {
        if (j < nqg) {
          const int8_t* sl = s_sl + (j * SLICES + gid) * ss + 4 * t4 + 64 * p;
          const uint32_t b00 = *reinterpret_cast<const uint32_t*>(sl);
          const uint32_t b10 = *reinterpret_cast<const uint32_t*>(sl + 16);
          const uint32_t b01 = *reinterpret_cast<const uint32_t*>(sl + 32);
          const uint32_t b11 = *reinterpret_cast<const uint32_t*>(sl + 48);
          mma_u8s8(acc[j], a0s0, a1s0, a2s0, a3s0, b00, b10);
          mma_u8s8(acc[j], a0s1, a1s1, a2s1, a3s1, b01, b11);
        }
      }
    }
    // rows of this tile as candidate lanes 0..15 (lane L <- row t0 + L)
    const int L = lane & 15;
    const bool row_ok = lane < 16 && t0 + L < n_c;
    const long long w0 = (t4 & 1) ? 128LL : 2097152LL;
    const long long w1 = (t4 & 1) ? 1LL : 16384LL;
    float2 lf = make_float2(0.f, 0.f);
    if (row_ok) lf = __ldg(reinterpret_cast<const float2*>(a.ix.long_factors) + lo + t0 + L);
#pragma unroll
    for (int j = 0; j < QG; ++j) {
      if (j >= nqg) continue;
      long long p0 = (long long)acc[j][0] * w0 + (long long)acc[j][1] * w1;
      long long p1 = (long long)acc[j][2] * w0 + (long long)acc[j][3] * w1;
      p0 += __shfl_xor_sync(FULL, p0, 1);
      p1 += __shfl_xor_sync(FULL, p1, 1);
      const long long l0 = __shfl_xor_sync(FULL, p0, 2);
      const long long l1 = __shfl_xor_sync(FULL, p1, 2);
      const int src = (L & 7) * 4;  // lane t4 == 0 of group (row & 7) holds the sums
      const long long hi0 = __shfl_sync(FULL, p0, src), hi1 = __shfl_sync(FULL, p1, src);
      const long long lw0 = __shfl_sync(FULL, l0, src), lw1 = __shfl_sync(FULL, l1, src);
      double d = dinf();
      if (row_ok) {
        const long long hi = (L >= 8) ? hi1 : hi0, lw = (L >= 8) ? lw1 : lw0;
        const double ip = dadd(dmul((double)hi, s_hs[j]), dmul((double)lw, s_ls[j]));
        d = dmax(dsub(dadd((double)lf.x, s_dq[j]), dmul((double)lf.y, dsub(ip, s_kb[j]))), 0.0);
      }
      const double kd = __shfl_sync(FULL, qd[j], k - 1);
      const int64_t ki = __shfl_sync(FULL, qi[j], k - 1);
      // any warp holding k candidates bounds the query's k-th distance
      const double bound = __longlong_as_double((long long)*(volatile unsigned long long*)&s_bnd[j]);
      const bool maybe = row_ok && d <= kd && d <= bound;
      if (!__any_sync(FULL, maybe)) continue;
      int64_t id = maybe ? (int64_t)__ldg(a.ix.pids + lo + t0 + L) : NO_ID;
      const bool pass = maybe && key_less(d, id, kd, ki);
      if (!__any_sync(FULL, pass)) continue;
      warp_fold(qd[j], qi[j], d, id, pass, k);
      const int64_t full_i = __shfl_sync(FULL, qi[j], k - 1);
      const double full_d = __shfl_sync(FULL, qd[j], k - 1);
      if (lane == 0 && full_i != NO_ID)
        atomicMin(&s_bnd[j], (unsigned long long)__double_as_longlong(full_d));
    }
  }
  // fold the 8 warp queues of each query into its pool
#pragma unroll
  for (int j = 0; j < QG; ++j) {
    if (j >= nqg) break;
    s_qd[wid][lane] = qd[j];
    s_qi[wid][lane] = qi[j];
    __syncthreads();
    if (wid == 0) {
      double pd = s_qd[0][lane];
      int64_t pi = s_qi[0][lane];
      for (int w = 1; w < WARPS; ++w) {
        if (s_qi[w][0] == NO_ID) continue;
        warp_merge32(pd, pi, s_qd[w][lane], s_qi[w][lane]);
      }
      const int64_t q = s_q[j];
      if (lane < k) {
        a.pool_ids[q * k + lane] = pi;
        a.pool_d[q * k + lane] = pd;
      }
      const int cnt = __popc(__ballot_sync(FULL, lane < k && pi != NO_ID));
      if (lane == 0) {
        a.pool_n[q] = cnt;
        if (a.stats) {
          a.stats[2 * q] = n_c;
          a.stats[2 * q + 1] = n_c;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ stage-1 inner products, list-major, int8 tensor cores
// ip_bitwise (search.py:163-183) is sum_j w_j sum_g popc(word & plane_j) with
// w_j the two's-complement weights of the query_bits planes, i.e. exactly the
// integer dot product sum_d bit[v,d] * qhat[q,d] of the 1-bit code with the
// quantized query.  For every (list, query probing it) pair that the
// per-query pass will scan, ip_list_kernel computes that dot for every vector
// of the list as an int8 GEMM on mma.sync m16n8k32 (u8 0/1 codes x s8 qhat,
// int32 accumulate: exact), reading each list's codes once per 64 queries
// instead of once per query.  The per-query pass then reads 2 bytes per
// (pair, vector) and replays the reference's threshold order unchanged.
//
// ip buffer layout: pair (list c, slot s) owns the row
//   ipbuf[pair_base[c] + s * rs(c) + v],  rs(c) = n_c rounded up to 8,
// slots numbered in the stable (list, query, probe) order of the pair sort.

struct IpArgs {
  ivrq_index_view ix;
  const int8_t* qhat;       // [nq][32 g] quantized queries (qhat_kernel)
  int g, nprobe, nlist;
  const int64_t* porder;    // pair indices (q * nprobe + p) sorted by list
  const int64_t* poff;      // [nlist + 2] bucket starts in porder
  const int64_t* pair_base; // [nlist + 1] element offset of each list's rows
  const int32_t* tpre;      // [nlist + 1] prefix of query groups (TQ pairs) per list
  void* ipbuf;              // int16 or int32 elements
};

constexpr int KCH = 8;  // 32-dim groups of code words per staged chunk

__device__ __forceinline__ void mma_s8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// 4 code bits (dims 4i..4i+3 of a word) -> 4 bytes of 0/1
__device__ __forceinline__ uint32_t nib_bytes(uint32_t w, int shift) {
  return (((w >> shift) & 0xFu) * 0x00204081u) & 0x01010101u;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 4 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// qhat[q][32 gi + i] = sum_j w_j bit_i(plane_j[gi]) (two's complement of query_bits bits)
__global__ void qhat_kernel(const uint32_t* __restrict__ planes, int64_t nq, int g, int qb, int8_t* __restrict__ qhat) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= nq * g) return;
  const int64_t q = it / g;
  const int gi = (int)(it % g);
  uint32_t pl[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) pl[j] = j < qb ? planes[(q * qb + j) * g + gi] : 0u;
  uint32_t out[8];
#pragma unroll
  for (int w4 = 0; w4 < 8; ++w4) {
    uint32_t packed = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int i = 4 * w4 + e;
      int v = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) v |= (int)((pl[j] >> i) & 1u) << j;
      v = (v << (32 - qb)) >> (32 - qb);
      packed |= ((uint32_t)v & 0xFFu) << (8 * e);
    }
    out[w4] = packed;
  }
  uint4* dst = reinterpret_cast<uint4*>(qhat + q * 32 * (int64_t)g + 32 * gi);
  dst[0] = make_uint4(out[0], out[1], out[2], out[3]);
  dst[1] = make_uint4(out[4], out[5], out[6], out[7]);
}

// One CTA per (list, group of <= TQ queries probing it), persistent over the
// groups.  The group's qhat rows sit in shared memory; the list's code words
// stream through a cp.async double buffer in (256 vectors x KCH groups)
// stages; each warp owns 32 vectors x all queries of the group.
template <typename IPT>
__global__ void __launch_bounds__(THREADS, 2) ip_list_kernel(IpArgs a) {
  extern __shared__ __align__(16) unsigned char ism[];
  const int g = a.g;
  const int ldq = 32 * g + TQ_PAD;  // bytes per query row of qhat
  int8_t* sq = reinterpret_cast<int8_t*>(ism);
  uint32_t* sw = reinterpret_cast<uint32_t*>(ism + (size_t)TQ * ldq);  // [2][KCH][TV]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gid = lane >> 2, t4 = lane & 3;
  const int total = a.tpre[a.nlist];
  const int nks = (g + KCH - 1) / KCH;
  for (int b = blockIdx.x; b < total; b += gridDim.x) {
    int lo_c = 0, hi_c = a.nlist;  // tpre[lo_c] <= b < tpre[hi_c]
    while (hi_c - lo_c > 1) {
      const int mid = (lo_c + hi_c) >> 1;
      if (a.tpre[mid] <= b) lo_c = mid; else hi_c = mid;
    }
    const int c = lo_c;
    const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
    const int qt = b - a.tpre[c];
    const int64_t pb = a.poff[c] + (int64_t)qt * TQ;
    const int nqt = (int)min((int64_t)TQ, a.poff[c + 1] - pb);
    const int nmt = (nqt + 15) >> 4;  // warp-uniform
    const uint32_t* words = a.ix.packed_msb + (int64_t)g * lo;
    const int64_t nvt = ceil_div(n_c, TV);
    const int nst = (int)(nvt * nks);
    auto issue = [&](int st) {
      const int64_t v0 = (st / nks) * (int64_t)TV;
      const int k0 = (st % nks) * KCH;
      uint32_t* dst = sw + (st & 1) * KCH * TV;
      for (int i = tid; i < KCH * TV; i += THREADS) {
        const int jj = i / TV, vv = i % TV;
        const int64_t v = v0 + vv;
        const bool ok = k0 + jj < g && v < n_c;
        cp_async4(dst + i, ok ? words + (int64_t)(k0 + jj) * n_c + v : words, ok);
      }
      cp_async_commit();
    };
    __syncthreads();  // the previous group is done with sq / sw
    issue(0);
    for (int i = tid; i < TQ * (8 * g); i += THREADS) {  // qhat rows, 4 bytes at a time
      const int r = i / (8 * g), w = i % (8 * g);
      uint32_t v = 0;
      if (r < nqt) v = __ldg(reinterpret_cast<const uint32_t*>(a.qhat + (a.porder[pb + r] / a.nprobe) * 32 * (int64_t)g) + w);
      *reinterpret_cast<uint32_t*>(sq + r * ldq + 4 * w) = v;
    }
    int acc[4][4][4];
    for (int st = 0; st < nst; ++st) {
      const int kc = st % nks;
      const int64_t v0 = (st / nks) * (int64_t)TV;
      if (kc == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = acc[i][j][2] = acc[i][j][3] = 0;
      }
      if (st + 1 < nst) {
        issue(st + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const uint32_t* w0 = sw + (st & 1) * KCH * TV + wid * 32 + gid;
      const int k0 = kc * KCH;
      const int kn = min(KCH, g - k0);
      for (int jj = 0; jj < kn; ++jj) {
        const int gi = k0 + jj;
        uint32_t bf[4][2];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
          const uint32_t w = w0[jj * TV + nt * 8];
          bf[nt][0] = nib_bytes(w, 4 * t4);
          bf[nt][1] = nib_bytes(w, 16 + 4 * t4);
        }
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          if (mt < nmt) {
            const int8_t* r0 = sq + (mt * 16 + gid) * ldq + 32 * gi + 4 * t4;
            const int8_t* r1 = r0 + 8 * ldq;
            uint32_t af[4];
            af[0] = *reinterpret_cast<const uint32_t*>(r0);
            af[1] = *reinterpret_cast<const uint32_t*>(r1);
            af[2] = *reinterpret_cast<const uint32_t*>(r0 + 16);
            af[3] = *reinterpret_cast<const uint32_t*>(r1 + 16);
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) mma_s8u8(acc[mt][nt], af, bf[nt][0], bf[nt][1]);
          }
        }
      }
      if (kc == nks - 1) {  // epilogue of this vector tile
        const int64_t rs = ip_row_stride(n_c);
        IPT* base = reinterpret_cast<IPT*>(a.ipbuf) + a.pair_base[c] + (int64_t)qt * TQ * rs;
        const int64_t vw = v0 + wid * 32;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) {
          if (mt >= nmt) continue;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int r = mt * 16 + gid + 8 * h;
            if (r >= nqt) continue;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
              const int64_t v = vw + nt * 8 + 2 * t4;  // even; v + 1 stays inside the padded row
              if (v >= n_c) continue;
              IPT* dst = base + (int64_t)r * rs + v;
              const int x0 = acc[mt][nt][2 * h], x1 = acc[mt][nt][2 * h + 1];
              if constexpr (sizeof(IPT) == 2) {
                *reinterpret_cast<uint32_t*>(dst) = ((uint32_t)x0 & 0xFFFFu) | ((uint32_t)x1 << 16);
              } else {
                *reinterpret_cast<int2*>(dst) = make_int2(x0, x1);
              }
            }
          }
        }
      }
      __syncthreads();  // buffer (st & 1) is refilled by issue(st + 2)
    }
  }
}

// pair keys: list of every in-range probe the per-query pass scans (the first
// in-range probe is excluded when the first-list phase handles it)
// excl: 0 every in-range probe, 1 all but the first in-range probe (scanned
// with the threshold still +inf, where the inner products are not needed),
// 2 none (prune off with refine on: no list needs them)
__global__ void pair_key_kernel(const int64_t* __restrict__ probe_ids, int64_t nq, int nprobe, int64_t list_lo,
                                int64_t list_hi, int excl, int32_t* __restrict__ keys) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const int32_t none = (int32_t)(list_hi - list_lo);
  bool first = excl == 1;
  for (int p = 0; p < nprobe; ++p) {
    const int64_t cg = probe_ids[q * nprobe + p];
    int32_t key = none;
    if (cg >= list_lo && cg < list_hi && excl != 2) {
      if (first) first = false;
      else key = (int32_t)(cg - list_lo);
    }
    keys[q * nprobe + p] = key;
  }
}

// slot of each pair inside its list's bucket
__global__ void pair_slot_kernel(const int64_t* __restrict__ porder, const int64_t* __restrict__ poff,
                                 const int32_t* __restrict__ keys, int64_t npairs, int32_t none,
                                 int32_t* __restrict__ pslot) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npairs) return;
  const int64_t pr = porder[i];
  const int32_t c = keys[pr];
  pslot[pr] = c < none ? (int32_t)(i - poff[c]) : -1;
}

// pair_base (elements) and tile prefix over the lists; one block.
// totals[0] = ip elements, totals[1] = tiles.
__global__ void __launch_bounds__(1024) pair_plan_kernel(const int64_t* __restrict__ offsets,
                                                         const int64_t* __restrict__ poff, int nlist, int grp,
                                                         int64_t* __restrict__ pair_base, int32_t* __restrict__ tpre,
                                                         int64_t* __restrict__ totals) {
  __shared__ int64_t s_e[32], s_t[32];
  __shared__ int64_t s_run_e, s_run_t;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    s_run_e = 0;
    s_run_t = 0;
  }
  __syncthreads();
  for (int c0 = 0; c0 < nlist; c0 += 1024) {
    const int c = c0 + tid;
    int64_t e = 0, t = 0;
    if (c < nlist) {
      const int64_t n_c = offsets[c + 1] - offsets[c], cnt = poff[c + 1] - poff[c];
      e = cnt * ip_row_stride(n_c);
      // grp > 0: groups of grp pairs; grp < 0: tiles of -grp rows of the list (lists with pairs)
      t = (n_c > 0 && cnt > 0) ? (grp > 0 ? ceil_div(cnt, grp) : ceil_div(n_c, -grp)) : 0;
    }
    int64_t ie = e, it = t;  // inclusive warp scans
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t xe = __shfl_up_sync(FULL, ie, o), xt = __shfl_up_sync(FULL, it, o);
      if (lane >= o) {
        ie += xe;
        it += xt;
      }
    }
    if (lane == 31) {
      s_e[wid] = ie;
      s_t[wid] = it;
    }
    __syncthreads();
    if (wid == 0) {
      int64_t we = s_e[lane], wt = s_t[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t xe = __shfl_up_sync(FULL, we, o), xt = __shfl_up_sync(FULL, wt, o);
        if (lane >= o) {
          we += xe;
          wt += xt;
        }
      }
      s_e[lane] = we;  // inclusive over warps
      s_t[lane] = wt;
    }
    __syncthreads();
    const int64_t before_e = s_run_e + (wid ? s_e[wid - 1] : 0) + ie - e;
    const int64_t before_t = s_run_t + (wid ? s_t[wid - 1] : 0) + it - t;
    if (c < nlist) {
      pair_base[c] = before_e;
      tpre[c] = (int32_t)before_t;
    }
    __syncthreads();
    if (tid == 0) {
      s_run_e += s_e[31];
      s_run_t += s_t[31];
    }
    __syncthreads();
  }
  if (tid == 0) {
    pair_base[nlist] = s_run_e;
    tpre[nlist] = (int32_t)s_run_t;
    totals[0] = s_run_e;
    totals[1] = s_run_t;
  }
}

// ------------------------------------------------------------ first lists, list-major refine
// Each query's first in-range list is scanned with the threshold at +inf
// (search.py:435 before any merge), so every vector is refined.  Queries that
// share a first list share its rcodes: one CTA takes a list and FQ of those
// queries, streams the list's rcode rows through shared memory (cp.async, 128
// rows x one 64-dim step per stage) and runs the int8 MMAs against all FQ
// queries' digit slices, writing the refined distance of every (query,
// vector) (refine_chunk's exact arithmetic) for the warp kernel to merge.
constexpr int FQ = 8;     // queries per group (n8 tiles of 8 digit slices)
constexpr int FROWS = 128;  // rcode rows per tile: 8 warps x 16

struct FdArgs {
  ivrq_index_view ix;
  int64_t list_lo;
  const int64_t* probe_ids;
  const double* probe_d2;
  int nprobe, nlist, kpad;
  const double* scalars;
  const int8_t* qslices;
  const int64_t* qorder;
  const int64_t* qoff;    // [nlist + 2] first-list buckets in qorder
  const int64_t* fbase;   // [nlist + 1]
  const int32_t* gpre;    // [nlist + 1] prefix of ceil(bucket / FQ)
  double* fdist;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 16 : 0));
}

template <bool NIB>
__global__ void __launch_bounds__(THREADS, 2) first_dist_kernel(FdArgs a) {
  extern __shared__ __align__(16) unsigned char fsm2[];
  __shared__ double s_dq[FQ], s_kb[FQ], s_hs[FQ], s_ls[FQ];
  __shared__ int64_t s_row[FQ];
  constexpr int CB = NIB ? 32 : 64;  // rcode bytes per row per 64-dim step
  const int kp = a.kpad, ss = kp + SPAD;
  int8_t* s_sl = reinterpret_cast<int8_t*>(fsm2);  // [FQ][SLICES][ss]
  uint8_t* s_a = reinterpret_cast<uint8_t*>(fsm2 + (size_t)FQ * SLICES * ss);  // [2][FROWS][CB]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gid = lane >> 2, t4 = lane & 3;
  const int np = kp / 64;
  const int total = a.gpre[a.nlist];
  const int64_t rb = a.ix.rcode_bytes;
  for (int b = blockIdx.x; b < total; b += gridDim.x) {
    int lo_c = 0, hi_c = a.nlist;
    while (hi_c - lo_c > 1) {
      const int mid = (lo_c + hi_c) >> 1;
      if (a.gpre[mid] <= b) lo_c = mid; else hi_c = mid;
    }
    const int c = lo_c;
    const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
    const int64_t qs = a.qoff[c] + (int64_t)(b - a.gpre[c]) * FQ;
    const int nqg = (int)min((int64_t)FQ, a.qoff[c + 1] - qs);
    const int64_t rs = ip_row_stride(n_c);
    const uint8_t* rows = a.ix.rcodes + lo * rb;
    const int nst = (int)ceil_div(n_c, FROWS) * np;
    auto issue = [&](int st) {
      const int64_t v0 = (int64_t)(st / np) * FROWS;
      const int p = st % np;
      uint8_t* dst = s_a + (st & 1) * FROWS * CB;
      for (int i = tid; i < FROWS * CB / 16; i += THREADS) {
        const int r = i / (CB / 16), part = i % (CB / 16);
        const bool ok = v0 + r < n_c;
        cp_async16(dst + r * CB + 16 * part, ok ? rows + (v0 + r) * rb + p * CB + 16 * part : rows, ok);
      }
      cp_async_commit();
    };
    __syncthreads();  // previous group done with shared memory
    if (nst > 0) issue(0);
    if (tid < FQ) {
      double dq = 0.0, kb = 0.0;
      int e = 0;
      int64_t row = -1;
      if (tid < nqg) {
        const int64_t q = a.qorder[qs + tid];
        for (int p = 0; p < a.nprobe; ++p) {  // the first in-range probe is list c
          if (a.probe_ids[q * a.nprobe + p] == c + a.list_lo) {
            dq = a.probe_d2[q * a.nprobe + p];
            break;
          }
        }
        kb = a.scalars[q * IVRQ_QS_COUNT + IVRQ_QS_KB_SUM];
        e = (int)a.scalars[q * IVRQ_QS_COUNT + IVRQ_QS_SLICE_EXP];
        row = a.fbase[c] + (qs + tid - a.qoff[c]) * rs;
      }
      s_dq[tid] = dq;
      s_kb[tid] = kb;
      s_hs[tid] = ldexp(1.0, e - 26);
      s_ls[tid] = ldexp(1.0, e - 54);
      s_row[tid] = row;
    }
    for (int i = tid; i < FQ * SLICES * kp / 4; i += THREADS) {
      const int j = (4 * i) / (SLICES * kp), rem = (4 * i) % (SLICES * kp);
      const int sidx = rem / kp, kk = rem % kp;
      uint32_t v = 0;
      if (j < nqg)
        v = __ldg(reinterpret_cast<const uint32_t*>(a.qslices + a.qorder[qs + j] * SLICES * (int64_t)kp) + rem / 4);
      *reinterpret_cast<uint32_t*>(s_sl + (j * SLICES + sidx) * ss + kk) = v;
    }
    int acc[FQ][4];
    for (int st = 0; st < nst; ++st) {
      const int p = st % np;
      const int64_t v0 = (int64_t)(st / np) * FROWS;
      if (p == 0) {
#pragma unroll
        for (int j = 0; j < FQ; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0;
      }
      if (st + 1 < nst) {
        issue(st + 1);
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
      __syncthreads();
      const uint8_t* ta = s_a + (st & 1) * FROWS * CB + (wid * 16 + gid) * CB;
      uint32_t as0[4], as1[4];
      if (NIB) {
        const uint2 x0 = *reinterpret_cast<const uint2*>(ta + 8 * t4);
        const uint2 x1 = *reinterpret_cast<const uint2*>(ta + 8 * CB + 8 * t4);
        as0[0] = x0.x & 0x0F0F0F0Fu;
        as0[2] = (x0.x >> 4) & 0x0F0F0F0Fu;
        as1[0] = x0.y & 0x0F0F0F0Fu;
        as1[2] = (x0.y >> 4) & 0x0F0F0F0Fu;
        as0[1] = x1.x & 0x0F0F0F0Fu;
        as0[3] = (x1.x >> 4) & 0x0F0F0F0Fu;
        as1[1] = x1.y & 0x0F0F0F0Fu;
        as1[3] = (x1.y >> 4) & 0x0F0F0F0Fu;
      } else {
        const uint4 x0 = *reinterpret_cast<const uint4*>(ta + 16 * t4);
        const uint4 x1 = *reinterpret_cast<const uint4*>(ta + 8 * CB + 16 * t4);
        as0[0] = x0.x;
        as0[2] = x0.y;
        as1[0] = x0.z;
        as1[2] = x0.w;
        as0[1] = x1.x;
        as0[3] = x1.y;
        as1[1] = x1.z;
        as1[3] = x1.w;
      }
#pragma unroll
      for (int j = 0; j < FQ; ++j) {
        if (j < nqg) {
          const int8_t* sl = s_sl + (j * SLICES + gid) * ss + 4 * t4 + 64 * p;
          const uint32_t b00 = *reinterpret_cast<const uint32_t*>(sl);
          const uint32_t b10 = *reinterpret_cast<const uint32_t*>(sl + 16);
          const uint32_t b01 = *reinterpret_cast<const uint32_t*>(sl + 32);
          const uint32_t b11 = *reinterpret_cast<const uint32_t*>(sl + 48);
          mma_u8s8(acc[j], as0[0], as0[1], as0[2], as0[3], b00, b10);
          mma_u8s8(acc[j], as1[0], as1[1], as1[2], as1[3], b01, b11);
        }
      }
      if (p == np - 1) {  // epilogue of this row tile (refine_chunk's arithmetic)
        const long long w0 = (t4 & 1) ? 128LL : 2097152LL;
        const long long w1 = (t4 & 1) ? 1LL : 16384LL;
        const int64_t r0 = v0 + wid * 16 + gid;
        float2 lf0 = make_float2(0.f, 0.f), lf1 = make_float2(0.f, 0.f);
        if (t4 == 0) {
          if (r0 < n_c) lf0 = __ldg(reinterpret_cast<const float2*>(a.ix.long_factors) + lo + r0);
          if (r0 + 8 < n_c) lf1 = __ldg(reinterpret_cast<const float2*>(a.ix.long_factors) + lo + r0 + 8);
        }
#pragma unroll
        for (int j = 0; j < FQ; ++j) {
          if (j >= nqg) break;
          long long p0 = (long long)acc[j][0] * w0 + (long long)acc[j][1] * w1;
          long long p1 = (long long)acc[j][2] * w0 + (long long)acc[j][3] * w1;
          p0 += __shfl_xor_sync(FULL, p0, 1);
          p1 += __shfl_xor_sync(FULL, p1, 1);
          const long long l0 = __shfl_xor_sync(FULL, p0, 2);
          const long long l1 = __shfl_xor_sync(FULL, p1, 2);
          if (t4 == 0) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int64_t r = r0 + 8 * h;
              if (r >= n_c) continue;
              const long long hi = h ? p1 : p0, lw = h ? l1 : l0;
              const float2 lf = h ? lf1 : lf0;
              const double ip = dadd(dmul((double)hi, s_hs[j]), dmul((double)lw, s_ls[j]));
              a.fdist[s_row[j] + r] =
                  dmax(dsub(dadd((double)lf.x, s_dq[j]), dmul((double)lf.y, dsub(ip, s_kb[j]))), 0.0);
            }
          }
        }
      }
      __syncthreads();  // buffer (st & 1) is refilled by issue(st + 2)
    }
  }
}

// ------------------------------------------------------------ refine of every probed pair on tcgen05
// A certified approximation of the refined distance (search.py:313-323) of
// every vector of every probed (list, query) pair, list-major on the
// 5th-generation tensor cores.  The exact refine (refine_chunk) assembles
// <u, q_rot> from the query's eight base-128 digits; here only the four most
// significant digits D0..D3 go through the tensor cores:
//   hi_v = sum_d u_vd (D0 128^3 + D1 128^2 + D2 128 + D3)_d,  ip ~ hi_v 2^(e-26),
// the neglected low half being at most U_max kpad 135274560 2^(e-54) in
// magnitude.  The distance from this ip is stored as float32 together with a
// per-query radius (rd_radius_kernel) that bounds its distance to the exact
// value; the per-query pass (scan_rda_kernel) decides with intervals and
// computes the exact value of the few entries whose decision the radius
// leaves open, and of its final top k, so results are the exact path's.
// Halving the digits halves the MMA work and the B operand, so a query group
// is twice as large (fewer passes over each list's codes) beside a deeper
// A ring.  For a list c and a group of G queries probing it,
// D[v][(j, s)] = <u_v, digit_s of q_j> is one int8 GEMM (M = 128 vectors per
// TMEM tile, N = 4 G digit rows, K = kpad) with the accumulator in TMEM.
// Warp roles per CTA:
//   warps 0-3  stage rcode tiles (128 rows x 128 B per stage) into a ring
//              (one TMA lane for 8-bit codes; all four warps unpack 4-bit codes),
//   warp 1     also loads the next group's digit rows: one bulk copy per K chunk
//              from the pre-swizzled pair-ordered array (tc_bpairs_kernel), as soon
//              as the previous group's MMAs retire (no CTA barrier between groups),
//   warp 4     issues tcgen05.mma (one elected lane) and commits,
//   warps 5-12 read the accumulator (tcgen05.ld; two warps per TMEM lane
//              quarter, each half of the group's queries), assemble hi_v in int64,
//              and write the approximate distance as float32.
constexpr int TCM = 128;     // vectors per tile = TMEM lanes
constexpr int TCKC = 128;    // K bytes per A stage (4 MMAs of K = 32)
constexpr int TCST = 6;      // A stages (tc_ip_kernel)
constexpr int TC_PROD = 4;  // producer warps
constexpr int TC_THREADS = 32 * (TC_PROD + 1 + 4);
#ifndef TCR_EPQ
#define TCR_EPQ 3
#endif
constexpr int TCR_EPI = 4 * TCR_EPQ;  // tc_refine epilogue warps: TCR_EPQ per TMEM lane quarter, each a share of the
                                      // group's queries
constexpr int TCR_THREADS = 32 * (TC_PROD + 1 + TCR_EPI);

constexpr int TCR_DIG = 4;  // most significant query digits on the tensor cores

struct TcArgs {
  CUtensorMap map_a;        // rcodes [N rows x rcode_bytes] (8-bit codes), box 128 B x 128 rows, 128B swizzle
  const int8_t* bslices;    // [nkc][npairs][4 rows x 128 B] pre-swizzled digit rows in pair order (tc_bpairs_kernel)
  int64_t npairs;
  ivrq_index_view ix;
  int kpad, G, nst, nib;
  const double* scalars;
  const double* probe_d2;
  int nprobe, nlist;
  const int64_t* porder;    // pair indices sorted by list
  const int64_t* poff;      // [nlist + 2]
  const int64_t* pair_base; // [nlist + 1]
  const int32_t* gpre;      // [nlist + 1] prefix of ceil(bucket / G)
  float* rdist;             // approximate refined distances (radius: rd_radius_kernel)
  // fused stage 1 (8-bit codes): the binary inner products <msb(u), qhat> from the same rcode tiles,
  // as (sum u qhat - sum s8(u) qhat) / 256 with u read as unsigned and as signed bytes
  const int8_t* bqhat;      // [nkc][npairs][128 B] (tc_qpairs_kernel), or null
  void* ipbuf;
  int ip32;
  // LUT mode (8-bit codes): the stage-1 estimate <msb(u), q> from the digit rows read both ways,
  // written as float32 (a certified approximation of the LUT sum, see scan_rda_kernel)
  int lut;
  int nib_hi;               // codes of <= 4 bits unpacked as u << nib_hi, nib_hi = 8 - bits (the fused stage 1
                            // reads the code's MSB as the sign bit), else 0
};

// byte offset of (row R, byte k < 128) in a 128B-swizzled K-major tile (8-row atoms of 1024 B)
__host__ __device__ inline uint32_t sw128_offset(int R, int k) {
  return (uint32_t)((R >> 3) * 1024 + (R & 7) * 128 + ((((k >> 4) ^ (R & 7)) & 7) << 4) + (k & 15));
}

// The refine's B operand, materialised in pair order so that one bulk copy per K chunk loads a
// whole query group: out[kc][i] (512 bytes) holds the four digit rows of the query of pair i
// (list-sorted order), pre-swizzled as rows 4 par .. 4 par + 3 of a 128B-swizzled 8-row atom,
// par = the pair's slot parity in its list's bucket (groups start at even slots, so consecutive
// pairs of a group fill one atom), digit d in row 4 par + d, K bytes [128 kc, 128 kc + 128) in
// rcode byte order P with qslices' mma.sync fragment order transposed:
// value(P = 64p + 16t + 4h + j) = qslices[q][d][64p + 16h + 4t + j]; zero past kpad.
__global__ void tc_bpairs_kernel(const int8_t* __restrict__ qslices, const int64_t* __restrict__ porder,
                                 const int32_t* __restrict__ pslot, int64_t npairs, int nprobe, int kp, int nkc,
                                 int8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16-byte chunk of one row
  if (t >= npairs * nkc * 32) return;
  const int w = (int)(t & 31), d = w >> 3, c16 = w & 7;
  const int64_t blk = t >> 5;  // (kc, i), kc major
  const int64_t i = blk % npairs;
  const int kc = (int)(blk / npairs);
  const int64_t pr = porder[i];
  const int32_t slot = pslot[pr];
  if (slot < 0) return;  // not a pair of this shard
  const int64_t q = pr / nprobe;
  const int P0 = kc * TCKC + 16 * c16;
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  if (P0 < kp) {
    const int p64 = P0 >> 6, t4 = (P0 >> 4) & 3;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(qslices + (q * SLICES + d) * kp + 64 * p64 + 4 * t4);
    v = make_uint4(src[0], src[4], src[8], src[12]);
  }
  const int R = 4 * (slot & 1) + d;  // row inside the 8-row atom
  *reinterpret_cast<uint4*>(out + blk * 512 + d * 128 + (((c16 ^ R) & 7) << 4)) = v;
}

// The fused stage 1's B operand: out[kc][i] (128 bytes) = the quantized query row (qhat_kernel) of
// pair i, K bytes [128 kc, 128 kc + 128) in dimension order (the rcode byte order of 8-bit codes),
// pre-swizzled as row (slot & 7) of a 128B-swizzled 8-row atom; zero past the row.
__global__ void tc_qpairs_kernel(const int8_t* __restrict__ qhat, const int64_t* __restrict__ porder,
                                 const int32_t* __restrict__ pslot, int64_t npairs, int nprobe, int rowb, int nkc,
                                 int nib, int8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // one 16-byte chunk
  if (t >= npairs * nkc * 8) return;
  const int c16 = (int)(t & 7);
  const int64_t blk = t >> 3;  // (kc, i), kc major
  const int64_t i = blk % npairs;
  const int kc = (int)(blk / npairs);
  const int64_t pr = porder[i];
  const int32_t slot = pslot[pr];
  if (slot < 0) return;
  const int P0 = kc * TCKC + 16 * c16;
  uint4 v = make_uint4(0u, 0u, 0u, 0u);
  const int8_t* row = qhat + (pr / nprobe) * (int64_t)rowb;
  if (!nib) {
    if (P0 < rowb) v = *reinterpret_cast<const uint4*>(row + P0);
  } else {  // 4-bit codes: element P of the unpacked tile holds dimension refine_kdim(slice_pos(P))
    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int P = P0 + e;
      const int kk = (P & ~0x3C) | ((P & 0x0C) << 2) | ((P & 0x30) >> 2);
      const int dim = refine_kdim(kk, true);
      const uint32_t b = dim < rowb ? (uint32_t)(uint8_t)row[dim] : 0u;
      w[e >> 2] |= b << (8 * (e & 3));
    }
    v = make_uint4(w[0], w[1], w[2], w[3]);
  }
  const int R = slot & 7;
  *reinterpret_cast<uint4*>(out + blk * 128 + (((c16 ^ R) & 7) << 4)) = v;
}

__host__ __device__ inline uint32_t tmem_cols(int n) {  // power of two >= 32 (<= 512)
  return n <= 32 ? 32u : n <= 64 ? 64u : n <= 128 ? 128u : n <= 256 ? 256u : 512u;
}

__host__ __device__ inline int round16(int n) { return (n + 15) & ~15; }

// stage-1 fusion of the refine: 0 none, 1 bitwise (qhat rows), 2 LUT (the digit rows read as signed too)
size_t tc_smem_bytes(int kpad, int G, int nst, int fusion) {
  const int nkc = (kpad + TCKC - 1) / TCKC;
  return 1024 + (size_t)nkc * (TCR_DIG * G + (fusion == 1 ? round16(G) : 0)) * TCKC + (size_t)nst * TCM * TCKC +
         256 + 2 * 64 * sizeof(double4);
}

// accumulator columns of one tile: 4 digit columns per query, and the fused stage 1's sums
__host__ __device__ inline int tc_ncol(int G, int fusion) {
  return TCR_DIG * G + (fusion == 1 ? 2 * round16(G) : fusion == 2 ? TCR_DIG * G : 0);
}

#ifdef IVRQ_TCR_TRACE  // development builds only: timeline of CTA 0's roles (plain stores, no atomics)
__device__ unsigned long long g_tcr_trace[16 * 4096];
#define TCR_EV(tag, idx)                                                                       \
  do {                                                                                         \
    if (blockIdx.x == 0) g_tcr_trace[((tag) << 12) | ((idx) & 4095)] = (unsigned long long)clock64(); \
  } while (0)
#else
#define TCR_EV(tag, idx) ((void)0)
#endif

template <int FUSION>  // 0 none, 1 bitwise stage 1 (qhat rows), 2 LUT estimate (digit rows read as signed)
__global__ void __launch_bounds__(TCR_THREADS, 1) tc_refine_kernel(const __grid_constant__ TcArgs a) {
  extern __shared__ __align__(1024) unsigned char tsm_raw[];
  unsigned char* tsm = reinterpret_cast<unsigned char*>(((uintptr_t)tsm_raw + 1023) & ~(uintptr_t)1023);
  const int G = a.G, kp = a.kpad, NST = a.nst;
  const int nkc = (kp + TCKC - 1) / TCKC;  // 128-byte K chunks
  constexpr bool fused = FUSION == 1;
  constexpr bool lutf = FUSION == 2;
  const int G16 = round16(G);
  // one K chunk of the group's B rows: the digit rows (G/2 atoms; G even), then (fused) the qhat rows
  // (G16/8 atoms), placed right after the group's own digit rows so one MMA covers both
  const uint32_t bkc = (uint32_t)(G / 2) * 1024 + (fused ? (uint32_t)(G16 / 8) * 1024 : 0u);
  int8_t* sB = reinterpret_cast<int8_t*>(tsm);                                   // [nkc][bkc]
  uint8_t* sA = reinterpret_cast<uint8_t*>(sB + (size_t)nkc * bkc);             // [NST][128 rows x 128 B] swizzled
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + (size_t)NST * TCM * TCKC);
  uint64_t* full = bars;                      // [NST]
  uint64_t* empty = bars + NST;               // [NST]
  uint64_t* accf = bars + 2 * NST;            // [2]
  uint64_t* acce = bars + 2 * NST + 2;        // [2]
  uint64_t* bfull = bars + 2 * NST + 4;       // [1]
  uint64_t* bempty = bars + 2 * NST + 5;      // [1] the group's MMAs are done with sB
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(bars + 2 * NST + 6);
  double4* s_qs = reinterpret_cast<double4*>(bars + 2 * NST + 8);  // [2][64] (dq, kb, hs, row base) per group slot
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int NCOL = tc_ncol(G, fused ? 1 : lutf ? 2 : 0);  // accumulator columns of one tile
  // a whole warp waiting on an mbarrier: one lane polls, the warp then re-converges
  auto wait1 = [&](uint64_t* bar, uint32_t parity) {
    if (lane == 0) tc::mbar_wait(bar, parity);
    __syncwarp();
  };
  if (tid == 0) {
    for (int i = 0; i < NST; ++i) {
      tc::mbar_init(&full[i], a.nib ? 32 * TC_PROD : 1);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&accf[i], 1);
      tc::mbar_init(&acce[i], 32 * TCR_EPI);
    }
    tc::mbar_init(bfull, 1);
    tc::mbar_init(bempty, 1);
    tc::fence_mbar_init();
  }
  if (wid == TC_PROD) tc::tmem_alloc(s_taddr, tmem_cols(2 * NCOL));
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *s_taddr;
  const int64_t rb = a.ix.rcode_bytes;
  // the two accumulators start at aligned column halves of the allocation
  const uint32_t acc_stride = tmem_cols(2 * NCOL) / 2;
  uint32_t it_prod = 0, it_mma = 0, tile_mma = 0, tile_epi = 0, grp = 0;
  const int total = a.gpre[a.nlist];
  for (int b = blockIdx.x; b < total; b += gridDim.x, ++grp) {
    int lo_c = 0, hi_c = a.nlist;
    while (hi_c - lo_c > 1) {
      const int mid = (lo_c + hi_c) >> 1;
      if (a.gpre[mid] <= b) lo_c = mid; else hi_c = mid;
    }
    const int c = lo_c;
    const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
    const int64_t ps = a.poff[c] + (int64_t)(b - a.gpre[c]) * G;
    const int nqg = (int)min((int64_t)G, a.poff[c + 1] - ps);
    const int ntile = (int)ceil_div(n_c, TCM);
    if (wid == 1) {
      // the group operand (its digit rows, pre-swizzled in pair order: one bulk copy per K chunk),
      // issued once the previous group's MMAs no longer read sB
      wait1(bempty, (grp & 1) ^ 1);
      if (lane == 0) TCR_EV(7, grp);
      if (lane == 0) tc::mbar_expect_tx(bfull, (uint32_t)(nqg * nkc * (fused ? 640 : 512)));
      __syncwarp();
      if (lane < nkc)
        tc::bulk_load(sB + lane * bkc, a.bslices + ((int64_t)lane * a.npairs + ps) * 512, (uint32_t)nqg * 512, bfull,
                      tc::kL2EvictFirst);
      else if (fused && lane < 2 * nkc)  // after the group's 4 ((nqg + 3) & ~3) digit rows
        tc::bulk_load(sB + (lane - nkc) * bkc + (((nqg + 3) & ~3) >> 1) * 1024,
                      a.bqhat + ((int64_t)(lane - nkc) * a.npairs + ps) * 128, (uint32_t)nqg * 128, bfull,
                      tc::kL2EvictFirst);
    }
    if (wid < TC_PROD) {
      // ---- producers: rcode tiles -> A ring
      if (!a.nib) {
        if (tid == 0) {
          for (int t = 0; t < ntile; ++t)
            for (int kc = 0; kc < nkc; ++kc, ++it_prod) {
              const int st = it_prod % NST;
              tc::mbar_wait(&empty[st], ((it_prod / NST) & 1) ^ 1);
              TCR_EV(1, it_prod);
              tc::mbar_expect_tx(&full[st], TCM * TCKC);
              // evict-last: the list's other query groups re-read these rows from L2
              tc::tma_load_2d_hint(sA + st * TCM * TCKC, &a.map_a, kc * TCKC, (int)(lo + (int64_t)t * TCM), &full[st],
                                   tc::kL2EvictLast);
            }
        }
      } else {
        // two dims per byte: 8 bytes -> 16 elements [lo(0..3) hi(0..3) lo(4..7) hi(4..7)], swizzled
        // stores; the next stage's bytes are loaded before this stage's slot is awaited
        const int pl = wid * 32 + lane;
        const uint8_t* rows = a.ix.rcodes + lo * rb;
        constexpr int PER = TCM * (TCKC / 16) / (32 * TC_PROD);
        auto load_stage = [&](int sidx, uint2 (&x)[PER]) {
          const int t = sidx / nkc, kb0 = (sidx % nkc) * TCKC;
#pragma unroll
          for (int e = 0; e < PER; ++e) {
            const int i = pl + e * 32 * TC_PROD;
            const int r = i / (TCKC / 16), pc = 16 * (i % (TCKC / 16));
            const int64_t v = (int64_t)t * TCM + r;
            x[e] = (v < n_c && kb0 + pc < kp) ? __ldg(reinterpret_cast<const uint2*>(rows + v * rb + (kb0 + pc) / 2))
                                              : make_uint2(0u, 0u);
          }
        };
        const int nsx = ntile * nkc;
        uint2 xn[PER];
        if (nsx > 0) load_stage(0, xn);
        for (int sidx = 0; sidx < nsx; ++sidx, ++it_prod) {
          uint2 xc[PER];
#pragma unroll
          for (int e = 0; e < PER; ++e) xc[e] = xn[e];
          if (sidx + 1 < nsx) load_stage(sidx + 1, xn);
          const int st = it_prod % NST;
          tc::mbar_wait(&empty[st], ((it_prod / NST) & 1) ^ 1);
          uint8_t* dst = sA + st * TCM * TCKC;
#pragma unroll
          for (int e = 0; e < PER; ++e) {
            const int i = pl + e * 32 * TC_PROD;
            const int r = i / (TCKC / 16), pc = 16 * (i % (TCKC / 16));
            const uint2 x = xc[e];
            // fused stage 1: u << (8 - bits), so the code's MSB is the byte's sign bit (a.nib_hi = 8 - bits)
            const int sh = a.nib_hi;
            *reinterpret_cast<uint4*>(dst + sw128_offset(r, pc)) =
                make_uint4((x.x & 0x0F0F0F0Fu) << sh, ((x.x >> 4) & 0x0F0F0F0Fu) << sh, (x.y & 0x0F0F0F0Fu) << sh,
                           ((x.y >> 4) & 0x0F0F0F0Fu) << sh);
          }
          tc::fence_smem_async();
          tc::mbar_arrive(&full[st]);
        }
      }
    } else if (wid == TC_PROD) {
      // ---- MMA issuer.  N = the group's 4 digit rows per query, rounded to 16 (a list probed by
      // few queries does not pay for a full group)
      // one MMA for the digit rows (and the qhat rows after them: sum u qhat), one for sum s8(u) qhat
      const int ndig = TCR_DIG * ((nqg + 3) & ~3);
      const uint32_t idesc = tc::idesc_i8(TCM, ndig + (fused ? round16(nqg) : 0), false, true);
      const uint32_t idq_s = tc::idesc_i8(TCM, round16(nqg), true, true);
      const uint32_t idd_s = tc::idesc_i8(TCM, ndig, true, true);
      wait1(bfull, grp & 1);
      if (lane == 0) TCR_EV(4, grp);
      for (int t = 0; t < ntile; ++t, ++tile_mma) {
        const int ab = tile_mma & 1;
        wait1(&acce[ab], ((tile_mma >> 1) & 1) ^ 1);
        if (lane == 0) TCR_EV(3, tile_mma);
        tc::fence_after_sync();
        for (int kc = 0; kc < nkc; ++kc, ++it_mma) {
          const int st = it_mma % NST;
          wait1(&full[st], (it_mma / NST) & 1);
          tc::fence_after_sync();
          if (lane == 0) {
            TCR_EV(2, it_mma);
            const int ks = min(TCKC, kp - kc * TCKC) / 32;
            for (int s2 = 0; s2 < ks; ++s2) {
              const uint64_t ad = tc::smem_desc_sw128(sA + st * TCM * TCKC + 32 * s2);
              const uint64_t bd = tc::smem_desc_sw128(sB + kc * bkc + 32 * s2);
              tc::mma_i8(tbase + ab * acc_stride, ad, bd, idesc, kc > 0 || s2 > 0);
              if (fused) {
                const uint64_t qd = tc::smem_desc_sw128(sB + kc * bkc + (ndig >> 3) * 1024 + 32 * s2);
                tc::mma_i8(tbase + ab * acc_stride + TCR_DIG * G + G16, ad, qd, idq_s, kc > 0 || s2 > 0);
              } else if (lutf) {  // the digit rows against u read as signed bytes
                tc::mma_i8(tbase + ab * acc_stride + TCR_DIG * G, ad, bd, idd_s, kc > 0 || s2 > 0);
              }
            }
            TCR_EV(8, it_mma);
            tc::commit(&empty[st]);
            if (kc == nkc - 1) tc::commit(&accf[ab]);
          }
          __syncwarp();
        }
      }
      if (lane == 0) tc::commit(bempty);  // sB free once this group's MMAs retire
      __syncwarp();
    } else {
      // ---- epilogue: row r of the tile is TMEM lane r (a warp reads lane quarter wid % 4); the
      // TCR_EPQ warps of a quarter split the group's queries.  The group's per-query scalars are
      // staged in shared memory (slot parity = group parity) by the first epilogue warps and read
      // as broadcasts.
      const int quarter = wid & 3, part = (wid - (TC_PROD + 1)) >> 2;
      const int r = quarter * 32 + lane;
      const int64_t rs = ip_row_stride(n_c);
      double4* qs = s_qs + (grp & 1) * 64;
      const int et = tid - 32 * (TC_PROD + 1);  // 0 .. 32 TCR_EPI - 1
      if (et < nqg) {
        const int64_t pi = ps + et;
        const int64_t pr = a.porder[pi];
        const int64_t q = pr / a.nprobe;
        qs[et] = make_double4(a.probe_d2[pr], a.scalars[q * IVRQ_QS_COUNT + IVRQ_QS_KB_SUM],
                              ldexp(1.0, (int)a.scalars[q * IVRQ_QS_COUNT + IVRQ_QS_SLICE_EXP] - 26),
                              __longlong_as_double(a.pair_base[c] + (pi - a.poff[c]) * rs));
      }
      // the slots are rewritten two groups later, after every epilogue warp passed this group's
      // first accumulator wait; all epilogue warps meet here so the writes are visible
      asm volatile("bar.sync 1, %0;" ::"r"(32 * TCR_EPI) : "memory");
      for (int t = 0; t < ntile; ++t, ++tile_epi) {
        const int ab = tile_epi & 1;
        const int64_t v = (int64_t)t * TCM + r;
        float2 lf = make_float2(0.f, 0.f);
        if (v < n_c) lf = __ldg(reinterpret_cast<const float2*>(a.ix.long_factors) + lo + v);
        const double lfx = (double)lf.x, lfy = (double)lf.y;
        wait1(&accf[ab], (tile_epi >> 1) & 1);
        if (lane == 0 && wid == TC_PROD + 1) TCR_EV(5, tile_epi);
        tc::fence_after_sync();
        for (int j0 = 8 * part; j0 < nqg; j0 += 8 * TCR_EPQ) {  // 8-query chunks, round robin over the parts
          uint32_t d[32];
          const uint32_t trow = tbase + ((uint32_t)(quarter * 32) << 16) + ab * acc_stride;
          tc::tmem_ld32(trow + TCR_DIG * j0, d);
          uint32_t du[8], ds8[8], ds[32];
          if (fused) {
            tc::tmem_ld8(trow + TCR_DIG * ((nqg + 3) & ~3) + j0, du);
            tc::tmem_ld8(trow + TCR_DIG * G + G16 + j0, ds8);
          }
          if (lutf) tc::tmem_ld32(trow + TCR_DIG * G + TCR_DIG * j0, ds);
          tc::tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            const int j = j0 + jj;
            if (j < nqg && v < n_c) {
              const double4 sq = qs[j];
              const int* D = reinterpret_cast<const int*>(d + TCR_DIG * jj);
              // hi = (D0 128 + D1) 2^14 + (D2 128 + D3): the int32 pairs cannot overflow (|D_s| <= U 64 kpad,
              // the dense path's kpad <= 960 for 8-bit codes), hi < 2^47 is exact in float64.  The distance
              // add + d_qc2 + scale (kb - hi 2^(e-26)) in this order: three roundings of at most 2^-53 M
              // each, inside rd_radius_kernel's 2^-50 M
              // (codes of <= 4 bits with the fused stage 1 come in as u 2^(8 - bits): exact multiples)
              const int sh = a.nib_hi;
              const double hi = fma((double)((D[0] >> sh) * 128 + (D[1] >> sh)), 16384.0,
                                    (double)((D[2] >> sh) * 128 + (D[3] >> sh)));
              const double t = fma(-hi, sq.z, sq.y);
              const float rd = fmaxf((float)fma(lfy, t, lfx + sq.x), 0.f);
              const int64_t at = __double_as_longlong(sq.w) + v;
              if (FUSION == 0) {
                __stcs(a.rdist + at, rd);  // streaming store: written once, read once by the per-query pass
              } else {
                float ipf;
                if (fused) {
                  // sum u qhat - sum s8(u) qhat = 256 sum msb(u) qhat, exactly (an integer below 2^24)
                  ipf = (float)(((int)du[jj] - (int)ds8[jj]) >> 8);
                } else {
                  // sum_d msb(u) D_d = (sum u D_d - sum s8(u) D_d) / 256, exactly; <msb, q> up to the
                  // neglected digits (|.| <= kpad L 2^(e-54)), then rounded to float32
                  int m[4];
#pragma unroll
                  for (int dd = 0; dd < 4; ++dd) m[dd] = ((int)D[dd] - (int)ds[TCR_DIG * jj + dd]) >> 8;
                  ipf = (float)(fma((double)(m[0] * 128 + m[1]), 16384.0, (double)(m[2] * 128 + m[3])) * sq.z);
                }
                // (distance, stage-1 value) side by side: one 8-byte load per vector in the per-query pass
                __stcs(reinterpret_cast<float2*>(a.rdist) + at, make_float2(rd, ipf));
              }
            }
          }
        }
        if (lane == 0 && wid == TC_PROD + 1) TCR_EV(6, tile_epi);
        tc::fence_before_sync();
        tc::mbar_arrive(&acce[ab]);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == TC_PROD) tc::tmem_dealloc(tbase, tmem_cols(2 * NCOL));
}

// Per-query radius of the approximate refined distances written by tc_refine_kernel:
// |stored - exact| <= rrad[q] + |stored| 2^-23 for every vector of the query's probed lists.
// With e the query's slice exponent, the neglected digits D4..D7 of each dimension are at most
// L = 64 (128^3 + 128^2 + 128 + 1) = 135274560 in magnitude, so the neglected part of the inner
// product is at most U kpad L 2^(e-54) (U = the largest code value, 2^bits - 1); the exact path's own
// rounding of ip (|ip| <= U kpad 2^e) adds 2^-53 |ip|; through est2 = max(add + d_qc2 - scale (ip - kb), 0)
// that scales by |scale| <= S, plus the float64 roundings of both evaluations, each at most 2^-52 of
// M = |add| + d_qc2 + |scale| (|ip| + |kb|) (four operations).  lfmax = (max |add|, max |scale|) over the
// index, as float bit patterns.  One thread per query.
__global__ void rd_radius_kernel(const double* __restrict__ scalars, const double* __restrict__ probe_d2,
                                 const uint32_t* __restrict__ lfmax, int64_t nq, int nprobe, int kp, int umax,
                                 double* __restrict__ rrad) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double* sc = scalars + q * IVRQ_QS_COUNT;
  const int e = (int)sc[IVRQ_QS_SLICE_EXP];
  double dqm = 0.0;
  for (int p = 0; p < nprobe; ++p) dqm = fmax(dqm, probe_d2[q * nprobe + p]);
  const double A = (double)__uint_as_float(lfmax[0]), S = (double)__uint_as_float(lfmax[1]);
  const double U = (double)umax * (double)kp;
  const double ipmax = ldexp(U, e);
  const double trunc = S * (U * ldexp(135274560.0, e - 54) + ldexp(ipmax, -53));
  const double M = A + dqm + S * (ipmax + fabs(sc[IVRQ_QS_KB_SUM]));
  rrad[q] = (trunc + ldexp(M, -50)) * (1.0 + 0x1p-20);
}

// (add, scale, err) of every vector packed for one 16-byte load in the per-query pass
__global__ void pack_short_kernel(const float* __restrict__ add, const float* __restrict__ scale,
                                  const float* __restrict__ err, int64_t n, float4* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = make_float4(__ldg(add + i), __ldg(scale + i), __ldg(err + i), 0.f);
}

// lfmax[0] = max |add|, lfmax[1] = max |scale| over the long factors (float bit patterns of
// non-negative values order like the values, so an integer max is exact); lfmax zeroed by the caller
__global__ void lf_max_kernel(const float2* __restrict__ lf, int64_t n, uint32_t* __restrict__ lfmax) {
  uint32_t ma = 0u, ms = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float2 v = __ldg(lf + i);
    ma = max(ma, __float_as_uint(fabsf(v.x)));
    ms = max(ms, __float_as_uint(fabsf(v.y)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ma = max(ma, __shfl_xor_sync(FULL, ma, o));
    ms = max(ms, __shfl_xor_sync(FULL, ms, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(lfmax, ma);
    atomicMax(lfmax + 1, ms);
  }
}

// ------------------------------------------------------------ stage-1 inner products on tcgen05
// The binary inner products ip = <bit_v, qhat_q> of every probed (list,
// query) pair (ip_list_kernel's integer, search.py:163-183), list-major on
// the 5th-generation tensor cores: A = the list's 1-bit codes expanded to
// 0/1 bytes by the producer warps (128 vectors x 128 dims per stage, written
// in the 128B-swizzled K-major layout), B = the group's quantized queries in
// pair order (one TMA box of up to 256 rows per 128-dim chunk), accumulator
// 128 x N int32 in TMEM, epilogue writes the int16/int32 inner products.
constexpr int IPQ_MAX = 256;  // queries per group (N <= 256), fewer when the group's qhat rows exceed ~120 KB

inline int ip_group_size(int g) {
  int q = (120 * 1024) / (32 * g);
  q = q > IPQ_MAX ? IPQ_MAX : q;
  return q < 16 ? 16 : q & ~15;
}

struct TcIpArgs {
  CUtensorMap map_b;        // qhat in pair order [npairs rows x 32 g], box 128 B x IPQ rows
  ivrq_index_view ix;
  int g, nlist, ip32, ipq;
  const int64_t* poff;      // [nlist + 2]
  const int64_t* pair_base; // [nlist + 1]
  const int32_t* gpre;      // [nlist + 1] prefix of ceil(bucket / ipq)
  void* ipbuf;
};

size_t tc_ip_smem_bytes(int g) {
  const int nkc = (32 * g + TCKC - 1) / TCKC;
  return 1024 + (size_t)nkc * ip_group_size(g) * TCKC + (size_t)TCST * TCM * TCKC + 256;
}

// qhat rows gathered into pair order: out[i] = qhat[porder[i] / nprobe] (the first total pairs)
__global__ void qhat_pairs_kernel(const int8_t* __restrict__ qhat, const int64_t* __restrict__ porder,
                                  const int64_t* __restrict__ poff, int nlist, int nprobe, int rowb,
                                  int8_t* __restrict__ out) {
  const int64_t npairs = poff[nlist];
  const int per = rowb / 16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npairs * per; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per;
    const int c16 = (int)(i % per);
    const int64_t q = porder[r] / nprobe;
    reinterpret_cast<uint4*>(out + r * rowb)[c16] = reinterpret_cast<const uint4*>(qhat + q * rowb)[c16];
  }
}

__global__ void __launch_bounds__(TC_THREADS, 1) tc_ip_kernel(const __grid_constant__ TcIpArgs a) {
  extern __shared__ __align__(1024) unsigned char ism_raw[];
  unsigned char* ism = reinterpret_cast<unsigned char*>(((uintptr_t)ism_raw + 1023) & ~(uintptr_t)1023);
  const int g = a.g, kb_total = 32 * g, IPQ = a.ipq;
  const int nkc = (kb_total + TCKC - 1) / TCKC;
  int8_t* sB = reinterpret_cast<int8_t*>(ism);                                   // [nkc][IPQ rows x 128 B]
  uint8_t* sA = reinterpret_cast<uint8_t*>(ism + (size_t)nkc * IPQ * TCKC);      // [TCST][128 rows x 128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + TCST * TCM * TCKC);
  uint64_t* full = bars;
  uint64_t* empty = bars + TCST;
  uint64_t* accf = bars + 2 * TCST;
  uint64_t* acce = bars + 2 * TCST + 2;
  uint64_t* bfull = bars + 2 * TCST + 4;
  uint64_t* bempty = bars + 2 * TCST + 5;  // the group's MMAs are done with sB
  uint32_t* s_taddr = reinterpret_cast<uint32_t*>(bars + 2 * TCST + 6);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < TCST; ++i) {
      tc::mbar_init(&full[i], 32 * TC_PROD);
      tc::mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&accf[i], 1);
      tc::mbar_init(&acce[i], 128);
    }
    tc::mbar_init(bfull, 1);
    tc::mbar_init(bempty, 1);
    tc::fence_mbar_init();
  }
  if (wid == TC_PROD) tc::tmem_alloc(s_taddr, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *s_taddr;
  uint32_t it_prod = 0, it_mma = 0, tile_mma = 0, tile_epi = 0, grp = 0;
  const int total = a.gpre[a.nlist];
  for (int b = blockIdx.x; b < total; b += gridDim.x, ++grp) {
    int lo_c = 0, hi_c = a.nlist;
    while (hi_c - lo_c > 1) {
      const int mid = (lo_c + hi_c) >> 1;
      if (a.gpre[mid] <= b) lo_c = mid; else hi_c = mid;
    }
    const int c = lo_c;
    const int64_t lo = a.ix.offsets[c], n_c = a.ix.offsets[c + 1] - lo;
    const int64_t ps = a.poff[c] + (int64_t)(b - a.gpre[c]) * IPQ;
    const int nqg = (int)min((int64_t)IPQ, a.poff[c + 1] - ps);
    const int N = (nqg + 15) & ~15;
    const int64_t rs = ip_row_stride(n_c);
    const int ntile = (int)ceil_div(n_c, TCM);
    // no CTA barrier between groups: the MMA warp reloads B once the previous group's MMAs retire
    // (bempty) while the producers keep filling the A ring and the epilogue drains the last tiles
    if (wid < TC_PROD) {
      // ---- producers: code words -> 0/1 bytes, swizzled (each thread: row r, one word = 32 dims = 2 x 16 B)
      const int pl = wid * 32 + lane;
      const uint32_t* words = a.ix.packed_msb + (int64_t)g * lo;
      constexpr int PER = TCM * (TCKC / 32) / (32 * TC_PROD);  // words per producer thread per stage
      // consecutive lanes -> consecutive vectors (coalesced); the next stage's words are loaded
      // before this stage's slot is awaited, so the load latency overlaps the pipeline
      auto load_stage = [&](int sidx, uint32_t (&w)[PER]) {
        const int t = sidx / nkc, kc = sidx % nkc;
#pragma unroll
        for (int e = 0; e < PER; ++e) {
          const int i = pl + e * 32 * TC_PROD;
          const int r = i % TCM, jw = i / TCM;
          const int gi = kc * (TCKC / 32) + jw;
          const int64_t v = (int64_t)t * TCM + r;
          w[e] = (v < n_c && gi < g) ? __ldg(words + (int64_t)gi * n_c + v) : 0u;
        }
      };
      const int nst = ntile * nkc;
      // words of the next PF stages in flight (registers): one load round trip per PF stages
      constexpr int PF = 4;
      uint32_t wq[PF][PER];
#pragma unroll
      for (int j = 0; j < PF; ++j)
        if (j < nst) load_stage(j, wq[j]);
      for (int s0 = 0; s0 < nst; s0 += PF) {
#pragma unroll
      for (int j = 0; j < PF; ++j) {
        const int sidx = s0 + j;
        if (sidx >= nst) break;
        uint32_t wc[PER];
#pragma unroll
        for (int e = 0; e < PER; ++e) wc[e] = wq[j][e];
        if (sidx + PF < nst) load_stage(sidx + PF, wq[j]);
        {
          const int st = it_prod % TCST;
          tc::mbar_wait(&empty[st], ((it_prod / TCST) & 1) ^ 1);
          uint8_t* dst = sA + st * TCM * TCKC;
#pragma unroll
          for (int e = 0; e < PER; ++e) {
            const int i = pl + e * 32 * TC_PROD;
            const int r = i % TCM, jw = i / TCM;
            const uint32_t w = wc[e];
            uint4 o0, o1;
            o0.x = nib_bytes(w, 0);
            o0.y = nib_bytes(w, 4);
            o0.z = nib_bytes(w, 8);
            o0.w = nib_bytes(w, 12);
            o1.x = nib_bytes(w, 16);
            o1.y = nib_bytes(w, 20);
            o1.z = nib_bytes(w, 24);
            o1.w = nib_bytes(w, 28);
            *reinterpret_cast<uint4*>(dst + sw128_offset(r, 32 * jw)) = o0;
            *reinterpret_cast<uint4*>(dst + sw128_offset(r, 32 * jw + 16)) = o1;
          }
          tc::fence_smem_async();
          tc::mbar_arrive(&full[st]);
        }
        ++it_prod;
      }
      }
    } else if (wid == TC_PROD) {
      // ---- MMA issuer
      const uint32_t idesc = tc::idesc_i8(TCM, N, false, true);
      tc::mbar_wait(bempty, (grp & 1) ^ 1);
      if (lane == 0) {  // B: the group's qhat rows (contiguous in pair order)
        tc::mbar_expect_tx(bfull, (uint32_t)(nkc * IPQ * TCKC));
        for (int kc = 0; kc < nkc; ++kc) tc::tma_load_2d(sB + kc * IPQ * TCKC, &a.map_b, kc * TCKC, (int)ps, bfull);
      }
      __syncwarp();
      tc::mbar_wait(bfull, grp & 1);
      for (int t = 0; t < ntile; ++t, ++tile_mma) {
        const int ab = tile_mma & 1;
        tc::mbar_wait(&acce[ab], ((tile_mma >> 1) & 1) ^ 1);
        tc::fence_after_sync();
        for (int kc = 0; kc < nkc; ++kc, ++it_mma) {
          const int st = it_mma % TCST;
          tc::mbar_wait(&full[st], (it_mma / TCST) & 1);
          tc::fence_after_sync();
          if (lane == 0) {
            const int ks = min(TCKC, kb_total - kc * TCKC) / 32;
            for (int s2 = 0; s2 < ks; ++s2) {
              const uint64_t ad = tc::smem_desc_sw128(sA + st * TCM * TCKC + 32 * s2);
              const uint64_t bd = tc::smem_desc_sw128(sB + kc * IPQ * TCKC + 32 * s2);
              tc::mma_i8(tbase + ab * IPQ, ad, bd, idesc, kc > 0 || s2 > 0);
            }
            tc::commit(&empty[st]);
            if (kc == nkc - 1) tc::commit(&accf[ab]);
          }
          __syncwarp();
        }
      }
      if (lane == 0) tc::commit(bempty);  // sB free once this group's MMAs retire
      __syncwarp();
    } else {
      // ---- epilogue: TMEM lane r = vector, column j = query slot
      const int quarter = wid & 3;
      const int r = quarter * 32 + lane;
      for (int t = 0; t < ntile; ++t, ++tile_epi) {
        const int ab = tile_epi & 1;
        const int64_t v = (int64_t)t * TCM + r;
        tc::mbar_wait(&accf[ab], (tile_epi >> 1) & 1);
        tc::fence_after_sync();
        for (int j0 = 0; j0 < nqg; j0 += 32) {
          uint32_t d[32];
          tc::tmem_ld32(tbase + ((uint32_t)(quarter * 32) << 16) + ab * IPQ + j0, d);
          tc::tmem_ld_wait();
          if (v < n_c) {
            const int jn = min(32, nqg - j0);
            if (a.ip32) {
              int32_t* base = reinterpret_cast<int32_t*>(a.ipbuf) + a.pair_base[c] + (ps - a.poff[c] + j0) * rs + v;
              for (int jj = 0; jj < jn; ++jj) base[jj * rs] = (int32_t)d[jj];
            } else {
              int16_t* base = reinterpret_cast<int16_t*>(a.ipbuf) + a.pair_base[c] + (ps - a.poff[c] + j0) * rs + v;
              for (int jj = 0; jj < jn; ++jj) base[jj * rs] = (int16_t)(int32_t)d[jj];
            }
          }
        }
        tc::fence_before_sync();
        tc::mbar_arrive(&acce[ab]);
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == TC_PROD) tc::tmem_dealloc(tbase, 512);
}

// first probed list of each query inside this shard's id range (ids ascend per query)
__global__ void first_probe_kernel(const int64_t* __restrict__ probe_ids, int64_t nq, int nprobe, int64_t list_lo,
                                   int64_t list_hi, int32_t* __restrict__ first) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int32_t f = (int32_t)(list_hi - list_lo);  // bucket "no list of this shard"
  for (int p = 0; p < nprobe; ++p) {
    const int64_t c = probe_ids[q * nprobe + p];
    if (c >= list_lo && c < list_hi) {
      f = (int32_t)(c - list_lo);
      break;
    }
  }
  first[q] = f;
}

// Merge `parts` per-query top-k lists (each ascending by (dist, id), counts
// given) into the k best -- the all-gather merge of list-sharded search
// (merge_topk, search.py:378-387).  One thread per query.
__global__ void merge_topk_kernel(const int64_t* __restrict__ ids, const double* __restrict__ dists,
                                  const int32_t* __restrict__ counts, int64_t nq, int parts, int k,
                                  int64_t* __restrict__ out_ids, double* __restrict__ out_dists,
                                  int32_t* __restrict__ out_counts) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int head[16];
  for (int p = 0; p < parts; ++p) head[p] = 0;
  int n = 0;
  while (n < k) {
    int best = -1;
    double bd = 0.0;
    int64_t bi = 0;
    for (int p = 0; p < parts; ++p) {
      const int64_t base = ((int64_t)p * nq + q) * k;
      if (head[p] >= counts[(int64_t)p * nq + q]) continue;
      const double d = dists[base + head[p]];
      const int64_t i = ids[base + head[p]];
      if (best < 0 || key_less(d, i, bd, bi)) {
        best = p;
        bd = d;
        bi = i;
      }
    }
    if (best < 0) break;
    ++head[best];
    out_ids[q * k + n] = bi;
    out_dists[q * k + n] = bd;
    ++n;
  }
  for (int i = n; i < k; ++i) {
    out_ids[q * k + i] = -1;
    out_dists[q * k + i] = dinf();
  }
  out_counts[q] = n;
}

template <bool REFINE, bool NIB>
int launch_warp(const Args& a, int ipb, cudaStream_t s);
template <int MODE>
int launch_mode(const Args& a, bool refine, bool nib, int ipb, cudaStream_t s);

inline int launch_rd(const Args& a, bool refine, int ipb, cudaStream_t s) {
  // 4 sub-chunks of 32 vectors per batch, register budget for 6 resident CTAs (B200 A/B: 1, 6, 8)
  if (!refine) {
    auto kern = ipb == 2 ? scan_rd_kernel<2, 4, 6> : scan_rd_kernel<4, 4, 6>;
    KernelTimer kt("scan_rd_kernel", s);
    kern<<<(unsigned)ceil_div(a.nq, RDW), RDW * 32, 0, s>>>(a);
    return check_launch("ivrq_search_scan");
  }
#ifndef RDA_MINB
#define RDA_MINB 4
#endif
#ifndef RDA_RSUB
#define RDA_RSUB 4
#endif
  auto kern = a.sf4 ? (ipb == 0 ? scan_rda_kernel<0, RDA_RSUB, RDA_MINB> : scan_rda_kernel<1, RDA_RSUB, RDA_MINB>)
                     : (ipb == 2 ? scan_rda_kernel<2, RDA_RSUB, RDA_MINB> : scan_rda_kernel<4, RDA_RSUB, RDA_MINB>);
  const size_t sm = (size_t)RDW * ((size_t)a.kpad * sizeof(int2) + 32 * 16);
  if (sm > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return fail(IVRQ_EUNSUP, "ivrq_search_scan: shared memory request too large");
  // the digit tables are shared memory per warp: ask for the full carveout so the register budget
  // (6 CTAs per SM), not the L1/shared split, sets the residency
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  {
    KernelTimer kt("scan_rd_kernel", s);
    // persistent: RDA_MINB CTAs per SM take query slots from a.rda_next
    const int64_t blocks = a.rda_next ? std::min<int64_t>(ceil_div(a.nq, RDW), (int64_t)RDA_MINB * sm_count_of_current_device())
                                      : ceil_div(a.nq, RDW);
    kern<<<(unsigned)blocks, RDW * 32, sm, s>>>(a);
  }
  IVRQ_TRY(check_launch("ivrq_search_scan"));
  {
    const size_t fsm = (size_t)a.kpad * sizeof(int2) + 32 * 16;
    if (fsm > 48 * 1024 &&
        cudaFuncSetAttribute(rda_final_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm) != cudaSuccess)
      return fail(IVRQ_EUNSUP, "ivrq_search_scan: shared memory request too large");
    rda_final_kernel<<<(unsigned)a.nq, FIN_W * 32, fsm, s>>>(a);
    IVRQ_TRY(check_launch("ivrq_search_scan(final exact top k)"));
  }
#ifdef IVRQ_RDA_STATS
  {
    unsigned long long h[6];
    cudaMemcpyFromSymbolAsync(h, g_rda_stats, sizeof(h), 0, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    fprintf(stderr, "[rda] queries %llu prune-resolutions %llu exact-values %llu mean rq/T %.3g reruns %llu\n", h[2],
            h[0], h[1], h[2] ? h[3] * 1e-12 / h[2] : 0.0, h[4]);
    static const unsigned long long zero[6] = {};
    cudaMemcpyToSymbolAsync(g_rda_stats, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, s);
  }
#endif
  // the exact rerun of the queries the approximate pass could not certify (normally none: the
  // grid's warps return at once)
  Args f = a;
  f.fix_only = a.fix_list;
  f.fix_only_count = a.fix_count;
  f.init_ids = a.init_ids;
  if (a.sf4) {  // fused stage 1 (no inner products in ipbuf): the per-query scan, stage 1 from the
    f.ipbuf = nullptr;  // planes or tables, exact throughout
    f.sf4 = nullptr;
    return ipb == 0 ? launch_mode<IVRQ_IP_LUT>(f, true, rcode_nibbles(a.ix.bits), 0, s)
                    : launch_mode<IVRQ_IP_BITWISE>(f, true, rcode_nibbles(a.ix.bits), 0, s);
  }
  return rcode_nibbles(a.ix.bits) ? launch_warp<true, true>(f, ipb, s) : launch_warp<true, false>(f, ipb, s);
}

template <bool REFINE, bool NIB>
int launch_warp(const Args& a, int ipb, cudaStream_t s) {
  const size_t sm = warp_smem_bytes(a.kpad, REFINE);
  // wide rows (D >= 1024: the digit slices take ~12 KB of shared memory per warp) trade residency
  // for registers: C5 (D = 1536) scan 15.4 ms at 6 vs 16.8 at 8; C4 (D = 96) 8.6 at 8 vs 10.0 at 6
  auto kern = a.kpad >= 1024 ? (ipb == 2 ? scan_warp_kernel<REFINE, NIB, 2, 6> : scan_warp_kernel<REFINE, NIB, 4, 6>)
                             : (ipb == 2 ? scan_warp_kernel<REFINE, NIB, 2, WQ_MINB>
                                         : scan_warp_kernel<REFINE, NIB, 4, WQ_MINB>);
  if (sm > 48 * 1024 && cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess)
    return fail(IVRQ_EUNSUP, "ivrq_search_scan: shared memory request too large");
  {
    KernelTimer kt("scan_warp_kernel", s);
    kern<<<(unsigned)ceil_div(a.nq, WQ), WQ * 32, sm, s>>>(a);
  }
  return check_launch("ivrq_search_scan");
}

template <int MODE, bool REFINE, bool NIB>
int launch_t(const Args& a, int ipb, cudaStream_t s) {
  const bool bigk = a.k > 32;
  if (ipb < 0) return launch_warp<REFINE, NIB>(a, -ipb, s);  // warp-per-query path
  const size_t sm = smem_bytes(a, MODE, REFINE, bigk);
  const bool qb4 = MODE == IVRQ_IP_BITWISE && a.qbits == 4;  // the SearchParams default
  auto kern = bigk ? (qb4 ? scan_kernel_bigk<MODE, REFINE, NIB, 4> : scan_kernel_bigk<MODE, REFINE, NIB, 0>)
              : ipb == 2 ? scan_kernel<MODE, REFINE, NIB, 0, 2>
              : ipb == 4 ? scan_kernel<MODE, REFINE, NIB, 0, 4>
                         : (qb4 ? scan_kernel<MODE, REFINE, NIB, 4, 0> : scan_kernel<MODE, REFINE, NIB, 0, 0>);
  if (sm > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return fail(IVRQ_EUNSUP, "ivrq_search_scan: shared memory request too large");
  }
  kern<<<(unsigned)(a.fix_only ? std::min<int64_t>(a.nq, 2 * sm_count_of_current_device()) : a.nq), THREADS, sm, s>>>(a);
  return check_launch("ivrq_search_scan");
}

template <int MODE>
int launch_mode(const Args& a, bool refine, bool nib, int ipb, cudaStream_t s) {
  if (!refine) return launch_t<MODE, false, false>(a, ipb, s);
  return nib ? launch_t<MODE, true, true>(a, ipb, s) : launch_t<MODE, true, false>(a, ipb, s);
}

// Path selection.  Every path computes the reference's arithmetic exactly, so
// they return identical ids, distances and survivor counts (tests/
// test_gpu_parity.py::test_tensor_core_stage1_matches_popcount_path); the
// defaults are the measured fastest per configuration.  The
// environment variables only force a path, for those equivalence tests.
struct ScanPolicy {
  bool tc_path, warp_path, rd_path, first_phase, first_dist, tc_ip;
  bool lut_rd;  // LUT mode through the certified list-major path
};

static int env_flag(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

static ScanPolicy scan_policy(const ivrq_index_view& ix, const ivrq_search_params& p, bool refine, bool chained,
                              int64_t nl) {
  ScanPolicy sp{};
  // bitwise mode, k <= 32: stage-1 inner products list-major on the tensor cores, then one
  // warp per query (first lists included)
  sp.tc_path = p.ip_mode == IVRQ_IP_BITWISE && p.k <= 32 && env_flag("IVRQ_TC_STAGE1", 1) != 0 && nl >= 1;
  sp.warp_path = sp.tc_path && env_flag("IVRQ_WARP_SCAN", 1) != 0;
  // every probed pair refined list-major on tcgen05 (then a streaming per-query pass): dense
  // refine costs (probed vectors) x kpad MACs against (survivors) x kpad gathered by the in-warp
  // refine.  Measured on the B200 with the certified 4-digit refine (round 2): dense wins at D <= 768
  // for every code width (C3; C2 3.08 vs 3.37 ms per step, C4 9.65 vs 10.5); at D = 1536 (C5) the
  // survivor-only path.
  const int tr = env_flag("IVRQ_TC_REFINE", -1);
  const bool dense = tr >= 0 ? tr != 0 : kpad64(ix.dims) <= 768;
  // (the epilogue's int32 digit pairs D0 * 128 + D1 stay below 2^31 for kpad <= 960 with 8-bit codes)
  const bool fits = rcode_nibbles(ix.bits) || kpad64(ix.dims) <= 960;
  sp.rd_path = sp.warp_path && (!refine || (ix.rcodes && dense && fits));
  // LUT mode on the same list-major path for 8-bit codes: the refine's digit rows read as signed bytes
  // give a certified approximation of the LUT stage 1 (scan_rda_kernel<LUT>)
  if (p.ip_mode == IVRQ_IP_LUT && p.k <= 32 && refine && (ix.bits == 8 || rcode_nibbles(ix.bits)) && ix.rcodes &&
      dense && fits && nl >= 1 &&
      env_flag("IVRQ_TC_STAGE1", 1) != 0 && env_flag("IVRQ_LUT_RD", 1) != 0) {
    sp.tc_path = sp.warp_path = sp.rd_path = true;
    sp.lut_rd = true;
  }
  sp.first_phase = refine && p.k <= 32 && !chained && env_flag("IVRQ_FIRST_LIST", !sp.warp_path) != 0;
  sp.first_dist = sp.warp_path && !sp.rd_path && refine && !chained && env_flag("IVRQ_FIRST_DIST", 1) != 0;
  // tcgen05 stage 1 for long codes; mma.sync tiles win for short ones (D <= 224)
  sp.tc_ip = env_flag("IVRQ_TC_IP", words_per_vector(ix.dims) >= 8 ? 1 : 0) != 0;
  return sp;
}

// tc_refine group size and A ring depth: the largest query group (<= 64: 4 G accumulator columns,
// double-buffered in 512) whose digit rows fit beside a ring of >= TCR_MIN_ST A stages
#ifndef TCR_MIN_ST
#define TCR_MIN_ST 4
#endif
// (bitwise fusion: G a multiple of 8, so every group starts an 8-row atom of qhat rows; every fusion:
// its extra sums within the 512 columns)
static bool tc_refine_shape(int kpad, int fusion, int& G, int& nst) {
  const size_t cap = 227 * 1024;
  const int step = fusion == 1 ? 8 : 4;
#ifdef TCR_FORCE_G  // development A/B builds only
  G = TCR_FORCE_G;
  for (nst = 10; nst >= 2; --nst)
    if (tc_smem_bytes(kpad, G, nst, fusion) <= cap && 2 * tc_ncol(G, fusion) <= 512) return true;
  return false;
#endif
  for (G = 64; G >= step; G -= step) {
    if (2 * tc_ncol(G, fusion) > 512) continue;
    for (nst = 10; nst >= TCR_MIN_ST; --nst)
      if (tc_smem_bytes(kpad, G, nst, fusion) <= cap) return true;
  }
  for (G = 64; G >= step; G -= step) {  // very wide rows: a shallower ring
    if (2 * tc_ncol(G, fusion) > 512) continue;
    for (nst = TCR_MIN_ST - 1; nst >= 2; --nst)
      if (tc_smem_bytes(kpad, G, nst, fusion) <= cap) return true;
  }
  return false;
}

}  // namespace scan
}  // namespace ivrq

using namespace ivrq;

extern "C" int ivrq_search_scan(const ivrq_index_view* index, const double* q_rot, const int64_t* probe_ids,
                                const double* probe_d2, const double* scalars, const uint32_t* planes,
                                const float* luts, const int8_t* qslices, int64_t nq,
                                const ivrq_search_params* params, int64_t* out_ids, double* out_dists,
                                int32_t* out_counts, int64_t* stats, void* stream) {
  const int64_t nl = index ? index->n_clusters : 0;
  return ivrq_search_scan_shard(index, 0, nl, q_rot, probe_ids, probe_d2, scalars, planes, luts, qslices, nq, params,
                                nullptr, nullptr, nullptr, out_ids, out_dists, out_counts, stats, stream);
}

extern "C" int ivrq_search_scan_shard(const ivrq_index_view* index, int64_t list_lo, int64_t list_hi,
                                      const double* q_rot, const int64_t* probe_ids, const double* probe_d2,
                                      const double* scalars, const uint32_t* planes, const float* luts,
                                      const int8_t* qslices, int64_t nq, const ivrq_search_params* params,
                                      const int64_t* init_ids, const double* init_dists,
                                      const int32_t* init_counts, int64_t* out_ids, double* out_dists,
                                      int32_t* out_counts, int64_t* stats, void* stream) {
  (void)q_rot;
  if (!index || !params) return fail(IVRQ_EINVAL, "ivrq_search_scan: null argument");
  if (list_hi - list_lo != index->n_clusters) return fail(IVRQ_EINVAL, "ivrq_search_scan: shard range mismatch");
  if (init_counts && (!init_ids || !init_dists)) return fail(IVRQ_EINVAL, "ivrq_search_scan: partial init pool");
  if (params->k < 1) return fail(IVRQ_EINVAL, "k must be >= 1");
  if (params->k > 4096) return fail(IVRQ_EUNSUP, "ivrq_search_scan: k > 4096 not supported");
  if (index->bits < 1 || index->bits > 8) return fail(IVRQ_EINVAL, "index bits out of range");
  if (nq == 0) return IVRQ_OK;
  const bool refine = params->refine && index->bits >= 2;
  if (refine && (!qslices || !index->rcodes)) return fail(IVRQ_EINVAL, "refine needs qslices and rcodes");
  scan::Args a{};
  a.ix = *index;
  a.probe_ids = probe_ids;
  a.probe_d2 = probe_d2;
  a.scalars = scalars;
  a.planes = planes;
  a.luts = luts;
  a.qslices = qslices;
  a.nq = nq;
  a.k = params->k;
  a.nprobe = params->n_probe;
  a.qbits = params->query_bits;
  a.prune = params->prune;
  a.list_lo = list_lo;
  a.list_hi = list_hi;
  a.init_ids = init_ids;
  a.init_dists = init_dists;
  a.init_counts = init_counts;
  a.g = words_per_vector(index->dims);
  a.kpad = kpad64(index->dims);
  int n2 = 1;
  while (n2 < scan::CHUNK + a.k) n2 <<= 1;
  a.sort_n = n2;
  a.out_ids = out_ids;
  a.out_dists = out_dists;
  a.out_counts = out_counts;
  a.stats = stats;
  a.l2_prefetch = 0;  // measured neutral
  const bool nib = rcode_nibbles(index->bits);
  cudaStream_t s = as_stream(stream);
  const int64_t nl = index->n_clusters;
  const scan::ScanPolicy pol = scan::scan_policy(*index, *params, refine, init_counts != nullptr, nl);
  Workspace ws(s);  // every scratch block below is freed when the call returns, on any path
  auto oom = [](const char* what) { return fail(IVRQ_ENOMEM, std::string("ivrq_search_scan: ") + what); };
  // Queries grouped by their first (lowest-id) probed list: that list is refined in full
  // (the threshold is still +inf), so neighbours in the grid share it through L2.  Results
  // do not depend on the order.
  int64_t *off = nullptr;
  if (nq > 1 && nl >= 1) {
    int32_t* first = nullptr;
    int64_t *cnt = nullptr, *order = nullptr;
    if (!ws.alloc(first, nq) || !ws.alloc(cnt, nl + 1) || !ws.alloc(off, nl + 2) || !ws.alloc(order, nq))
      return oom("workspace allocation failed");
    scan::first_probe_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, s>>>(probe_ids, nq, a.nprobe, list_lo, list_hi,
                                                                         first);
    IVRQ_TRY(check_launch("ivrq_search_scan(order)"));
    IVRQ_TRY(ivrq_counting_sort(first, nq, (int32_t)(nl + 1), cnt, off, order, stream));
    a.qorder = order;
    if (pol.first_phase) {
      int32_t* gpre = nullptr;
      int64_t* pool_ids = nullptr;
      double* pool_d = nullptr;
      int32_t* pool_n = nullptr;
      if (!ws.alloc(gpre, nl + 1) || !ws.alloc(pool_ids, nq * a.k) || !ws.alloc(pool_d, nq * a.k) ||
          !ws.alloc(pool_n, nq))
        return oom("workspace allocation failed");
      cudaMemsetAsync(pool_n, 0, nq * sizeof(int32_t), s);
      if (stats) cudaMemsetAsync(stats, 0, 2 * nq * sizeof(int64_t), s);
      scan::group_prefix_kernel<<<1, 1, 0, s>>>(off, (int)nl, gpre);
      scan::FArgs fa{};
      fa.ix = *index;
      fa.list_lo = list_lo;
      fa.list_hi = list_hi;
      fa.probe_ids = probe_ids;
      fa.probe_d2 = probe_d2;
      fa.nprobe = a.nprobe;
      fa.scalars = scalars;
      fa.qslices = qslices;
      fa.kpad = a.kpad;
      fa.qorder = order;
      fa.qoff = off;
      fa.gpre = gpre;
      fa.nlist = (int)nl;
      fa.k = a.k;
      fa.pool_ids = pool_ids;
      fa.pool_d = pool_d;
      fa.pool_n = pool_n;
      fa.stats = stats;
      const size_t fsm = (size_t)scan::QG * scan::SLICES * (a.kpad + scan::SPAD);
      auto fk = nib ? scan::first_list_kernel<true> : scan::first_list_kernel<false>;
      if (fsm > 48 * 1024 &&
          cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm) != cudaSuccess)
        return fail(IVRQ_EUNSUP, "ivrq_search_scan: dims too large for the first-list phase");
      fk<<<(unsigned)(ceil_div(nq, scan::QG) + nl), scan::THREADS, fsm, s>>>(fa);
      IVRQ_TRY(check_launch("ivrq_search_scan(first lists)"));
      a.init_ids = pool_ids;
      a.init_dists = pool_d;
      a.init_counts = pool_n;
      a.skip_first = 1;
    }
  }
  // first lists refined list-major for the warp-per-query kernel (run on the main stream,
  // concurrently with the stage-1 inner products on the side stream)
  std::function<int()> refine_launch;
  if (pol.first_dist && a.qorder) {
    int64_t *fbase = nullptr, *ftot = nullptr;
    int32_t* fgpre = nullptr;
    if (!ws.alloc(fbase, nl + 1) || !ws.alloc(fgpre, nl + 1) || !ws.alloc(ftot, 2))
      return oom("workspace allocation failed");
    scan::pair_plan_kernel<<<1, 1024, 0, s>>>(index->offsets, off, (int)nl, scan::FQ, fbase, fgpre, ftot);
    IVRQ_TRY(check_launch("ivrq_search_scan(first-list plan)"));
    int64_t tot[2] = {0, 0};
    if (index->max_list > 0) {
      tot[0] = nq * scan::ip_row_stride(index->max_list);  // one first-list row per query at most
    } else if (cudaMemcpyAsync(tot, ftot, sizeof(tot), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
               cudaStreamSynchronize(s) != cudaSuccess) {
      return fail(IVRQ_ECUDA, "ivrq_search_scan: first-list plan readback failed");
    }
    if (tot[0] > 0) {
      double* fdist = nullptr;
      if (!ws.alloc(fdist, (size_t)tot[0])) return oom("first-list distance buffer allocation failed");
      scan::FdArgs fa{};
      fa.ix = *index;
      fa.list_lo = list_lo;
      fa.probe_ids = probe_ids;
      fa.probe_d2 = probe_d2;
      fa.nprobe = a.nprobe;
      fa.nlist = (int)nl;
      fa.kpad = a.kpad;
      fa.scalars = scalars;
      fa.qslices = qslices;
      fa.qorder = a.qorder;
      fa.qoff = off;
      fa.fbase = fbase;
      fa.gpre = fgpre;
      fa.fdist = fdist;
      const size_t fsm = (size_t)scan::FQ * scan::SLICES * (a.kpad + scan::SPAD) +
                         2 * (size_t)scan::FROWS * (nib ? 32 : 64);
      auto fk = nib ? scan::first_dist_kernel<true> : scan::first_dist_kernel<false>;
      if (fsm > 48 * 1024 &&
          cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm) != cudaSuccess)
        return fail(IVRQ_EUNSUP, "ivrq_search_scan: dims too large for the first-list refine");
      refine_launch = [fk, fa, fsm, s]() {
        fk<<<(unsigned)(2 * sm_count_of_current_device()), scan::THREADS, fsm, s>>>(fa);
        return check_launch("ivrq_search_scan(first-list refine)");
      };
      a.fdist = fdist;
      a.fbase = fbase;
      a.qoff = off;
    }
  }
  // list-major stage-1 inner products on the int8 tensor cores (bitwise mode, k <= 32)
  int ipb = 0;
  const int64_t ipmax = (int64_t)words_per_vector(index->dims) * 32 << (params->query_bits - 1);
  if (pol.tc_path) {
    ipb = pol.lut_rd ? 4 : ipmax <= 32768 ? 2 : 4;  // LUT: float32 stage-1 estimates
    const int64_t npairs = nq * a.nprobe;
    const int excl = pol.rd_path     ? 0
                     : pol.warp_path ? (refine && !a.prune ? 2 : (refine && !init_counts ? 1 : 0))
                                     : (a.skip_first ? 1 : 0);
    int32_t *pkeys = nullptr, *pslot = nullptr, *tpre = nullptr;
    int64_t *pcnt = nullptr, *poff = nullptr, *porder = nullptr, *pbase = nullptr, *ptot = nullptr;
    if (!ws.alloc(pkeys, npairs) || !ws.alloc(pslot, npairs) || !ws.alloc(porder, npairs) ||
        !ws.alloc(pcnt, nl + 1) || !ws.alloc(poff, nl + 2) || !ws.alloc(pbase, nl + 1) || !ws.alloc(tpre, nl + 1) ||
        !ws.alloc(ptot, 2))
      return oom("workspace allocation failed");
    scan::pair_key_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, s>>>(probe_ids, nq, a.nprobe, list_lo, list_hi,
                                                                      excl, pkeys);
    IVRQ_TRY(check_launch("ivrq_search_scan(pair keys)"));
    IVRQ_TRY(ivrq_counting_sort(pkeys, npairs, (int32_t)(nl + 1), pcnt, poff, porder, stream));
    scan::pair_slot_kernel<<<(unsigned)ceil_div(npairs, 256), 256, 0, s>>>(porder, poff, pkeys, npairs,
                                                                          (int32_t)nl, pslot);
    scan::pair_plan_kernel<<<1, 1024, 0, s>>>(index->offsets, poff, (int)nl, scan::TQ, pbase, tpre, ptot);
    IVRQ_TRY(check_launch("ivrq_search_scan(pair plan)"));
    // ip buffer: bounded by every pair owning a row of the largest list (no host round trip)
    // while the buffers stay within 8 GiB of the 180 GB of HBM, else the exact total read back
    int64_t tot[2] = {0, 0};
    if (excl == 2) {
      tot[0] = 0;
    } else if (index->max_list > 0 &&
               npairs * scan::ip_row_stride(index->max_list) * (ipb + (pol.rd_path && refine ? 4 : 0)) <=
                   (int64_t(8) << 30)) {
      tot[0] = npairs * scan::ip_row_stride(index->max_list);
    } else if (cudaMemcpyAsync(tot, ptot, sizeof(tot), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
               cudaStreamSynchronize(s) != cudaSuccess) {
      return fail(IVRQ_ECUDA, "ivrq_search_scan: pair plan readback failed");
    }
    if (tot[0] > 0) {
      uint8_t* ipbuf = nullptr;
      int8_t* qhat = nullptr;
      // (the fused refine writes the stage-1 values beside its distances: no separate buffer)
      const bool fused_stage1 = pol.rd_path && refine && (index->bits == 8 || nib);
      if (!ws.alloc(ipbuf, fused_stage1 ? 16 : (size_t)tot[0] * ipb) || !ws.alloc(qhat, (size_t)nq * 32 * a.g))
        return oom("inner-product buffer allocation failed");
      // 8-bit codes: the stage-1 inner products come out of the refine's own MMAs (no separate pass;
      // msb(u) = u >> 7 is what the signed reading of the byte subtracts)
      const bool fused = pol.rd_path && refine && (index->bits == 8 || nib) && !pol.lut_rd;
      const int fusion = fused ? 1 : pol.lut_rd ? 2 : 0;
      if (pol.rd_path && refine) {
        // refined distance of every probed pair on tcgen05 (concurrent with the inner products):
        // one work item per (list, group of G queries probing it)
        int G = 0, nb = 0;
        if (!scan::tc_refine_shape(a.kpad, fusion, G, nb))
          return fail(IVRQ_EUNSUP, "ivrq_search_scan: dims too large for the tensor-core refine");
        float* rdist = nullptr;
        double* rrad = nullptr;
        int32_t *rgpre = nullptr, *fix = nullptr;
        uint32_t* lfmax = nullptr;
        int64_t* rscratch = nullptr;
        int8_t* tcsl = nullptr;
        const int nkc = (a.kpad + scan::TCKC - 1) / scan::TCKC;
        if (!ws.alloc(rdist, (size_t)tot[0] * (fusion ? 2 : 1)) || !ws.alloc(rgpre, nl + 1) ||
            !ws.alloc(rscratch, nl + 3) ||
            !ws.alloc(tcsl, (size_t)npairs * nkc * 512) || !ws.alloc(rrad, nq) || !ws.alloc(fix, nq + 2) ||
            !ws.alloc(lfmax, 2))
          return oom("refined-distance buffer allocation failed");
        if (index->size >= (int64_t(1) << 40) || a.nprobe >= (1 << 20))
          return fail(IVRQ_EUNSUP, "ivrq_search_scan: index or n_probe too large for the refine pass");
        scan::pair_plan_kernel<<<1, 1024, 0, s>>>(index->offsets, poff, (int)nl, G, rscratch, rgpre, rscratch + nl + 1);
        IVRQ_TRY(check_launch("ivrq_search_scan(refine plan)"));
        scan::tc_bpairs_kernel<<<(unsigned)ceil_div(npairs * nkc * 32, 256), 256, 0, s>>>(
            qslices, porder, pslot, npairs, a.nprobe, a.kpad, nkc, tcsl);
        cudaMemsetAsync(lfmax, 0, 2 * sizeof(uint32_t), s);
        cudaMemsetAsync(fix, 0, sizeof(int32_t), s);
        cudaMemsetAsync(fix + nq + 1, 0, sizeof(int32_t), s);
        scan::lf_max_kernel<<<(unsigned)(2 * sm_count_of_current_device()), 256, 0, s>>>(
            reinterpret_cast<const float2*>(index->long_factors), index->size, lfmax);
        scan::rd_radius_kernel<<<(unsigned)ceil_div(nq, 128), 128, 0, s>>>(
            scalars, probe_d2, lfmax, nq, a.nprobe, a.kpad, (1 << index->bits) - 1, rrad);
        IVRQ_TRY(check_launch("ivrq_search_scan(refine radius)"));
        a.rrad = rrad;
        a.fix_count = fix;
        a.fix_list = fix + 1;
        a.rda_next = fix + nq + 1;
        if (fusion) {  // the per-query pass reads (distance, stage-1 value) pairs and packed short factors
          float4* sf4 = nullptr;
          if (!ws.alloc(sf4, (size_t)index->size)) return oom("workspace allocation failed");
          scan::pack_short_kernel<<<(unsigned)(4 * sm_count_of_current_device()), 256, 0, s>>>(
              index->short_add, index->short_scale, index->short_err, index->size, sf4);
          a.sf4 = sf4;
        }
        if (!ws.alloc(a.fin_d, (size_t)nq * 32) || !ws.alloc(a.fin_e, (size_t)nq * 32))
          return oom("refined-distance buffer allocation failed");
        scan::TcArgs ta{};
        // A: the rcode rows (8-bit codes; 4-bit indexes are unpacked by the producer warps instead)
        if (!nib && !tc::make_tmap_u8_sw128(&ta.map_a, index->rcodes, (uint64_t)index->rcode_bytes,
                                            (uint64_t)index->size, (uint64_t)index->rcode_bytes, scan::TCKC,
                                            scan::TCM))
          return fail(IVRQ_ECUDA, "ivrq_search_scan: TMA tensor map encoding failed");
        ta.bslices = tcsl;
        ta.npairs = npairs;
        ta.ix = *index;
        ta.kpad = a.kpad;
        ta.G = G;
        ta.nst = nb;
        ta.nib = nib ? 1 : 0;
        ta.scalars = scalars;
        ta.probe_d2 = probe_d2;
        ta.nprobe = a.nprobe;
        ta.nlist = (int)nl;
        ta.porder = porder;
        ta.poff = poff;
        ta.pair_base = pbase;
        ta.gpre = rgpre;
        ta.rdist = rdist;
        if (fused) {
          int8_t* qpairs4 = nullptr;
          if (!ws.alloc(qpairs4, (size_t)npairs * nkc * 128)) return oom("workspace allocation failed");
          scan::qhat_kernel<<<(unsigned)ceil_div(nq * a.g, 256), 256, 0, s>>>(planes, nq, a.g, a.qbits, qhat);
          scan::tc_qpairs_kernel<<<(unsigned)ceil_div(npairs * nkc * 8, 256), 256, 0, s>>>(
              qhat, porder, pslot, npairs, a.nprobe, 32 * a.g, nkc, nib ? 1 : 0, qpairs4);
          IVRQ_TRY(check_launch("ivrq_search_scan(fused stage-1 operand)"));
          ta.bqhat = qpairs4;
          ta.ipbuf = ipbuf;
          ta.ip32 = ipb == 4 ? 1 : 0;
        }
        if (pol.lut_rd) {
          ta.lut = 1;
          ta.ipbuf = ipbuf;
        }
        ta.nib_hi = (nib && fusion) ? 8 - index->bits : 0;
        const size_t tsm = scan::tc_smem_bytes(a.kpad, G, nb, fusion);
        auto rk = fusion == 1 ? scan::tc_refine_kernel<1> : fusion == 2 ? scan::tc_refine_kernel<2>
                                                                        : scan::tc_refine_kernel<0>;
        if (cudaFuncSetAttribute(rk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm) != cudaSuccess)
          return fail(IVRQ_EUNSUP, "ivrq_search_scan: dims too large for the tensor-core refine");
        refine_launch = [ta, tsm, s, rk]() {
          {
            KernelTimer kt("tc_refine_kernel", s);
            rk<<<(unsigned)sm_count_of_current_device(), scan::TCR_THREADS, tsm, s>>>(ta);
          }
#ifdef IVRQ_TCR_TRACE
          {
            static std::vector<unsigned long long> h(16 * 4096);
            cudaMemcpyFromSymbolAsync(h.data(), scan::g_tcr_trace, h.size() * 8, 0, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (const char* path = getenv("IVRQ_TCR_TRACE_OUT")) {
              if (FILE* f = fopen(path, "wb")) {
                fwrite(h.data(), 8, h.size(), f);
                fclose(f);
              }
            }
            cudaMemsetAsync(nullptr, 0, 0, s);
            void* sym = nullptr;
            cudaGetSymbolAddress(&sym, scan::g_tcr_trace);
            cudaMemsetAsync(sym, 0, h.size() * 8, s);
          }
#endif
          return check_launch("ivrq_search_scan(tensor-core refine)");
        };
        a.rdist = rdist;
      }
      if (fusion) {
        IVRQ_TRY(refine_launch());  // writes the stage-1 inner products (or LUT estimates) as well
        refine_launch = nullptr;
      } else
      {
        // fork: the stage-1 inner products on the side stream, the refine on s; both only read
        // the index and the prepared queries.  The fork joins on every return path.
        StreamFork fork(s, refine_launch ? side_stream() : nullptr);
        cudaStream_t si = fork.side();
        scan::qhat_kernel<<<(unsigned)ceil_div(nq * a.g, 256), 256, 0, si>>>(planes, nq, a.g, a.qbits, qhat);
        if (pol.tc_ip) {
          // stage-1 inner products on tcgen05: qhat rows gathered into pair order, then list-major GEMM tiles
          const int rowb = 32 * a.g;
          int8_t* qpairs = nullptr;
          int32_t* igpre = nullptr;
          int64_t* iscratch = nullptr;
          if (!ws.alloc(qpairs, (size_t)npairs * rowb, si) || !ws.alloc(igpre, nl + 1, si) ||
              !ws.alloc(iscratch, nl + 3, si))
            return oom("workspace allocation failed");
          const int ipq = scan::ip_group_size(a.g);
          scan::pair_plan_kernel<<<1, 1024, 0, si>>>(index->offsets, poff, (int)nl, ipq, iscratch, igpre,
                                                      iscratch + nl + 1);
          scan::qhat_pairs_kernel<<<(unsigned)(4 * sm_count_of_current_device()), 256, 0, si>>>(
              qhat, porder, poff, (int)nl, a.nprobe, rowb, qpairs);
          scan::TcIpArgs ta{};
          if (!tc::make_tmap_u8_sw128(&ta.map_b, qpairs, (uint64_t)rowb, (uint64_t)npairs, (uint64_t)rowb,
                                      scan::TCKC, ipq))
            return fail(IVRQ_ECUDA, "ivrq_search_scan: TMA tensor map encoding failed");
          ta.ix = *index;
          ta.g = a.g;
          ta.nlist = (int)nl;
          ta.ip32 = ipb == 4 ? 1 : 0;
          ta.ipq = ipq;
          ta.poff = poff;
          ta.pair_base = pbase;
          ta.gpre = igpre;
          ta.ipbuf = ipbuf;
          const size_t tsm = scan::tc_ip_smem_bytes(a.g);
          if (cudaFuncSetAttribute(scan::tc_ip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm) !=
              cudaSuccess)
            return fail(IVRQ_EUNSUP, "ivrq_search_scan: dims too large for the tensor-core stage 1");
          KernelTimer kt("tc_ip_kernel", si);
          scan::tc_ip_kernel<<<(unsigned)sm_count_of_current_device(), scan::TC_THREADS, tsm, si>>>(ta);
        } else {
          scan::IpArgs ia{};
          ia.ix = *index;
          ia.qhat = qhat;
          ia.g = a.g;
          ia.nprobe = a.nprobe;
          ia.nlist = (int)nl;
          ia.porder = porder;
          ia.poff = poff;
          ia.pair_base = pbase;
          ia.tpre = tpre;
          ia.ipbuf = ipbuf;
          const size_t ism =
              (size_t)scan::TQ * (32 * a.g + scan::TQ_PAD) + 2 * sizeof(uint32_t) * scan::KCH * scan::TV;
          auto ik = ipb == 2 ? scan::ip_list_kernel<int16_t> : scan::ip_list_kernel<int32_t>;
          if (ism > 48 * 1024 &&
              cudaFuncSetAttribute(ik, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ism) != cudaSuccess)
            return fail(IVRQ_EUNSUP, "ivrq_search_scan: dims too large for the tensor-core stage 1");
          KernelTimer kt("ip_list_kernel", si);
          ik<<<(unsigned)(2 * sm_count_of_current_device()), scan::THREADS, ism, si>>>(ia);
        }
        IVRQ_TRY(check_launch("ivrq_search_scan(stage-1 tiles)"));
        if (refine_launch) {
          IVRQ_TRY(refine_launch());
          refine_launch = nullptr;
        }
      }  // joined
      a.ipbuf = ipbuf;
      a.pslot = pslot;
      a.pair_base = pbase;
    }
  }
  if (refine_launch) IVRQ_TRY(refine_launch());
  if (pol.warp_path) {  // both warp kernels walk the per-probe metadata
    const int64_t np = nq * a.nprobe;
    int64_t *m_lo = nullptr, *m_base = nullptr;
    int32_t* m_nc = nullptr;
    if (!ws.alloc(m_lo, np) || !ws.alloc(m_base, np) || !ws.alloc(m_nc, np)) return oom("workspace allocation failed");
    scan::probe_meta_kernel<<<(unsigned)ceil_div(np, 256), 256, 0, s>>>(a, m_lo, m_nc, m_base);
    IVRQ_TRY(check_launch("ivrq_search_scan(probe metadata)"));
    a.m_lo = m_lo;
    a.m_nc = m_nc;
    a.m_base = m_base;
  }
  if (params->ip_mode == IVRQ_IP_BITWISE) {
    if (pol.rd_path && a.ipbuf) return scan::launch_rd(a, refine, ipb, s);
    return scan::launch_mode<IVRQ_IP_BITWISE>(a, refine, nib, pol.warp_path ? -ipb : ipb, s);
  }
  if (pol.lut_rd && a.ipbuf) return scan::launch_rd(a, refine, 0, s);  // ipb 0: float32 LUT estimates
  return scan::launch_mode<IVRQ_IP_LUT>(a, refine, nib, 0, s);
}

extern "C" int ivrq_merge_topk(const int64_t* ids, const double* dists, const int32_t* counts, int64_t nq,
                               int32_t parts, int32_t k, int64_t* out_ids, double* out_dists, int32_t* out_counts,
                               void* stream) {
  if (parts < 1 || parts > 16 || k < 1) return fail(IVRQ_EINVAL, "ivrq_merge_topk: parts must be in [1, 16]");
  if (nq == 0) return IVRQ_OK;
  scan::merge_topk_kernel<<<(unsigned)ceil_div(nq, 128), 128, 0, as_stream(stream)>>>(
      ids, dists, counts, nq, parts, k, out_ids, out_dists, out_counts);
  return check_launch("ivrq_merge_topk");
}
