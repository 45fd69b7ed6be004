// Search path: query rotation, coarse probe, query preparation and the fused
// two-stage list scan.  Reference: search.py (search_batch 390-454).
#include <algorithm>
#include <cstdlib>

#include "ivrq_common.cuh"
#include "ivrq_gemm.cuh"

namespace ivrq {

int probe_tc(const double* q_rot, int64_t nq, int32_t dims, const float* centroids, const double* centroid_sqnorms,
             int32_t n_clusters, int32_t n_probe, int32_t order_by_id, int64_t* ids, double* d2, const double* q_sq,
             cudaStream_t s);

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
                               uint32_t* __restrict__ planes, float* __restrict__ luts, int8_t* __restrict__ qslices,
                               int stage_rows) {
  extern __shared__ double prep_rows[];  // [warps][d] when launched with shared memory, else unused
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const double* xg = q_rot + q * d;
  const int g = words_per_vector(d);
  const double* x = xg;
  if (stage_rows) {  // the row is read coalesced into shared memory once; the serial pairwise sum below
                     // then walks shared memory instead of issuing dependent global loads
    double* row = prep_rows + (size_t)(threadIdx.x >> 5) * d;
    for (int i = lane; i < d; i += 32) row[i] = xg[i];
    __syncwarp();
    x = row;
  }
  double sum_q = 0.0;
  if (lane == 0) sum_q = pairwise_sum_seq(x, d);
  sum_q = __shfl_sync(0xffffffffu, sum_q, 0);
  {
    double l1 = 0.0;  // an upper bound of sum |q| (every partial sum rounded up)
    for (int i = lane; i < d; i += 32) l1 = __dadd_ru(l1, fabs(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l1 = __dadd_ru(l1, __shfl_xor_sync(0xffffffffu, l1, o));
    if (lane == 0) scalars[q * IVRQ_QS_COUNT + IVRQ_QS_L1] = l1;
  }
  const double k_b = ((double)((1 << index_bits) - 1)) / 2.0;
  double* sc = scalars + q * IVRQ_QS_COUNT;
  if (qslices) {
    // q_rot as Q * 2^(e-54), |Q| < 2^54, Q = sum_s D_s 128^(7-s) with balanced
    // digits D_s in [-64, 63]; stored per slice in the refine's K order.
    double mx = 0.0;
    for (int i = lane; i < d; i += 32) mx = dmax(mx, fabs(x[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = dmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
    const int kp = kpad64(d);
    const bool nib = rcode_nibbles(index_bits);
    int8_t* out = qslices + q * 8 * (int64_t)kp;
    for (int k = lane; k < kp; k += 32) {
      const int dim = refine_kdim(k, nib);
      long long Q = dim < d ? llrint(ldexp(x[dim], 54 - e)) : 0;
      for (int s = 7; s >= 0; --s) {
        const long long r = ((Q + 64) & 127) - 64;
        out[s * kp + k] = (int8_t)r;
        Q = (Q - r) >> 7;
      }
    }
    if (lane == 0) sc[IVRQ_QS_SLICE_EXP] = (double)e;
  }
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

template <typename TC>
static int probe_gemm_select(const double* q_rot, int64_t nq, int32_t dims, const TC* centroids,
                             const double* centroid_sqnorms, int32_t n_clusters, int32_t n_probe, int32_t order_by_id,
                             int64_t* ids, double* d2, double* dist, const double* q_sq, int64_t rows, cudaStream_t s);

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
  // path switch for tests (both paths select the same clusters): IVRQ_TC_PROBE=0 forces the float64 GEMM
  const bool tc_probe = getenv("IVRQ_TC_PROBE") ? atoi(getenv("IVRQ_TC_PROBE")) != 0 : true;
  if (tc_probe) {
    return probe_tc(q_rot, nq, dims, centroids, centroid_sqnorms, n_clusters, n_probe, order_by_id, ids, d2, q_sq, s);
  }
  return probe_gemm_select(q_rot, nq, dims, centroids, centroid_sqnorms, n_clusters, n_probe, order_by_id, ids, d2,
                           dist, q_sq, rows, s);
}

extern "C" int ivrq_select_clusters_f64(const double* q_rot, int64_t nq, int32_t dims, const double* centroids,
                                        const double* centroid_sqnorms, int32_t n_clusters, int32_t n_probe,
                                        int32_t order_by_id, int64_t* ids, double* d2, void* workspace,
                                        size_t workspace_bytes, void* stream) {
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
  return probe_gemm_select(q_rot, nq, dims, centroids, centroid_sqnorms, n_clusters, n_probe, order_by_id, ids, d2,
                           dist, q_sq, rows, s);
}

// float64 GEMM probe (DMMA) + exact selection, centroids of type TC
template <typename TC>
static int probe_gemm_select(const double* q_rot, int64_t nq, int32_t dims, const TC* centroids,
                             const double* centroid_sqnorms, int32_t n_clusters, int32_t n_probe, int32_t order_by_id,
                             int64_t* ids, double* d2, double* dist, const double* q_sq, int64_t rows,
                             cudaStream_t s) {
  gemm::RowMajor<TC> lb{centroids, n_clusters, dims};
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
                                    double* scalars, uint32_t* planes, float* luts, int8_t* qslices,
                                    void* stream) {
  if (!params) return fail(IVRQ_EINVAL, "ivrq_prepare_queries: null params");
  if (params->ip_mode == IVRQ_IP_BITWISE && (params->query_bits < 2 || params->query_bits > 8))
    return fail(IVRQ_EINVAL, "query_bits must be in [2, 8]");
  if (nq == 0) return IVRQ_OK;  // empty batches: the (empty) buffers may be null
  if (params->ip_mode == IVRQ_IP_BITWISE && !planes) return fail(IVRQ_EINVAL, "bitwise mode needs planes");
  if (params->ip_mode == IVRQ_IP_LUT && !luts) return fail(IVRQ_EINVAL, "lut mode needs luts");
  if (params->refine && index_bits >= 2 && !qslices) return fail(IVRQ_EINVAL, "refine needs qslices");
  // rows staged in shared memory (up to 48 KB per block: 4 warps at D <= 1536, fewer beyond)
  int wpb = 4;
  while (wpb > 1 && (size_t)wpb * dims * sizeof(double) > 48 * 1024) --wpb;
  const size_t psm = (size_t)wpb * dims * sizeof(double);
  const int stage = psm <= 48 * 1024 ? 1 : 0;
  prepare_kernel<<<(unsigned)ceil_div(nq, wpb), wpb * 32, stage ? psm : 0, as_stream(stream)>>>(
      q_rot, nq, dims, params->ip_mode, params->query_bits, index_bits, eps_bound, scalars, planes, luts,
      (params->refine && index_bits >= 2) ? qslices : nullptr, stage);
  return check_launch("ivrq_prepare_queries");
}

extern "C" int64_t ivrq_rcode_row_bytes(int32_t dims, int32_t bits) { return rcode_row_bytes_of(dims, bits); }
