// Build path: k-means++ seeding, Lloyd labelling/update, stable CSR assembly,
// residual normalisation + rotation and the warp-per-vector RaBitQ encoder.
// Reference: index.py build_index (190-281), clustering.py, codec.py.
#include <algorithm>
#include <cstdlib>
#include <functional>
#include <vector>

#include "ivrq_common.cuh"
#include "ivrq_gemm.cuh"
#include "ivrq_rowchain.cuh"

namespace ivrq {

template <typename T>
static int dalloc(T** p, size_t count, cudaStream_t s, const char* what) {
  if (count == 0) count = 1;
  cudaError_t e = pool_malloc(reinterpret_cast<void**>(p), count * sizeof(T), s);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(IVRQ_ENOMEM, std::string(what) + ": stream-ordered allocation failed");
  }
  return IVRQ_OK;
}

// ============================================================ k-means++ seeding
// d2[i] = einsum((x_i - c)^2) with c = centers[j] (float64 of an x row),
// optionally min-ed into the existing d2 (clustering.py:66-67, 77-78).
__global__ void __launch_bounds__(rowchain::THREADS) kpp_update_kernel(const float* __restrict__ x, int64_t n, int d,
                                                                       const double* __restrict__ center,
                                                                       double* __restrict__ d2, int init,
                                                                       const int* __restrict__ halt) {
  using namespace rowchain;
  if (halt && *halt) return;
  __shared__ Tile<float> tile;
  __shared__ double cs[CH];
  const int64_t row0 = (int64_t)blockIdx.x * ROWS;
  const int r = threadIdx.x >> 1, lane = threadIdx.x & 1;
  const bool vec = (d % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  auto src = [&](int64_t gr) { return x + gr * d; };
  double acc = 0.0;
  for (int c0 = 0; c0 < d; c0 += CH) {
    const int cw = min(CH, d - c0);
    __syncthreads();
    stage_tile(tile, src, row0, n, c0, cw, vec);
    if (threadIdx.x < CH) cs[threadIdx.x] = threadIdx.x < cw ? center[c0 + threadIdx.x] : 0.0;
    __syncthreads();
    acc = chain_chunk(acc, lane, cw, [&](int k) {
      const double df = dsub((double)tile.v[r][k], cs[k]);
      return dmul(df, df);
    });
  }
  const double v = finish(acc);
  if (lane == 0 && row0 + r < n) {
    if (init) d2[row0 + r] = v;
    else d2[row0 + r] = dmin(d2[row0 + r], v);  // np.minimum(d2, new, out=d2)
  }
}

// NumPy pairwise tree over d2: leaves are the <=128-element segments of the
// recursion (a function of n only), precomputed on the host.
__global__ void kpp_leaf_kernel(const double* __restrict__ d2, const int64_t* __restrict__ leaf_start,
                                const int32_t* __restrict__ leaf_len, int nleaf, double* __restrict__ node_val,
                                const int* __restrict__ halt) {
  if (halt && *halt) return;
  int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= nleaf) return;
  node_val[l] = pairwise_leaf(d2 + leaf_start[l], leaf_len[l]);
}

// ---- exact searchsorted(cumsum(d2), target) without the sequential walk (almost always)
// NumPy's cumsum S_i rounds after every addition; with d2 >= 0 it is monotone and
// |S_i - P_i| <= (i + 1) u S_i (u = 2^-53) against the exact prefix P_i.  The block
// computes P_i in double-double (error ~2^-100 P), finds the first i with P_i >=
// target, and accepts i when target lies outside the rounding band on both sides:
// P_i - target > band and target - P_{i-1} > band imply S_i >= target > S_{i-1},
// which is exactly NumPy's answer.  Otherwise (|target - P| within ~i 2^-52 P:
// vanishingly rare) the caller walks the sequential chain.
__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
}
struct DD {
  double hi, lo;
};
__device__ __forceinline__ DD dd_add(DD a, DD b) {
  double s, e;
  two_sum(a.hi, b.hi, s, e);
  e = __dadd_rn(e, __dadd_rn(a.lo, b.lo));
  double s2, e2;
  two_sum(s, e, s2, e2);
  return DD{s2, e2};
}
__device__ __forceinline__ DD dd_add1(DD a, double b) {
  double s, e;
  two_sum(a.hi, b, s, e);
  e = __dadd_rn(e, a.lo);
  double s2, e2;
  two_sum(s, e, s2, e2);
  return DD{s2, e2};
}
// a - b as a double (a, b double-double, a ~ b): accurate to ~2^-100 |a|
__device__ __forceinline__ double dd_diff(DD a, double b) { return __dadd_rn(__dsub_rn(a.hi, b), a.lo); }

__device__ bool kpp_fast_exact(const double* __restrict__ d2, int64_t n, double target, int64_t* out_idx,
                               double* s_hi /* shared, [2 * blockDim.x] */, const double* __restrict__ leaf_sum,
                               const int64_t* __restrict__ leaf_start, const int32_t* __restrict__ leaf_len,
                               int nleaf) {
  // Prefix over the pairwise-tree leaves (<= 128 contiguous elements each, their float64 sums already
  // computed by kpp_leaf_kernel, relative error <= 128 u), double-double accumulation, then the
  // crossing leaf walked element by element in double-double.  The band adds the leaf-sum error.
  double* s_lo = s_hi + blockDim.x;
  __shared__ int s_seg;
  __shared__ int s_ok;
  __shared__ int64_t s_res;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int per = (nleaf + nt - 1) / nt;
  const int l0 = tid * per, l1 = min(nleaf, l0 + per);
  DD t{0.0, 0.0};
  for (int l = l0; l < l1; ++l) t = dd_add1(t, leaf_sum[l]);
  s_hi[tid] = t.hi;
  s_lo[tid] = t.lo;
  if (tid == 0) {
    s_seg = nt;
    s_ok = 0;
    s_res = n - 1;
  }
  __syncthreads();
  for (int o = 1; o < nt; o <<= 1) {  // inclusive scan (Hillis-Steele, double-double)
    DD v{s_hi[tid], s_lo[tid]};
    if (tid >= o) v = dd_add(v, DD{s_hi[tid - o], s_lo[tid - o]});
    __syncthreads();
    s_hi[tid] = v.hi;
    s_lo[tid] = v.lo;
    __syncthreads();
  }
  const DD incl{s_hi[tid], s_lo[tid]};
  const DD excl = tid ? DD{s_hi[tid - 1], s_lo[tid - 1]} : DD{0.0, 0.0};
  const double total_hi = s_hi[nt - 1];
  const double leaf_err = 0x1p-44 * total_hi;  // >= 4 x 128 u x (sum of the leaves before the crossing)
  if (l0 < l1 && dd_diff(incl, target) >= 0.0 && dd_diff(excl, target) < 0.0) atomicMin(&s_seg, tid);
  __syncthreads();
  if (tid == s_seg) {
    DD run = excl;
    int L = l1 - 1;
    for (int l = l0; l < l1; ++l) {  // crossing leaf
      const DD nx = dd_add1(run, leaf_sum[l]);
      if (dd_diff(nx, target) >= 0.0) {
        L = l;
        break;
      }
      run = nx;
    }
    DD prev = run;
    int64_t hit = -1;
    const int64_t st = leaf_start[L];
    const int len = leaf_len[L];
    for (int i = 0; i < len; ++i) {
      prev = run;
      run = dd_add1(run, d2[st + i]);
      if (dd_diff(run, target) >= 0.0) {
        hit = st + i;
        break;
      }
    }
    if (hit >= 0) {
      const double band = (double)(hit + 2) * 0x1p-51 * run.hi + leaf_err + 0x1p-90 * total_hi;
      const double above = dd_diff(run, target), below = -dd_diff(prev, target);
      if (above > band && (hit == 0 || below > band)) {
        s_res = hit;
        s_ok = 1;
      }
    }
  } else if (tid == 0 && s_seg == nt) {
    const DD all{s_hi[nt - 1], s_lo[nt - 1]};
    const double band = (double)(n + 1) * 0x1p-51 * all.hi + leaf_err;
    if (-dd_diff(all, target) > band) {  // past the end: the reference's index is clamped to n - 1
      s_res = n - 1;
      s_ok = 1;
    }
  }
  __syncthreads();
  const bool ok = s_ok != 0;
  if (ok && tid == 0) *out_idx = s_res;
  __syncthreads();
  return ok;
}

// Combine the tree (internal nodes in increasing height order), compute
// target = r * total and searchsorted(cumsum(d2), target) with the sequential
// cumsum of NumPy (exact_scan) or a blocked scan for very large n; then copy
// the chosen row into centers[j].
__global__ void __launch_bounds__(1024) kpp_select_kernel(
    const float* __restrict__ x, int64_t n, int d, const double* __restrict__ d2, double* __restrict__ node_val,
    const int32_t* __restrict__ node_left, const int32_t* __restrict__ node_right,
    const int32_t* __restrict__ level_begin, int nlevels, int nleaf, int root, const double* __restrict__ draws,
    int draw_kind, int j, double* __restrict__ centers, int32_t* __restrict__ zero_step, int* __restrict__ halt,
    int exact_scan, double* __restrict__ block_sums, const int64_t* __restrict__ leaf_start,
    const int32_t* __restrict__ leaf_len) {
  __shared__ int64_t s_idx;
  __shared__ int s_stop;
  if (*halt) return;
  const int tid = threadIdx.x;
  if (draw_kind == 1) {
    if (tid == 0) s_idx = (int64_t)draws[j];
    __syncthreads();
  } else {
    for (int lv = 0; lv < nlevels; ++lv) {
      for (int nd = level_begin[lv] + tid; nd < level_begin[lv + 1]; nd += blockDim.x)
        node_val[nleaf + nd] = dadd(node_val[node_left[nd]], node_val[node_right[nd]]);
      __syncthreads();
    }
    const double total = dadd(0.0, node_val[root]);
    if (tid == 0) s_stop = 0;
    __syncthreads();
    if (!(total > 0.0)) {
      if (tid == 0) {
        atomicCAS(zero_step, -1, j);
        *halt = 1;
      }
      return;
    }
    const double target = dmul(draws[j], total);
    constexpr int SC = 2048;
    __shared__ double sbuf[2][SC];  // sequential walk staging; also the fast path's scan buffer
    if (exact_scan == 1 && kpp_fast_exact(d2, n, target, &s_idx, &sbuf[0][0], node_val, leaf_start, leaf_len, nleaf)) {
      // decided without the sequential walk (see kpp_fast_exact)
    } else if (exact_scan) {
      // NumPy's sequential cumsum, walked by one thread out of shared memory
      // while the rest of the block streams the next chunk in.
      __shared__ int s_found;
      if (tid == 0) {
        s_found = 0;
        s_idx = n - 1;
      }
      double cs = 0.0;
      for (int64_t i = tid; i < min((int64_t)SC, n); i += blockDim.x) sbuf[0][i] = d2[i];
      __syncthreads();
      int cur = 0;
      for (int64_t base = 0; base < n; base += SC) {
        const int64_t nb = base + SC;
        if (tid >= 32) {
          for (int64_t i = nb + tid - 32; i < min(nb + SC, n); i += blockDim.x - 32) sbuf[cur ^ 1][i - nb] = d2[i];
        } else if (tid == 0) {
          const int len = (int)min((int64_t)SC, n - base);
          const double* b = sbuf[cur];
          int hit = -1;
          // d2 >= 0 makes the running sum monotone: a branch-free pass over the
          // chunk decides whether the crossing lies inside it; only that chunk
          // is walked again with the compares.
          double end = cs;
#pragma unroll 8
          for (int i = 0; i < len; ++i) end = dadd(end, b[i]);
          if (end >= target) {
            for (int i = 0; i < len; ++i) {
              cs = dadd(cs, b[i]);
              if (cs >= target) { hit = i; break; }
            }
          } else {
            cs = end;
          }
          if (hit >= 0) {
            s_found = 1;
            s_idx = min(base + hit, n - 1);
          }
        }
        __syncthreads();
        if (s_found) break;
        cur ^= 1;
      }
    } else {
      // large n: a deterministic blocked cumsum (not NumPy's sequential
      // rounding): the pairwise-tree leaf sums (contiguous
      // <=128-element segments, already in node_val) are prefix-summed by the
      // block, the first leaf whose prefix reaches the target is found in
      // parallel, and that leaf is walked element by element.
      __shared__ double s_tot[1024];
      __shared__ int s_leaf;
      const int per = (nleaf + blockDim.x - 1) / blockDim.x;
      const int l0 = tid * per, l1 = min(nleaf, l0 + per);
      double t = 0.0;
      for (int l = l0; l < l1; ++l) t = dadd(t, node_val[l]);
      s_tot[tid] = t;
      if (tid == 0) s_leaf = nleaf;
      __syncthreads();
      if (tid == 0) {
        double run = 0.0;
        for (int i = 0; i < (int)blockDim.x; ++i) {
          const double v = s_tot[i];
          s_tot[i] = run;
          run = dadd(run, v);
        }
      }
      __syncthreads();
      double run = s_tot[tid];
      for (int l = l0; l < l1; ++l) {
        const double nx = dadd(run, node_val[l]);
        if (nx >= target) {
          atomicMin(&s_leaf, l);
          break;
        }
        run = nx;
      }
      __syncthreads();
      if (tid == 0) {
        const int L = s_leaf;
        int64_t idx = n - 1;
        if (L < nleaf) {
          const int tl = L / per;
          double cs = s_tot[tl];
          for (int l = tl * per; l < L; ++l) cs = dadd(cs, node_val[l]);
          const int64_t st = leaf_start[L];
          const int len = leaf_len[L];
          idx = st + len - 1;
          for (int i = 0; i < len; ++i) {
            cs = dadd(cs, d2[st + i]);
            if (cs >= target) {
              idx = st + i;
              break;
            }
          }
        }
        s_idx = idx < n - 1 ? idx : n - 1;
      }
      (void)block_sums;
    }
    __syncthreads();
  }
  const int64_t idx = s_idx;
  for (int k = tid; k < d; k += blockDim.x) centers[(int64_t)j * d + k] = (double)x[idx * d + k];
}

// ============================================================ labels
struct LabelDist {
  const double* x_sq;
  const double* c_sq;
  __device__ __forceinline__ double operator()(int64_t r, int64_t c, double dot) const {
    return dsub(dadd(x_sq[r], c_sq[c]), dmul(2.0, dot));
  }
};

// ============================================================ counting sort
constexpr int CS_THREADS = 256;

// Per tile: local count per label and each row's rank among equal labels in
// row order (warp-synchronous match over 32-row steps keeps it stable).
__global__ void cs_local_kernel(const int32_t* __restrict__ labels, int64_t n, int k, int64_t tile,
                                int32_t* __restrict__ tcount, int32_t* __restrict__ rank) {
  extern __shared__ int32_t cnt[];  // [k]
  const int64_t t = blockIdx.x;
  for (int c = threadIdx.x; c < k; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int64_t r0 = t * tile, r1 = min(n, r0 + tile);
    for (int64_t rb = r0; rb < r1; rb += 32) {
      const int64_t r = rb + lane;
      const bool valid = r < r1;
      const int lab = valid ? labels[r] : -1 - lane;
      unsigned peers = __match_any_sync(0xffffffffu, lab);
      int base = valid ? cnt[lab] : 0;
      __syncwarp();
      if (valid) {
        rank[r] = base + __popc(peers & ((1u << lane) - 1u));
        int leader = __ffs(peers) - 1;
        if (lane == leader) cnt[lab] = base + __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) tcount[t * k + c] = cnt[c];
}

__global__ void cs_counts_kernel(const int32_t* __restrict__ tcount, int64_t ntiles, int k, int64_t* __restrict__ counts) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  int64_t s = 0;
  for (int64_t t = 0; t < ntiles; ++t) s += tcount[t * k + c];
  counts[c] = s;
}

__global__ void __launch_bounds__(1024) cs_scan_kernel(const int64_t* __restrict__ counts, int k,
                                                      int64_t* __restrict__ offsets) {
  // exclusive prefix of the label counts: one block, each thread a contiguous
  // run of labels, warp-shuffle scans of the run totals
  __shared__ int64_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int per = (k + blockDim.x - 1) / blockDim.x;
  const int c0 = min(k, tid * per), c1 = min(k, c0 + per);
  int64_t t = 0;
  for (int c = c0; c < c1; ++c) t += counts[c];
  int64_t incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int64_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += v;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  int64_t run = incl - t + (wid ? wsum[wid - 1] : 0);
  if (tid == 0) offsets[0] = 0;
  for (int c = c0; c < c1; ++c) {
    run += counts[c];
    offsets[c + 1] = run;
  }
}

__global__ void cs_base_kernel(int32_t* __restrict__ tcount, int64_t ntiles, int k, const int64_t* __restrict__ offsets) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  int64_t run = offsets[c];
  for (int64_t t = 0; t < ntiles; ++t) {
    int32_t v = tcount[t * k + c];
    tcount[t * k + c] = (int32_t)(run - offsets[c]);  // base relative to the label's offset
    run += v;
  }
}

__global__ void cs_scatter_kernel(const int32_t* __restrict__ labels, const int32_t* __restrict__ rank, int64_t n,
                                  int k, int64_t tile, const int32_t* __restrict__ tbase,
                                  const int64_t* __restrict__ offsets, int64_t* __restrict__ order) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  int lab = labels[r];
  int64_t t = r / tile;
  order[offsets[lab] + tbase[t * k + lab] + rank[r]] = r;
}

// ============================================================ reseed (clustering.py:100-107)
__global__ void __launch_bounds__(1024) reseed_kernel(int32_t* labels, double* dmin, int64_t n, int64_t* counts, int k,
                                                      int32_t* n_empty_out) {
  __shared__ double bd[32];
  __shared__ int64_t bi[32];
  __shared__ int32_t wcnt[32];
  __shared__ int32_t elist[1024];
  __shared__ int s_ne;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int nw = blockDim.x >> 5;
  int ne_total = 0;
  for (int c0 = 0; c0 < k; c0 += blockDim.x) {
    // ordered compaction of the empty clusters of this chunk
    const int c = c0 + tid;
    const bool empty = c < k && counts[c] == 0;
    const unsigned b = __ballot_sync(0xffffffffu, empty);
    if (lane == 0) wcnt[wid] = __popc(b);
    __syncthreads();
    if (tid == 0) {
      int s = 0;
      for (int w = 0; w < nw; ++w) {
        int t = wcnt[w];
        wcnt[w] = s;
        s += t;
      }
      s_ne = s;
    }
    __syncthreads();
    if (empty) elist[wcnt[wid] + __popc(b & ((1u << lane) - 1u))] = c;
    __syncthreads();
    const int ne = s_ne;
    ne_total += ne;
    for (int e = 0; e < ne; ++e) {
      const int j = elist[e];
      double best = -__longlong_as_double(0x7ff0000000000000LL);
      int64_t besti = n;
      for (int64_t i = tid; i < n; i += blockDim.x) {
        double v = dmin[i];
        if (v > best) { best = v; besti = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, best, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, besti, o);
        if (ov > best || (ov == best && oi < besti)) { best = ov; besti = oi; }
      }
      if (lane == 0) { bd[wid] = best; bi[wid] = besti; }
      __syncthreads();
      if (tid == 0) {
        double bb = bd[0];
        int64_t ii = bi[0];
        for (int w = 1; w < nw; ++w)
          if (bd[w] > bb || (bd[w] == bb && bi[w] < ii)) { bb = bd[w]; ii = bi[w]; }
        labels[ii] = j;
        dmin[ii] = -1.0;
      }
      __syncthreads();
    }
  }
  if (tid == 0) *n_empty_out = ne_total;
}

// ============================================================ centroid update
// Sequential per-(cluster, dim) sums in row order, like np.add.reduceat on the
// stable-sorted rows, then division by the count (clustering.py:108-112).
__global__ void update_kernel(const float* __restrict__ x, int64_t n, const int64_t* __restrict__ order,
                              const int64_t* __restrict__ offsets, int k, int d, double* __restrict__ centers) {
  const int c = blockIdx.x;
  const int64_t s = offsets[c], e = offsets[c + 1];
  const double cnt = (double)(e - s);
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double acc;
    if (s < e) {
      acc = (double)x[order[s] * d + j];
      for (int64_t r = s + 1; r < e; ++r) acc = dadd(acc, (double)x[order[r] * d + j]);
    } else {
      // reduceat with a non-increasing index pair returns the row at the index
      acc = s < n ? (double)x[order[s] * d + j] : 0.0;
    }
    centers[(int64_t)c * d + j] = ddiv(acc, cnt);
  }
}

// Chained centroid sums for data-parallel Lloyd (np.add.reduceat over rows in ascending
// order, clustering.py:108-112, split across ranks that own ascending row blocks): the
// running per-cluster sum continues from the previous rank's (init_sums, init_counts) over
// this rank's rows of the cluster, in order.  With total_counts the centres are written
// (sum / count); otherwise the running sums and counts are handed on.
__global__ void chain_sums_kernel(const float* __restrict__ x, const int64_t* __restrict__ order,
                                  const int64_t* __restrict__ offsets, int k, int d,
                                  const double* __restrict__ init_sums, const int64_t* __restrict__ init_counts,
                                  const int64_t* __restrict__ total_counts, double* __restrict__ out,
                                  int64_t* __restrict__ out_counts) {
  const int c = blockIdx.x;
  const int64_t s = offsets[c], e = offsets[c + 1];
  const int64_t before = init_counts ? init_counts[c] : 0;
  for (int j = threadIdx.x; j < d; j += blockDim.x) {
    double acc = before > 0 ? init_sums[(int64_t)c * d + j] : 0.0;
    int64_t r = s;
    if (before == 0 && r < e) acc = (double)x[order[r++] * d + j];  // reduceat starts from the first row
    for (; r < e; ++r) acc = dadd(acc, (double)x[order[r] * d + j]);
    out[(int64_t)c * d + j] = total_counts ? ddiv(acc, (double)total_counts[c]) : acc;
  }
  if (threadIdx.x == 0 && out_counts) out_counts[c] = before + (e - s);
}

// ============================================================ normalise + rotate
// dist[r] = sqrt(einsum(diff, diff)), diff = x[order[r]] - cent32[labels[order[r]]]
__global__ void __launch_bounds__(rowchain::THREADS) resid_norm_kernel(const float* __restrict__ x,
                                                                       const int64_t* __restrict__ order,
                                                                       const int32_t* __restrict__ labels,
                                                                       const float* __restrict__ cent, int64_t n,
                                                                       int d, double* __restrict__ dist) {
  using namespace rowchain;
  __shared__ Tile<float> tx, tc;
  const int64_t row0 = (int64_t)blockIdx.x * ROWS;
  const int r = threadIdx.x >> 1, lane = threadIdx.x & 1;
  const bool vec = (d % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(cent) & 15) == 0);
  auto srcx = [&](int64_t gr) { return x + (order ? order[gr] : gr) * d; };
  auto srcc = [&](int64_t gr) { return cent + (int64_t)labels[order ? order[gr] : gr] * d; };
  double acc = 0.0;
  for (int c0 = 0; c0 < d; c0 += CH) {
    const int cw = min(CH, d - c0);
    __syncthreads();
    stage_tile(tx, srcx, row0, n, c0, cw, vec);
    stage_tile(tc, srcc, row0, n, c0, cw, vec);
    __syncthreads();
    acc = chain_chunk(acc, lane, cw, [&](int k) {
      const double df = dsub((double)tx.v[r][k], (double)tc.v[r][k]);
      return dmul(df, df);
    });
  }
  const double v = finish(acc);
  if (lane == 0 && row0 + r < n) dist[row0 + r] = dsqrt(v);
}

struct ResidLoader {
  const float* x;
  const int64_t* order;
  const int32_t* labels;
  const float* cent;
  const double* dist;
  int d;
  __device__ __forceinline__ double operator()(int64_t r, int k) const {
    const int64_t s = order ? order[r] : r;
    const double dd = dist[r];
    if (dd == 0.0) return 0.0;  // o[d == 0] = 0 (codec.py:150)
    double df = dsub((double)x[s * d + k], (double)cent[(int64_t)labels[s] * d + k]);
    return ddiv(df, dd);
  }
  __device__ __forceinline__ void load8(int64_t r, int k, int K, double (&out)[8]) const {
    const int64_t s = order ? order[r] : r;
    const double dd = dist[r];
    const float* xr = x + s * d;
    const float* cr = cent + (int64_t)labels[s] * d;
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int kk = k + e;
      out[e] = (kk < K && dd != 0.0) ? ddiv(dsub((double)xr[kk], (double)cr[kk]), dd) : 0.0;
    }
  }
};

struct StoreF32 {
  float* out;
  int64_t ld;
  __device__ __forceinline__ void operator()(int64_t r, int64_t c, double v) const {
    out[r * ld + c] = __double2float_rn(v);
  }
};

// ============================================================ encoder
namespace enc {

constexpr int WARPS = 4;

// t * o in the array dtype, + (k_b + 0.5) == 2^(B-1), floor, clip (codec.py:163-174)
template <typename T>
__device__ __forceinline__ int round_code(T t, T o, int bits) {
  T v;
  if constexpr (sizeof(T) == 4) {
    v = floorf(fadd(fmul(t, o), (float)(1 << (bits - 1))));
  } else {
    v = floor(dadd(dmul(t, o), (double)(1 << (bits - 1))));
  }
  const T hi = (T)((1 << bits) - 1);
  v = v < (T)0 ? (T)0 : v;
  v = v > hi ? hi : v;
  return (int)v;
}

// cosine objective of one rescaling factor (codec.py:192-198): the numerator
// follows NumPy's einsum order, the denominator is exact in integers.
template <typename T>
__device__ __forceinline__ double objective(const T* o, int d, T t, int bits) {
  const int m = (1 << bits) - 1;  // 2u - m = 2 * (u - k_b)
  EinsumAcc acc;
  long long den4 = 0;
  int i = 0;
  for (; i + 8 <= d; i += 8) {
    double p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      T ov = o[i + q];
      int u = round_code<T>(t, ov, bits);
      int c2 = 2 * u - m;
      den4 += c2 * c2;
      p[q] = dmul(0.5 * (double)c2, (double)ov);
    }
    acc.block8(p);
  }
  for (; i < d; i += 2) {
    T o0 = o[i];
    int u0 = round_code<T>(t, o0, bits);
    int c0 = 2 * u0 - m;
    den4 += c0 * c0;
    double p0 = dmul(0.5 * (double)c0, (double)o0);
    bool has1 = (i + 1) < d;
    double p1 = 0.0;
    if (has1) {
      T o1 = o[i + 1];
      int u1 = round_code<T>(t, o1, bits);
      int c1 = 2 * u1 - m;
      den4 += c1 * c1;
      p1 = dmul(0.5 * (double)c1, (double)o1);
    }
    acc.pair(p0, p1, has1);
  }
  const double num = acc.result();
  const double den = dsqrt((double)den4 * 0.25);
  return ddiv(num, den);
}

template <typename T>
__device__ __forceinline__ T tsub(T a, T b) {
  if constexpr (sizeof(T) == 4) return fsub(a, b); else return dsub(a, b);
}
template <typename T>
__device__ __forceinline__ T tadd(T a, T b) {
  if constexpr (sizeof(T) == 4) return fadd(a, b); else return dadd(a, b);
}
template <typename T>
__device__ __forceinline__ T tmul(T a, T b) {
  if constexpr (sizeof(T) == 4) return fmul(a, b); else return dmul(a, b);
}
template <typename T>
__device__ __forceinline__ T tdiv(T a, T b) {
  if constexpr (sizeof(T) == 4) return fdiv(a, b); else return ddiv(a, b);
}

// warp-wide "first maximum": larger objective wins, ties go to the earlier sample
__device__ __forceinline__ void warp_best(double& v, int& s) {
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int os = __shfl_xor_sync(0xffffffffu, s, o);
    if (ov > v || (ov == v && os < s)) { v = ov; s = os; }
  }
}

struct Out {
  uint32_t* packed;
  uint8_t* rc;
  int64_t rb;
  float* sadd;
  float* sscale;
  float* serr;
  float* lf;
  uint8_t* codes;
  double* t_out;
  int32_t* bad;
};

template <typename T>
__global__ void __launch_bounds__(WARPS * 32) encode_kernel(const T* __restrict__ o_rot, const double* __restrict__ dist,
                                                           const float* __restrict__ cent_rot,
                                                           const int64_t* __restrict__ offsets, int nlist, int64_t n,
                                                           int d, int bits, int n_coarse, int n_fine, double eps,
                                                           Out out) {
  extern __shared__ __align__(16) unsigned char esm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = words_per_vector(d);
  const int eb = bits - 1;
  T* so = reinterpret_cast<T*>(esm) + (size_t)w * g * 32;
  uint8_t* su = reinterpret_cast<uint8_t*>(reinterpret_cast<T*>(esm) + (size_t)WARPS * g * 32) + (size_t)w * g * 32;

  const int64_t r = (int64_t)blockIdx.x * WARPS + w;
  if (r >= n) return;
  // cluster of row r: last c with offsets[c] <= r (non-empty)
  int lo_c = 0, hi_c = nlist;  // offsets[lo_c] <= r < offsets[hi_c]
  while (hi_c - lo_c > 1) {
    int mid = (lo_c + hi_c) >> 1;
    if (offsets[mid] <= r) lo_c = mid; else hi_c = mid;
  }
  const int c = lo_c;
  const int64_t lo = offsets[c], n_c = offsets[c + 1] - lo;
  const int64_t v = r - lo;

  for (int i = lane; i < g * 32; i += 32) so[i] = i < d ? o_rot[r * d + i] : (T)0;
  __syncwarp();
  // unit-row check (codec.py:154-160): einsum(o, o) in float64
  {
    double a0 = 0.0;
    if (lane < 2) {
      int i = 0;
      for (; i + 8 <= d; i += 8)
#pragma unroll
        for (int blk = 3; blk >= 0; --blk) {
          double ov = (double)so[i + 2 * blk + lane];
          a0 = dadd(dmul(ov, ov), a0);
        }
      for (; i < d; i += 2) {
        double ov = (i + lane) < d ? (double)so[i + lane] : 0.0;
        a0 = dadd(dmul(ov, ov), a0);
      }
    }
    double a1 = __shfl_sync(0xffffffffu, a0, 1);
    if (lane == 0) {
      double nrm = dsqrt(dadd(0.0, dadd(a0, a1)));
      if (nrm != 0.0 && fabs(nrm - 1.0) > 1e-4) atomicAdd(out.bad, 1);
    }
  }
  // max |o| in the array dtype
  T mx = (T)0;
  for (int i = lane; i < d; i += 32) {
    T a = so[i] < (T)0 ? -so[i] : so[i];
    mx = a > mx ? a : mx;
  }
  for (int o = 16; o > 0; o >>= 1) {
    T om = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = om > mx ? om : mx;
  }
  const bool zero = mx == (T)0;
  T best_t;
  if (bits == 1) {
    for (int i = lane; i < d; i += 32) su[i] = zero ? 1 : (so[i] > (T)0 ? 1 : 0);
    best_t = zero ? (T)0 : tdiv((T)0.5, mx);
  } else {
    const T safe = zero ? (T)1 : mx;
    const T t_start = tdiv((T)0.5, safe);
    const double kcoef = ((double)(1 << (bits - 1)) - 0.5) * (1.0 + 6.0 / (double)(1 << (bits - 1)));
    const T t_end = tdiv((T)kcoef, safe);
    // coarse grid (codec.py:233-236)
    const T step = tdiv(tsub(t_end, t_start), (T)(n_coarse - 1));
    double bv = -__longlong_as_double(0x7ff0000000000000LL);
    int bs = 0x7fffffff;
    for (int s = lane; s < n_coarse; s += 32) {
      T t = tadd(t_start, tmul((T)s, step));
      double ob = objective<T>(so, d, t, bits);
      if (ob > bv) { bv = ob; bs = s; }
    }
    warp_best(bv, bs);
    T bt = tadd(t_start, tmul((T)bs, step));
    // fine grid around the coarse winner (codec.py:236-240)
    const T delta = step;
    T lo_t = tsub(bt, delta);
    lo_t = lo_t > t_start ? lo_t : t_start;
    T hi_t = tadd(bt, delta);
    hi_t = hi_t < t_end ? hi_t : t_end;
    const T fstep = tdiv(tsub(hi_t, lo_t), (T)(n_fine - 1));
    double fv = -__longlong_as_double(0x7ff0000000000000LL);
    int fs = 0x7fffffff;
    for (int s = lane; s < n_fine; s += 32) {
      T t = tadd(lo_t, tmul((T)s, fstep));
      double ob = objective<T>(so, d, t, bits);
      if (ob > fv) { fv = ob; fs = s; }
    }
    warp_best(fv, fs);
    if (fv > bv) bt = tadd(lo_t, tmul((T)fs, fstep));
    best_t = bt;
    const int mid = 1 << (bits - 1);
    for (int i = lane; i < d; i += 32) su[i] = zero ? (uint8_t)mid : (uint8_t)round_code<T>(bt, so[i], bits);
    if (zero) best_t = (T)0;
  }
  for (int i = d + lane; i < g * 32; i += 32) su[i] = 0;
  __syncwarp();
  if (out.codes)
    for (int i = lane; i < d; i += 32) out.codes[r * d + i] = su[i];
  if (out.t_out && lane == 0) out.t_out[r] = (double)best_t;

  // ---- pack the MSB plane into the interleaved list layout (codec.py:404-413)
  for (int gi = 0; gi < g; ++gi) {
    int dim = gi * 32 + lane;
    unsigned bit = dim < d ? (unsigned)(su[dim] >> eb) & 1u : 0u;
    unsigned word = __ballot_sync(0xffffffffu, bit);
    if (lane == 0) out.packed[g * lo + (int64_t)gi * n_c + v] = word;
  }
  // ---- full codes for the tensor-core refine (rcodes layout, ivrq_b200.h);
  // the IVRQ1 ex-codes (codec.py:432-444) are their low bits.
  if (eb > 0) {
    const int kp = kpad64(d);
    uint8_t* dst = out.rc + r * out.rb;
    if (rcode_nibbles(bits)) {
      for (int j = lane; j < kp / 2; j += 32) {
        const int d0 = 2 * j, d1 = 2 * j + 1;
        const uint32_t lo4 = d0 < d ? su[d0] : 0u, hi4 = d1 < d ? su[d1] : 0u;
        dst[j] = (uint8_t)(lo4 | (hi4 << 4));
      }
    } else {
      for (int j = lane; j < kp; j += 32) dst[j] = j < d ? su[j] : (uint8_t)0;
    }
  }
  // ---- factors (codec.py:355-379): five einsums, lanes 2e / 2e+1 own the
  // two accumulators of einsum e.
  const double k_b = ((double)((1 << bits) - 1)) / 2.0;
  const float* cr = cent_rot + (int64_t)c * d;
  double acc = 0.0;
  const int e = lane >> 1, l = lane & 1;
  auto term = [&](int dim) -> double {
    const double u = (double)su[dim];
    const double xb = dsub((double)(su[dim] >> eb), 0.5);
    const double x = dsub(u, k_b);
    const double ov = (double)so[dim];
    switch (e) {
      case 0: return dmul(xb, ov);
      case 1: return dmul(x, x);
      case 2: return dmul(x, ov);
      case 3: return dmul(xb, (double)cr[dim]);
      default: return dmul(x, (double)cr[dim]);
    }
  };
  if (e < 5) {
    int i = 0;
    for (; i + 8 <= d; i += 8)
#pragma unroll
      for (int blk = 3; blk >= 0; --blk) acc = dadd(term(i + 2 * blk + l), acc);
    for (; i < d; i += 2) {
      double p = (i + l) < d ? term(i + l) : 0.0;
      acc = dadd(p, acc);
    }
  }
  double res[5];
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    double a0 = __shfl_sync(0xffffffffu, acc, 2 * q);
    double a1 = __shfl_sync(0xffffffffu, acc, 2 * q + 1);
    res[q] = dadd(0.0, dadd(a0, a1));
  }
  if (lane == 0) {
    const double dd = dist[r];
    double s_add = 0.0, s_scale = 0.0, s_err = 0.0, l_add = 0.0, l_scale = 0.0;
    if (dd > 0.0) {
      const double norm_b = dmul(0.5, dsqrt((double)d));
      double cos_b = ddiv(res[0], norm_b);
      const double norm_x = dsqrt(res[1]);
      double cos_x = ddiv(res[2], norm_x);
      cos_b = dmax(cos_b, 1e-6);
      cos_x = dmax(cos_x, 1e-6);
      const double two_d = dmul(2.0, dd);
      const double dsq = dmul(dd, dd);
      s_scale = ddiv(two_d, dmul(norm_b, cos_b));
      s_add = dadd(dsq, dmul(s_scale, res[3]));
      const double cb2 = dmul(cos_b, cos_b);
      const double var = ddiv(dmax(dsub(1.0, cb2), 0.0), dmul(cb2, (double)max(d - 1, 1)));
      s_err = dmul(dmul(two_d, eps), dsqrt(var));
      l_scale = ddiv(two_d, dmul(norm_x, cos_x));
      l_add = dadd(dsq, dmul(l_scale, res[4]));
    }
    out.sadd[r] = (float)s_add;
    out.sscale[r] = (float)s_scale;
    out.serr[r] = (float)s_err;
    out.lf[2 * r] = (float)l_add;
    out.lf[2 * r + 1] = (float)l_scale;
  }
}

}  // namespace enc

// Pairwise-sum recursion tree of NumPy for length n (host side).
struct PairwiseTree {
  std::vector<int64_t> leaf_start;
  std::vector<int32_t> leaf_len;
  std::vector<int32_t> left, right;  // internal nodes; child ids: <nleaf leaf, else nleaf + internal
  std::vector<int32_t> level_begin;  // internal nodes grouped by height
  int root = 0;
};

static void build_pairwise_tree(int64_t n, PairwiseTree& t) {
  struct Node { int id; int height; };
  std::vector<std::pair<int32_t, int32_t>> internal;  // (left,right) before renumbering
  std::vector<int> heights;
  // recursive build returning (encoded id, height); encoded: leaf -> -(leaf+1), internal -> index
  std::function<std::pair<int64_t, int>(int64_t, int64_t)> rec = [&](int64_t s, int64_t len) -> std::pair<int64_t, int> {
    if (len <= 128) {
      t.leaf_start.push_back(s);
      t.leaf_len.push_back((int32_t)len);
      return {-(int64_t)t.leaf_start.size(), 0};
    }
    int64_t n2 = len / 2;
    n2 -= n2 % 8;
    auto a = rec(s, n2);
    auto b = rec(s + n2, len - n2);
    internal.push_back({(int32_t)a.first, (int32_t)b.first});
    int h = 1 + std::max(a.second, b.second);
    heights.push_back(h);
    return {(int64_t)internal.size() - 1, h};
  };
  auto root = rec(0, n);
  const int nleaf = (int)t.leaf_start.size();
  const int nint = (int)internal.size();
  if (nint == 0) {
    t.root = 0;
    t.level_begin = {0};
    return;
  }
  int maxh = *std::max_element(heights.begin(), heights.end());
  std::vector<int> perm;  // new order of internal nodes by height
  t.level_begin.clear();
  for (int h = 1; h <= maxh; ++h) {
    t.level_begin.push_back((int)perm.size());
    for (int i = 0; i < nint; ++i)
      if (heights[i] == h) perm.push_back(i);
  }
  t.level_begin.push_back((int)perm.size());
  std::vector<int> newid(nint);
  for (int i = 0; i < nint; ++i) newid[perm[i]] = i;
  auto enc = [&](int32_t code) -> int32_t { return code < 0 ? (-code - 1) : nleaf + newid[code]; };
  t.left.resize(nint);
  t.right.resize(nint);
  for (int i = 0; i < nint; ++i) {
    t.left[i] = enc(internal[perm[i]].first);
    t.right[i] = enc(internal[perm[i]].second);
  }
  t.root = nleaf + newid[(int)root.first];
}

}  // namespace ivrq

using namespace ivrq;

extern "C" int ivrq_kmeanspp(const float* x, int64_t n, int32_t d, int32_t n_clusters, int32_t j_begin, int32_t j_end,
                             const double* draws, int32_t draw_kind, double* centers, double* d2, int32_t* zero_step,
                             void* stream) {
  if (n <= 0 || d <= 0 || n_clusters < 1 || n_clusters > n) return fail(IVRQ_EINVAL, "ivrq_kmeanspp: bad sizes");
  if (j_begin < 0 || j_end > n_clusters || j_begin >= j_end) return IVRQ_OK;
  cudaStream_t s = as_stream(stream);
  PairwiseTree tree;
  build_pairwise_tree(n, tree);
  const int nleaf = (int)tree.leaf_start.size();
  const int nint = (int)tree.left.size();
  const int nlevels = (int)tree.level_begin.size() - 1;
  // device copies of the tree + scratch
  int64_t* dls;
  int32_t *dll, *dl, *dr, *dlb;
  double *nodes, *bsums;
  int* halt;
  IVRQ_TRY(dalloc(&dls, nleaf, s, "kmeanspp"));
  IVRQ_TRY(dalloc(&dll, nleaf, s, "kmeanspp"));
  IVRQ_TRY(dalloc(&dl, std::max(nint, 1), s, "kmeanspp"));
  IVRQ_TRY(dalloc(&dr, std::max(nint, 1), s, "kmeanspp"));
  IVRQ_TRY(dalloc(&dlb, nlevels + 1, s, "kmeanspp"));
  IVRQ_TRY(dalloc(&nodes, nleaf + nint, s, "kmeanspp"));
  IVRQ_TRY(dalloc(&bsums, (size_t)ceil_div(n, 1024), s, "kmeanspp"));
  IVRQ_TRY(dalloc(&halt, 1, s, "kmeanspp"));
  cudaMemcpyAsync(dls, tree.leaf_start.data(), nleaf * sizeof(int64_t), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dll, tree.leaf_len.data(), nleaf * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  if (nint) {
    cudaMemcpyAsync(dl, tree.left.data(), nint * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(dr, tree.right.data(), nint * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  }
  cudaMemcpyAsync(dlb, tree.level_begin.data(), (nlevels + 1) * sizeof(int32_t), cudaMemcpyHostToDevice, s);
  cudaMemsetAsync(halt, 0, sizeof(int), s);
  // NumPy's sequential cumsum decisions are replayed exactly for any n: the
  // double-double prefix with a rounding band decides almost every step in
  // parallel (kpp_fast_exact); the sequential walk remains for the band cases.
  // IVRQ_KPP_EXACT_MAX caps n for the exact replay (beyond: the blocked scan);
  // IVRQ_KPP_SEQUENTIAL=1 forces the walk for every step (tests).
  const char* ex_env = getenv("IVRQ_KPP_EXACT_MAX");
  const int64_t exact_max = ex_env ? atoll(ex_env) : ((int64_t)1 << 40);
  const char* seq_env = getenv("IVRQ_KPP_SEQUENTIAL");
  const int exact = n <= exact_max ? ((seq_env && atoi(seq_env)) ? 2 : 1) : 0;
  const unsigned ub = (unsigned)ceil_div(n, rowchain::ROWS);
  int j = j_begin;
  if (j == 0) {
    // centers[0] = x[first]; d2 = |x - c0|^2
    kpp_select_kernel<<<1, 1024, 0, s>>>(x, n, d, d2, nodes, dl, dr, dlb, nlevels, nleaf, tree.root, draws, 1, 0,
                                         centers, zero_step, halt, exact, bsums, dls, dll);
    kpp_update_kernel<<<ub, rowchain::THREADS, 0, s>>>(x, n, d, centers, d2, 1, halt);
    j = 1;
  }
  for (; j < j_end; ++j) {
    kpp_leaf_kernel<<<(unsigned)ceil_div(nleaf, 256), 256, 0, s>>>(d2, dls, dll, nleaf, nodes, halt);
    kpp_select_kernel<<<1, 1024, 0, s>>>(x, n, d, d2, nodes, dl, dr, dlb, nlevels, nleaf, tree.root, draws,
                                         draw_kind, j, centers, zero_step, halt, exact, bsums, dls, dll);
    kpp_update_kernel<<<ub, rowchain::THREADS, 0, s>>>(x, n, d, centers + (int64_t)j * d, d2, 0, halt);
  }
  IVRQ_TRY(check_launch("ivrq_kmeanspp"));
  cudaFreeAsync(dls, s);
  cudaFreeAsync(dll, s);
  cudaFreeAsync(dl, s);
  cudaFreeAsync(dr, s);
  cudaFreeAsync(dlb, s);
  cudaFreeAsync(nodes, s);
  cudaFreeAsync(bsums, s);
  cudaFreeAsync(halt, s);
  return IVRQ_OK;
}

extern "C" int ivrq_assign(const float* x, int64_t n, int32_t d, const double* centers, const double* centroid_sqnorms,
                           int32_t k, int32_t* labels, double* dmin, void* stream) {
  if (n < 0 || d <= 0 || k < 1) return fail(IVRQ_EINVAL, "ivrq_assign: bad sizes");
  if (n == 0) return IVRQ_OK;
  cudaStream_t s = as_stream(stream);
  double* x_sq;
  IVRQ_TRY(dalloc(&x_sq, n, s, "ivrq_assign"));
  IVRQ_TRY(ivrq_row_sqnorms(x, 0, n, d, x_sq, stream));
  gemm::RowMajor<float> la{x, n, d};
  gemm::RowMajor<double> lb{centers, k, d};
  LabelDist dist{x_sq, centroid_sqnorms};
  int rc = gemm::launch_gemm_argmin(la, n, lb, k, d, dist, labels, dmin, s, "ivrq_assign");
  cudaFreeAsync(x_sq, s);
  return rc;
}

extern "C" int ivrq_counting_sort(const int32_t* labels, int64_t n, int32_t k, int64_t* counts, int64_t* offsets,
                                  int64_t* order, void* stream) {
  if (n < 0 || k < 1) return fail(IVRQ_EINVAL, "ivrq_counting_sort: bad sizes");
  cudaStream_t s = as_stream(stream);
  if (n == 0) {
    cudaMemsetAsync(counts, 0, k * sizeof(int64_t), s);
    cudaMemsetAsync(offsets, 0, (k + 1) * sizeof(int64_t), s);
    return check_launch("ivrq_counting_sort");
  }
  if ((size_t)k * 4 > 200 * 1024) return fail(IVRQ_EUNSUP, "ivrq_counting_sort: too many clusters");
  int64_t tile = 256;  // short serial walks per CTA (one warp per tile): the search's pair sorts are small
  // tiles x labels stays within max(n, 2^20) entries: the per-label passes over
  // the tile counts (cs_counts, cs_base) are then no larger than the rows
  while (ceil_div(n, tile) * (int64_t)k > std::max(n, (int64_t)1 << 20) && tile < (int64_t)1 << 16) tile *= 2;
  const int64_t ntiles = ceil_div(n, tile);
  int32_t *tcount, *rank;
  IVRQ_TRY(dalloc(&tcount, (size_t)(ntiles * k), s, "ivrq_counting_sort"));
  IVRQ_TRY(dalloc(&rank, (size_t)n, s, "ivrq_counting_sort"));
  const size_t sm = (size_t)k * 4;
  if (sm > 48 * 1024) cudaFuncSetAttribute(cs_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cs_local_kernel<<<(unsigned)ntiles, 128, sm, s>>>(labels, n, k, tile, tcount, rank);
  cs_counts_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, s>>>(tcount, ntiles, k, counts);
  cs_scan_kernel<<<1, 1024, 0, s>>>(counts, k, offsets);
  cs_base_kernel<<<(unsigned)ceil_div(k, 256), 256, 0, s>>>(tcount, ntiles, k, offsets);
  cs_scatter_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(labels, rank, n, k, tile, tcount, offsets, order);
  int rc = check_launch("ivrq_counting_sort");
  cudaFreeAsync(tcount, s);
  cudaFreeAsync(rank, s);
  return rc;
}

extern "C" int ivrq_kmeans_reseed(int32_t* labels, double* dmin, int64_t n, int64_t* counts, int32_t k,
                                  int32_t* n_empty_out, void* stream) {
  if (n <= 0 || k < 1) return fail(IVRQ_EINVAL, "ivrq_kmeans_reseed: bad sizes");
  reseed_kernel<<<1, 1024, 0, as_stream(stream)>>>(labels, dmin, n, counts, k, n_empty_out);
  return check_launch("ivrq_kmeans_reseed");
}

extern "C" int ivrq_kmeans_chain_sums(const float* x, const int64_t* order, const int64_t* offsets, int32_t k,
                                      int32_t d, const double* init_sums, const int64_t* init_counts,
                                      const int64_t* total_counts, double* out, int64_t* out_counts, void* stream) {
  if (k < 1 || d < 1) return fail(IVRQ_EINVAL, "ivrq_kmeans_chain_sums: bad sizes");
  if ((init_sums == nullptr) != (init_counts == nullptr))
    return fail(IVRQ_EINVAL, "ivrq_kmeans_chain_sums: init sums and counts go together");
  chain_sums_kernel<<<k, 128, 0, as_stream(stream)>>>(x, order, offsets, k, d, init_sums, init_counts, total_counts,
                                                      out, out_counts);
  return check_launch("ivrq_kmeans_chain_sums");
}

extern "C" int ivrq_kmeans_update(const float* x, int64_t n, const int64_t* order, const int64_t* offsets, int32_t k,
                                  int32_t d, double* centers, void* stream) {
  if (k < 1 || d <= 0) return fail(IVRQ_EINVAL, "ivrq_kmeans_update: bad sizes");
  update_kernel<<<(unsigned)k, std::min(256, ((d + 31) / 32) * 32), 0, as_stream(stream)>>>(x, n, order, offsets, k,
                                                                                           d, centers);
  return check_launch("ivrq_kmeans_update");
}

extern "C" int ivrq_normalize_rotate(const float* x, const int64_t* order, const int32_t* labels, const float* cent32,
                                     const float* rotation, int64_t n, int32_t d, float* o_rot, double* dist,
                                     void* stream) {
  if (n < 0 || d <= 0) return fail(IVRQ_EINVAL, "ivrq_normalize_rotate: bad sizes");
  if (n == 0) return IVRQ_OK;
  cudaStream_t s = as_stream(stream);
  resid_norm_kernel<<<(unsigned)ceil_div(n, rowchain::ROWS), rowchain::THREADS, 0, s>>>(x, order, labels, cent32, n, d,
                                                                                        dist);
  IVRQ_TRY(check_launch("ivrq_normalize_rotate(norm)"));
  ResidLoader la{x, order, labels, cent32, dist, d};
  gemm::RowMajor<float> lb{rotation, d, d};
  StoreF32 epi{o_rot, d};
  return gemm::launch_gemm(la, n, lb, d, d, epi, s, "ivrq_normalize_rotate(gemm)");
}

extern "C" int ivrq_rotate_rows_f32(const float* x, int64_t n, int32_t d, const float* rotation, float* out,
                                    void* stream) {
  if (n < 0 || d <= 0) return fail(IVRQ_EINVAL, "ivrq_rotate_rows_f32: bad sizes");
  gemm::RowMajor<float> la{x, n, d};
  gemm::RowMajor<float> lb{rotation, d, d};
  StoreF32 epi{out, d};
  return gemm::launch_gemm(la, n, lb, d, d, epi, as_stream(stream), "ivrq_rotate_rows_f32");
}

extern "C" int ivrq_encode(const void* o_rot, int32_t o_is_f64, const double* dist, const float* cent_rot,
                           const int64_t* offsets, int32_t n_clusters, int64_t n, int32_t d, int32_t bits,
                           int32_t n_coarse, int32_t n_fine, double eps_bound, uint32_t* packed_msb,
                           uint8_t* rcodes, float* short_add, float* short_scale, float* short_err,
                           float* long_factors, uint8_t* codes, double* t_out, int32_t* bad_rows, void* stream) {
  if (bits < 1 || bits > 8) return fail(IVRQ_EINVAL, "bits must be in [1, 8]");
  if (n_coarse < 2 || n_fine < 2) return fail(IVRQ_EINVAL, "n_coarse and n_fine must both be >= 2");
  if (bits > 1 && !rcodes) return fail(IVRQ_EINVAL, "ivrq_encode: rcodes required for bits > 1");
  if (n == 0) return IVRQ_OK;
  if (d > 4096) return fail(IVRQ_EUNSUP, "ivrq_encode: dims > 4096");
  enc::Out out{packed_msb, rcodes, rcode_row_bytes_of(d, bits), short_add, short_scale, short_err, long_factors,
               codes, t_out, bad_rows};
  const int g = words_per_vector(d);
  cudaStream_t s = as_stream(stream);
  const unsigned grid = (unsigned)ceil_div(n, enc::WARPS);
  if (o_is_f64) {
    size_t sm = (size_t)enc::WARPS * g * 32 * (sizeof(double) + 1);
    if (sm > 48 * 1024) cudaFuncSetAttribute(enc::encode_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    enc::encode_kernel<double><<<grid, enc::WARPS * 32, sm, s>>>((const double*)o_rot, dist, cent_rot, offsets,
                                                                  n_clusters, n, d, bits, n_coarse, n_fine, eps_bound,
                                                                  out);
  } else {
    size_t sm = (size_t)enc::WARPS * g * 32 * (sizeof(float) + 1);
    if (sm > 48 * 1024) cudaFuncSetAttribute(enc::encode_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    enc::encode_kernel<float><<<grid, enc::WARPS * 32, sm, s>>>((const float*)o_rot, dist, cent_rot, offsets,
                                                                n_clusters, n, d, bits, n_coarse, n_fine, eps_bound,
                                                                out);
  }
  return check_launch("ivrq_encode");
}

// ============================================================ rcodes from IVRQ1 arrays
namespace ivrq {
// One warp per row: u = msb << eb | ex with msb from the interleaved plane of
// the row's list and ex from the LSB-first ex-code byte stream.
__global__ void make_rcodes_kernel(const uint32_t* __restrict__ packed, const int64_t* __restrict__ offsets, int nlist,
                                   const uint8_t* __restrict__ ex, int64_t n, int d, int bits,
                                   uint8_t* __restrict__ rc) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= n) return;
  int lo_c = 0, hi_c = nlist;
  while (hi_c - lo_c > 1) {
    const int mid = (lo_c + hi_c) >> 1;
    if (offsets[mid] <= r) lo_c = mid; else hi_c = mid;
  }
  const int64_t lo = offsets[lo_c], n_c = offsets[lo_c + 1] - lo, v = r - lo;
  const int g = words_per_vector(d), eb = bits - 1;
  const int64_t bpv = ((int64_t)d * eb + 7) / 8;
  const uint8_t* exr = ex + r * bpv;
  auto code = [&](int dim) -> uint32_t {
    if (dim >= d) return 0u;
    const uint32_t msb = (packed[(int64_t)g * lo + (int64_t)(dim >> 5) * n_c + v] >> (dim & 31)) & 1u;
    uint32_t e = 0;
    for (int b = 0; b < eb; ++b) {
      const int64_t bit = (int64_t)dim * eb + b;
      e |= (uint32_t)((exr[bit >> 3] >> (bit & 7)) & 1) << b;
    }
    return (msb << eb) | e;
  };
  const int kp = kpad64(d);
  uint8_t* dst = rc + r * rcode_row_bytes_of(d, bits);
  if (rcode_nibbles(bits)) {
    for (int j = lane; j < kp / 2; j += 32) dst[j] = (uint8_t)(code(2 * j) | (code(2 * j + 1) << 4));
  } else {
    for (int j = lane; j < kp; j += 32) dst[j] = (uint8_t)code(j);
  }
}
}  // namespace ivrq

extern "C" int ivrq_make_rcodes(const uint32_t* packed_msb, const int64_t* offsets, int32_t n_clusters,
                                const uint8_t* excodes, int64_t n, int32_t d, int32_t bits, uint8_t* rcodes,
                                void* stream) {
  if (bits < 2 || bits > 8 || d <= 0 || n < 0) return fail(IVRQ_EINVAL, "ivrq_make_rcodes: bad sizes");
  if (n == 0) return IVRQ_OK;
  make_rcodes_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, as_stream(stream)>>>(packed_msb, offsets, n_clusters,
                                                                              excodes, n, d, bits, rcodes);
  return check_launch("ivrq_make_rcodes");
}
