/*
 * ivrq_b200.h -- C ABI of the B200-native IVF-RaBitQ hot path.
 *
 * Every entry point takes plain device pointers, sizes and an explicit CUDA
 * stream (passed as `void*`, i.e. a cudaStream_t).  Nothing here mentions a
 * framework type; the Python host package (paper_2602_23999_b200) binds these
 * with ctypes, and any other host (C++, a cgo/JNI stub) can bind them the same
 * way.  All functions are asynchronous on `stream` unless documented
 * otherwise, return IVRQ_OK (0) on success and a negative IVRQ_E* code on
 * failure; the message of the last failure on the calling thread is returned
 * by ivrq_last_error().
 *
 * Citations are to the reference package /root/reference/pkg/src/ivfrabitq
 * (file:line); each entry point names the reference function it replaces.
 *
 * Layout of a device index:
 *   offsets     int64 [n_clusters+1]          CSR row pointers (index.py:100)
 *   packed_msb  uint32[size*g]                per-list interleaved 1-bit codes,
 *                                             word (group j, row v of list c) at
 *                                             g*offsets[c] + j*n_c + v
 *                                             (codec.py:98-115, index.py:114-118)
 *   short_add/short_scale/short_err float[size]   SoA split of short_factors
 *   long_factors float2[size]                 (add, scale)  (index.py:104)
 *   rcodes      uint8 [size*rcode_bytes]      full unsigned codes u = msb<<(bits-1) | ex
 *                                             per vector for the tensor-core refine:
 *                                             kpad = round_up(dims, 64); bits >= 5:
 *                                             one byte per dim (kpad bytes); 2 <= bits
 *                                             <= 4: two dims per byte, dim 2j in the
 *                                             low nibble (kpad/2 bytes); none for
 *                                             bits == 1.  The IVRQ1 ex-codes
 *                                             (codec.py:432-444) are u's low bits.
 *   pids        int64 [size]                  original row ids (index.py:105)
 *   centroids   float [n_clusters*dims]       rotated centroids (index.py:235)
 *   centroid_sqnorms double[n_clusters]       einsum-order squared norms
 *                                             (clustering.py:26-30)
 *   rotation    float [dims*dims]             (linalg.py:25-40, index.py:233)
 * with g = ceil(dims/32).
 */
#ifndef IVRQ_B200_H
#define IVRQ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IVRQ_ABI_VERSION 1

#if defined(__GNUC__)
#define IVRQ_API __attribute__((visibility("default")))
#else
#define IVRQ_API
#endif

enum {
  IVRQ_OK = 0,
  IVRQ_EINVAL = -1,  /* bad argument: maps to ValueError in the host API   */
  IVRQ_ECUDA = -2,   /* CUDA runtime / launch failure                      */
  IVRQ_ENOMEM = -3,  /* workspace too small / allocation failure           */
  IVRQ_EUNSUP = -4   /* configuration outside what the kernels support     */
};

enum { IVRQ_IP_LUT = 0, IVRQ_IP_BITWISE = 1 };

typedef struct {
  int32_t dims;
  int32_t bits;
  int32_t n_clusters;
  int32_t max_list;    /* largest inverted list (rows); 0 = unknown (the scan then reads it back) */
  int64_t size;
  double eps_bound;
  const int64_t* offsets;
  const uint32_t* packed_msb;
  const float* short_add;
  const float* short_scale;
  const float* short_err;
  const float* long_factors;
  const uint8_t* rcodes;
  int64_t rcode_bytes; /* row stride of rcodes, ivrq_rcode_row_bytes(dims, bits) */
  const int64_t* pids;
  const float* centroids;
  const double* centroid_sqnorms;
  const float* rotation;
} ivrq_index_view;

/* SearchParams (search.py:56-81), validated by the host before the call. */
typedef struct {
  int32_t k;
  int32_t n_probe;
  int32_t ip_mode;    /* IVRQ_IP_LUT or IVRQ_IP_BITWISE */
  int32_t query_bits; /* 2..8, bitwise mode only */
  int32_t refine;     /* forced off for 1-bit indexes (search.py:362) */
  int32_t prune;      /* 0 pins every threshold at +inf (search.py:435) */
} ivrq_search_params;

/* Per-query scalars written by ivrq_prepare_queries (QueryState, search.py:84-104). */
enum {
  IVRQ_QS_SUM_Q = 0,      /* q_rot.sum(), NumPy pairwise order (search.py:189) */
  IVRQ_QS_DELTA = 1,      /* delta_q (search.py:195)                           */
  IVRQ_QS_CODE_SUM = 2,   /* code_sum_q (search.py:104, 208)                   */
  IVRQ_QS_IP_MARGIN = 3,  /* ip_margin (search.py:213)                         */
  IVRQ_QS_KB_SUM = 4,     /* k_b * sum_q used by the refine (search.py:323)    */
  IVRQ_QS_HALF_CODE = 5,  /* 0.5 * code_sum_q (search.py:281)                  */
  IVRQ_QS_SLICE_EXP = 6,  /* e: q_rot ~ sum_s slice_s * 128^(7-s) * 2^(e-55)   */
  IVRQ_QS_L1 = 7,         /* sum |q_rot| (bounds of the certified LUT stage 1)   */
  IVRQ_QS_COUNT = 8
};

/* ---------------------------------------------------------------- misc */
IVRQ_API int ivrq_abi_version(void);
IVRQ_API const char* ivrq_last_error(void);
/* Number of SMs of `device` (synchronous; for host-side grid sizing). */
IVRQ_API int ivrq_device_sm_count(int device, int* out);

/* Return the library's cached scratch memory on the current device to the driver
 * (synchronises `stream` first).  Scratch comes from a private stream-ordered pool
 * that keeps up to IVRQ_POOL_KEEP_BYTES (default 4 GiB) mapped between calls; the
 * process-wide default CUDA pool is never reconfigured. */
IVRQ_API int ivrq_release_memory(void* stream);

/* Enqueue on `stream` a wait until *flag >= value (cuStreamWaitValue32, GEQ).  `flag` is a
 * word of page-locked host memory that the host raises once it has staged a piece of a
 * query batch; search_batch enqueues the whole search first and publishes the pieces as
 * they are copied (host-side pipeline of reference search.py:390-454).  IVRQ_EUNSUP when
 * the driver has no stream memory operations (the caller then stages before enqueueing). */
IVRQ_API int ivrq_stream_wait_flag(const uint32_t* flag, uint32_t value, void* stream);

/* Copy `rows` rows of `row_bytes` from host `src` into page-locked `dst` on `nthreads` native
 * threads, in `npieces` row pieces: thread t copies part t of each piece in piece order, then
 * atomically increments flags[p] (page-locked, npieces words, zeroed here).  Piece p is staged
 * once flags[p] == nthreads: a stream waits for it with ivrq_stream_wait_flag(flags + p,
 * nthreads), the host with ivrq_stage_wait.  Returns at once; ivrq_stage_join(*handle) joins
 * the threads (call it exactly once, after which src may be released). */
IVRQ_API int ivrq_stage_rows(void* dst, const void* src, int64_t rows, int64_t row_bytes, int32_t npieces,
                             int32_t nthreads, uint32_t* flags, void** handle);
IVRQ_API int ivrq_stage_wait(const uint32_t* flags, int32_t piece, int32_t nthreads);
IVRQ_API int ivrq_stage_join(void* handle);

/* Bytes per vector of the rcodes layout (0 for bits == 1). */
IVRQ_API int64_t ivrq_rcode_row_bytes(int32_t dims, int32_t bits);

/* Row-wise np.einsum("ij,ij->i", X, X) in float64, bit-exact to NumPy's
 * 2-lane reduction order.  Replaces Centroids.from_values
 * (clustering.py:26-30) and the x_sq/q_sq terms (clustering.py:49, search.py:240).
 * x_is_f64: 0 -> x is float[n*d], 1 -> x is double[n*d]. */
IVRQ_API int ivrq_row_sqnorms(const void* x, int x_is_f64, int64_t n, int32_t d, double* out,
                     void* stream);

/* out[m][n] = sum_k a[m][k] * b[n][k] in float64 (rotate(), linalg.py:43-50).
 * a_is_f64/b_is_f64 select float or double operands. */
IVRQ_API int ivrq_matmul_nt(const void* a, int a_is_f64, const void* b, int b_is_f64, int64_t m,
                            int64_t n, int32_t k, double* out, void* stream);

/* ---------------------------------------------------------------- search */
/* q_rot = q @ rotation^T in float64 (search.py:422, prepare_query 217-223).
 * q_is_f64: 0 -> q float[nq*d], 1 -> q double[nq*d]. */
IVRQ_API int ivrq_rotate_queries(const void* q, int q_is_f64, int64_t nq, int32_t dims,
                        const float* rotation, double* q_rot, void* stream);

/* Exact n_probe nearest centroids (select_clusters, search.py:226-244):
 * d = max((|q|^2 + |c|^2) - 2<q,c>, 0) in float64, ties to the smaller id.
 * Writes ids/d2 [nq*n_probe] in ascending (distance, id) order.
 * Workspace: ivrq_select_clusters_workspace(nq, n_clusters) bytes. */
IVRQ_API size_t ivrq_select_clusters_workspace(int64_t nq, int32_t n_clusters);
IVRQ_API int ivrq_select_clusters(const double* q_rot, int64_t nq, int32_t dims, const float* centroids,
                         const double* centroid_sqnorms, int32_t n_clusters, int32_t n_probe,
                         int64_t* ids, double* d2, void* workspace, size_t workspace_bytes,
                         void* stream);
/* Same selection, written in ascending cluster-id order when order_by_id != 0
 * (the order in which search_batch visits the probes, search.py:429). */
IVRQ_API int ivrq_select_clusters_ordered(const double* q_rot, int64_t nq, int32_t dims,
                                 const float* centroids, const double* centroid_sqnorms,
                                 int32_t n_clusters, int32_t n_probe, int32_t order_by_id,
                                 int64_t* ids, double* d2, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* Same selection against float64 centroids (select_clusters takes any Centroids,
 * e.g. train_kmeans' float64 output): the float64 GEMM (DMMA) path. */
IVRQ_API int ivrq_select_clusters_f64(const double* q_rot, int64_t nq, int32_t dims, const double* centroids,
                                      const double* centroid_sqnorms, int32_t n_clusters, int32_t n_probe,
                                      int32_t order_by_id, int64_t* ids, double* d2, void* workspace,
                                      size_t workspace_bytes, void* stream);

/* Per-query state (_prepare_from_rotated, search.py:186-214; build_luts 115-132).
 * scalars: double[nq*IVRQ_QS_COUNT]; planes: uint32[nq*query_bits*g] (bitwise
 * mode, else may be NULL); luts: float[nq*8*g*16] (lut mode, else may be NULL);
 * qslices: int8[nq*8*kpad] (refine of a multi-bit index, else may be NULL):
 * q_rot as a 55-bit fixed-point number split into 8 balanced base-128 digits,
 * laid out in the K order of the refine's int8 MMA fragments. */
IVRQ_API int ivrq_prepare_queries(const double* q_rot, int64_t nq, int32_t dims,
                         const ivrq_search_params* params, int32_t index_bits, double eps_bound,
                         double* scalars, uint32_t* planes, float* luts, int8_t* qslices,
                         void* stream);

/* The fused two-stage list scan + top-k (the per-query loop of search_batch,
 * search.py:425-448, with cluster_local_search 326-375 and merge_topk 378-387).
 * Each query visits its probed lists in ascending cluster id and carries its
 * pruning threshold from list to list exactly as the reference does.
 * probe_ids/probe_d2: [nq*n_probe] as written by ivrq_select_clusters_ordered
 * (ascending id).  scalars/planes/luts/qslices come from ivrq_prepare_queries;
 * q_rot is not read (the refine uses the exact digit slices of q_rot).
 * Outputs: out_ids int64[nq*k], out_dists double[nq*k] (ascending (dist, id)),
 * out_counts int32[nq]; stats (may be NULL) int64[nq*2] = (vectors probed,
 * stage-1 survivors) per query. */
IVRQ_API int ivrq_search_scan(const ivrq_index_view* index, const double* q_rot,
                              const int64_t* probe_ids, const double* probe_d2,
                              const double* scalars, const uint32_t* planes, const float* luts,
                              const int8_t* qslices, int64_t nq, const ivrq_search_params* params,
                              int64_t* out_ids, double* out_dists, int32_t* out_counts,
                              int64_t* stats, void* stream);

/* List-sharded scan: the index holds global clusters [list_lo, list_hi) renumbered
 * from 0; probes outside the range are skipped.  init_ids/init_dists/init_counts
 * (all NULL or all given; [nq*k] ascending, counts [nq]) seed each query's pool and
 * threshold -- shard g continuing the ascending-id walk of shard g-1 reproduces
 * search.py:429-447 exactly across GPUs. */
IVRQ_API int ivrq_search_scan_shard(const ivrq_index_view* index, int64_t list_lo, int64_t list_hi,
                                    const double* q_rot, const int64_t* probe_ids,
                                    const double* probe_d2, const double* scalars,
                                    const uint32_t* planes, const float* luts, const int8_t* qslices,
                                    int64_t nq, const ivrq_search_params* params,
                                    const int64_t* init_ids, const double* init_dists,
                                    const int32_t* init_counts, int64_t* out_ids, double* out_dists,
                                    int32_t* out_counts, int64_t* stats, void* stream);

/* Merge `parts` (<= 16) per-query top-k lists laid out [parts][nq][k] (ascending,
 * counts [parts][nq]) into the k best by (dist, id) (merge_topk, search.py:378-387):
 * the all-gather merge of list-sharded search. */
IVRQ_API int ivrq_merge_topk(const int64_t* ids, const double* dists, const int32_t* counts,
                             int64_t nq, int32_t parts, int32_t k, int64_t* out_ids,
                             double* out_dists, int32_t* out_counts, void* stream);

/* ---------------------------------------------------------------- sub-operators
 * The reference's finer-grained API (search.py:84-375, codec.py:118-151, 262-303,
 * 383-401), one call per operator.  All pointers are device pointers. */

/* ip_bitwise (search.py:163-183): words uint32[groups*n] laid out (groups, n)
 * (a list's interleaved slice), planes uint32[query_bits*groups]; out int64[n]. */
IVRQ_API int ivrq_ip_bitwise(const uint32_t* words, int32_t groups, int64_t n, const uint32_t* planes,
                             int32_t query_bits, int64_t* out, void* stream);

/* ip_lut (search.py:146-160): nibbles uint8[n*blocks], luts float[blocks*16]; out double[n]. */
IVRQ_API int ivrq_ip_lut(const uint8_t* nibbles, int64_t n, int32_t blocks, const float* luts, double* out,
                         void* stream);

/* estimate_stage1 (search.py:270-287): ip double[n], short_factors double[n*3]
 * (add, scale, err), d_qc2 double[n]; est2/lb2 double[n]. */
IVRQ_API int ivrq_estimate_stage1(const double* ip, const double* short_factors, int64_t n, const double* d_qc2,
                                  double code_sum_q, double ip_margin, double* est2, double* lb2, void* stream);

/* refine_stage2 (search.py:290-310): ex double[n*dims] ex-code values, ip_binary
 * double[n], long_factors double[n*2], q_rot double[dims], d_qc2 double[n]; out double[n].
 * bits < 2 -> IVRQ_EINVAL (no ex-code exists for 1-bit indexes). */
IVRQ_API int ivrq_refine_stage2(const double* ex, int64_t n, int32_t dims, const double* ip_binary,
                                const double* long_factors, const double* q_rot, double sum_q, const double* d_qc2,
                                int32_t bits, double* out, void* stream);

/* cluster_local_search (search.py:326-375) for one query and one cluster: stage-1
 * estimates, prune lb2 <= threshold, refinement of the survivors, local top-k by
 * (dist, pid).  qstate: HOST double[IVRQ_QS_COUNT] (sum_q, delta, code_sum, ip_margin);
 * planes (bitwise) / luts (lut) as ivrq_prepare_queries writes them for one query
 * (device); d_qc2: HOST pointer to the squared query-centroid distance, or NULL
 * (then computed on the device from the centroid).  Outputs out_ids int64[k],
 * out_dists double[k], out_count int32[1].  list_size = the cluster's row count;
 * workspace: ivrq_cluster_local_search_workspace(list_size) bytes. */
IVRQ_API size_t ivrq_cluster_local_search_workspace(int64_t list_size);
IVRQ_API int ivrq_cluster_local_search(const ivrq_index_view* index, int64_t cluster, const double* q_rot,
                                       const uint32_t* planes, const float* luts, const double* qstate,
                                       const ivrq_search_params* params, double threshold, const double* d_qc2,
                                       int64_t* out_ids, double* out_dists, int32_t* out_count, void* workspace,
                                       size_t workspace_bytes, int64_t list_size, void* stream);

/* compute_factors_batch (codec.py:322-380): u uint8[n*dims], o double[n*dims],
 * dist double[n], c_rot double[n*dims]; short_factors double[n*3], long_factors
 * double[n*2], low_quality uint8[n]. */
IVRQ_API int ivrq_compute_factors(const uint8_t* u, const double* o, const double* dist, const double* c_rot,
                                  int64_t n, int32_t dims, int32_t bits, double eps_bound, double* short_factors,
                                  double* long_factors, uint8_t* low_quality, void* stream);

/* normalize_residuals (codec.py:138-151; dd_norm = 0, einsum-order norm) and
 * normalize_residual (codec.py:118-135; dd_norm = 1, the norm as a double-double
 * dot rounded once): x, c double[n*dims]; o double[n*dims], dist double[n]. */
IVRQ_API int ivrq_normalize_residuals(const double* x, const double* c, int64_t n, int32_t dims, int32_t dd_norm,
                                      double* o, double* dist, void* stream);

/* quantize_oracle (codec.py:262-303) for one vector o double[dims]: out uint8[dims].
 * The host enforces the reference's enumeration guard dims*2^(bits-1) <= 2^15.
 * workspace: ivrq_quantize_oracle_workspace(dims, bits) bytes. */
IVRQ_API size_t ivrq_quantize_oracle_workspace(int32_t dims, int32_t bits);
IVRQ_API int ivrq_quantize_oracle(const double* o, int32_t dims, int32_t bits, uint8_t* out, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- build */
/* k-means++ seeding (_kmeans_pp_init, clustering.py:60-79) on x float[n*d]
 * (values are upcast to float64 exactly as the reference does).  Runs steps
 * j in [j_begin, j_end) given host-drawn randomness:
 *   draw_kind 0: draws[j] is rng.random() (double), used when total > 0;
 *   draw_kind 1: draws[j] is rng.integers(n) (stored as double, exact).
 * When j_begin == 0, draws[0] holds `first` (rng.integers(n)) and d2 is
 * initialised.  zero_step (device int32[1], caller-initialised to -1) receives
 * the first step whose total was <= 0 under draw_kind 0; steps from there on
 * must be re-run with draw_kind 1.  centers: double[n_clusters*d].
 * d2: double[n] state carried between calls.  Temporaries come from the
 * stream-ordered allocator (cudaMallocAsync). */
IVRQ_API int ivrq_kmeanspp(const float* x, int64_t n, int32_t d, int32_t n_clusters, int32_t j_begin,
                  int32_t j_end, const double* draws, int32_t draw_kind, double* centers,
                  double* d2, int32_t* zero_step, void* stream);

/* Nearest-centroid labels (_label_chunks / assign, clustering.py:41-57, 116-125):
 * d = (x_sq + c_sq) - 2<x,c> in float64, argmin ties to the smaller id,
 * dmin = max(d[label], 0).  centers double[k*d]; labels int32[n]; dmin may be NULL. */
IVRQ_API int ivrq_assign(const float* x, int64_t n, int32_t d, const double* centers,
                const double* centroid_sqnorms, int32_t k, int32_t* labels, double* dmin,
                void* stream);

/* Stable counting sort by label (np.bincount + np.argsort(kind="stable"),
 * index.py:226-229, clustering.py:99-109): counts int64[k], offsets int64[k+1],
 * order int64[n] (row ids, ascending within a label). */
IVRQ_API int ivrq_counting_sort(const int32_t* labels, int64_t n, int32_t k, int64_t* counts,
                       int64_t* offsets, int64_t* order, void* stream);

/* Empty-cluster reseeding of one Lloyd iteration (clustering.py:100-107):
 * for each empty cluster j in ascending order, the first row with maximal
 * dmin gets label j and dmin -1.  counts are updated in place.
 * n_empty_out (device int32[1]) receives the number of empties. */
IVRQ_API int ivrq_kmeans_reseed(int32_t* labels, double* dmin, int64_t n, int64_t* counts, int32_t k,
                       int32_t* n_empty_out, void* stream);

/* Centroid update: centers[c] = (sequential row-order sum of x[order[...]] over
 * the segment of c) / counts[c]  (np.add.reduceat + divide, clustering.py:108-112),
 * including reduceat's rule for an empty segment (the single row at its start). */
IVRQ_API int ivrq_kmeans_update(const float* x, int64_t n, const int64_t* order, const int64_t* offsets,
                       int32_t k, int32_t d, double* centers, void* stream);

/* Data-parallel form of the centroid update for ranks that own ascending row blocks:
 * per cluster c, the sequential sum continues from init_sums[c] (after init_counts[c]
 * rows of earlier ranks; both NULL on the first rank) over this rank's rows of c
 * (order/offsets from ivrq_counting_sort of the local labels), so the chain over ranks
 * reproduces np.add.reduceat's row order exactly.  total_counts NULL: out = running
 * sums double[k*d], out_counts = running counts (for the next rank); otherwise out =
 * centres (sum / total_counts[c]). */
IVRQ_API int ivrq_kmeans_chain_sums(const float* x, const int64_t* order, const int64_t* offsets, int32_t k,
                                    int32_t d, const double* init_sums, const int64_t* init_counts,
                                    const int64_t* total_counts, double* out, int64_t* out_counts, void* stream);

/* Residual normalisation + rotation (normalize_residuals codec.py:138-151;
 * index.py:237-238): for output row r, source row s = order[r] and centroid
 * c = labels[s]: diff = x[s] - cent32[c] (float64), dist[r] = sqrt(einsum(diff,diff)),
 * o = diff / dist (0 for a degenerate row), o_rot[r] = float32(o @ rotation^T)
 * with float64 accumulation. */
IVRQ_API int ivrq_normalize_rotate(const float* x, const int64_t* order, const int32_t* labels,
                          const float* cent32, const float* rotation, int64_t n, int32_t d,
                          float* o_rot, double* dist, void* stream);

/* cent_rot = float32(cent32 @ rotation^T) (index.py:235), float64 accumulation. */
IVRQ_API int ivrq_rotate_rows_f32(const float* x, int64_t n, int32_t d, const float* rotation, float* out,
                         void* stream);

/* rcodes of an index given in IVRQ1 arrays (load_index path): u rebuilt from the
 * interleaved MSB plane and the ex-code byte stream (excodes uint8[n*bpv]). */
IVRQ_API int ivrq_make_rcodes(const uint32_t* packed_msb, const int64_t* offsets, int32_t n_clusters,
                              const uint8_t* excodes, int64_t n, int32_t d, int32_t bits,
                              uint8_t* rcodes, void* stream);

/* RaBitQ encoder, one warp per vector (quantize_batch codec.py:204-244,
 * split_planes 306-319, compute_factors_batch 322-380, pack_interleaved 404-413,
 * pack_excodes 432-444), writing the device list layout directly.
 * o_rot float[n*d] or double[n*d] (o_is_f64; the grid search runs in that
 * dtype exactly like NumPy does), unit or zero rows in CSR order, dist double[n], cent_rot
 * float[n_clusters*d], offsets int64[n_clusters+1].
 * Outputs: packed_msb, rcodes (NULL when bits == 1), short SoA, long float2,
 * optionally codes uint8[n*d] (full unsigned codes u) and t float[n].
 * bad_rows (device int32[1], caller-initialised 0) counts rows whose norm
 * differs from 1 by more than 1e-4 (_check_unit_rows, codec.py:154-160). */
IVRQ_API int ivrq_encode(const void* o_rot, int32_t o_is_f64, const double* dist, const float* cent_rot,
                const int64_t* offsets, int32_t n_clusters, int64_t n, int32_t d, int32_t bits,
                int32_t n_coarse, int32_t n_fine, double eps_bound, uint32_t* packed_msb,
                uint8_t* rcodes, float* short_add, float* short_scale, float* short_err,
                float* long_factors, uint8_t* codes, double* t_out, int32_t* bad_rows,
                void* stream);

/* Per-kernel timing for benchmarks (no reference counterpart).  While enabled,
 * the search records CUDA events on the launching stream around its dominant
 * kernels ("tc_refine_kernel", "scan_rd_kernel", "scan_warp_kernel",
 * "tc_ip_kernel", "ip_list_kernel"); enabling starts a new window.
 * ivrq_kernel_time waits for the recorded events of `name` and returns their
 * summed duration and launch count. */
IVRQ_API int ivrq_kernel_timing(int32_t enable);
IVRQ_API int ivrq_kernel_time(const char* name, double* total_ms, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* IVRQ_B200_H */
