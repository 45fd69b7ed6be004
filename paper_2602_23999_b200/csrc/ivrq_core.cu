// Error state, device queries and the einsum-order row norms.
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdlib>
#include <algorithm>
#include <condition_variable>
#if defined(__x86_64__)
#include <emmintrin.h>
#endif
#include <cstring>
#include <deque>
#include <pthread.h>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "ivrq_common.cuh"
#include "ivrq_rowchain.cuh"
#include "ivrq_tc.cuh"

namespace ivrq {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    return fail(IVRQ_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  }
  return IVRQ_OK;
}

cudaMemPool_t library_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    // keep up to min(16 GiB, 1/8 of the device) of freed workspace mapped: a search's buffers (C3
    // ~2.5 GB, C4 ~5 GB) are then reused across calls instead of being unmapped and mapped again
    // at every call; ivrq_release_memory trims the pool on demand
    const char* env = getenv("IVRQ_POOL_KEEP_BYTES");
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    uint64_t keep = env ? strtoull(env, nullptr, 10) : std::min<uint64_t>(uint64_t(16) << 30, total_b / 8);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = pool;
  }
  return pools[dev];
}

cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t s) {
  cudaMemPool_t pool = library_pool();
  if (!pool) return cudaMallocAsync(p, bytes, s);
  return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

namespace tc {
bool make_tmap_u8_sw128(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride,
                        uint32_t box_inner, uint32_t box_outer) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return false;
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tc

namespace {
struct TimedLaunch {
  std::string name;
  cudaEvent_t begin, end;
};
std::mutex g_kt_mu;
std::vector<TimedLaunch> g_kt;
std::atomic<int> g_kt_on{0};
}  // namespace

bool kernel_timing_enabled() { return g_kt_on.load(std::memory_order_relaxed) != 0; }

void kernel_timing_record(const char* name, cudaEvent_t begin, cudaEvent_t end) {
  std::lock_guard<std::mutex> lk(g_kt_mu);
  g_kt.push_back({name, begin, end});
}

cudaStream_t side_stream() {
  static thread_local cudaStream_t streams[32] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 32) return nullptr;
  if (!streams[dev] && cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking) != cudaSuccess) {
    streams[dev] = nullptr;
  }
  return streams[dev];
}

int sm_count_of_current_device() {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) return 148;
  return v;
}

// Row-wise einsum("ij,ij->i", x, x): NumPy's two accumulator lanes run on two
// threads per row over 128-bit staged tiles (ivrq_rowchain.cuh).
template <typename T>
__global__ void __launch_bounds__(rowchain::THREADS) row_sqnorm_kernel(const T* __restrict__ x, int64_t n, int d,
                                                                      double* __restrict__ out) {
  using namespace rowchain;
  __shared__ Tile<T> tile;
  const int64_t row0 = (int64_t)blockIdx.x * ROWS;
  const int r = threadIdx.x >> 1, lane = threadIdx.x & 1;
  const bool vec = (d % Tile<T>::VEC == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  auto src = [&](int64_t gr) { return x + gr * d; };
  double acc = 0.0;
  for (int c0 = 0; c0 < d; c0 += CH) {
    const int cw = min(CH, d - c0);
    __syncthreads();
    stage_tile(tile, src, row0, n, c0, cw, vec);
    __syncthreads();
    acc = chain_chunk(acc, lane, cw, [&](int k) {
      const double v = (double)tile.v[r][k];
      return dmul(v, v);
    });
  }
  const double res = finish(acc);
  if (lane == 0 && row0 + r < n) out[row0 + r] = res;
}

}  // namespace ivrq

using namespace ivrq;

extern "C" int ivrq_abi_version(void) { return IVRQ_ABI_VERSION; }

extern "C" int ivrq_kernel_timing(int32_t enable) {
  std::lock_guard<std::mutex> lk(ivrq::g_kt_mu);
  if (enable) {  // a new measurement window: drop what the previous one recorded
    for (auto& t : ivrq::g_kt) {
      cudaEventSynchronize(t.end);
      cudaEventDestroy(t.begin);
      cudaEventDestroy(t.end);
    }
    ivrq::g_kt.clear();
  }
  ivrq::g_kt_on.store(enable ? 1 : 0);
  return IVRQ_OK;
}

extern "C" int ivrq_kernel_time(const char* name, double* total_ms, int64_t* launches) {
  if (!name || !total_ms || !launches) return ivrq::fail(IVRQ_EINVAL, "ivrq_kernel_time: null argument");
  std::lock_guard<std::mutex> lk(ivrq::g_kt_mu);
  double tot = 0.0;
  int64_t n = 0;
  for (auto& t : ivrq::g_kt) {
    if (t.name != name) continue;
    if (cudaEventSynchronize(t.end) != cudaSuccess) return ivrq::fail(IVRQ_ECUDA, "ivrq_kernel_time: event wait failed");
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, t.begin, t.end) != cudaSuccess)
      return ivrq::fail(IVRQ_ECUDA, "ivrq_kernel_time: elapsed time unavailable");
    tot += ms;
    ++n;
  }
  *total_ms = tot;
  *launches = n;
  return IVRQ_OK;
}

extern "C" const char* ivrq_last_error(void) { return g_last_error.c_str(); }

extern "C" int ivrq_release_memory(void* stream) {
  cudaMemPool_t pool = library_pool();
  if (!pool) return IVRQ_OK;
  if (cudaStreamSynchronize(as_stream(stream)) != cudaSuccess || cudaMemPoolTrimTo(pool, 0) != cudaSuccess)
    return fail(IVRQ_ECUDA, "ivrq_release_memory: pool trim failed");
  return IVRQ_OK;
}

extern "C" int ivrq_stream_wait_flag(const uint32_t* flag, uint32_t value, void* stream) {
  // cuStreamWaitValue32(GEQ) on a page-locked host word: work enqueued after it on `stream`
  // (the H2D copy of a piece of a host batch) starts only once the host has published the
  // piece, so a whole search is enqueued before its queries are staged (search.py pipeline)
  using WaitFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
  static WaitFn wait = nullptr;
  if (!wait) {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(IVRQ_EUNSUP, "ivrq_stream_wait_flag: cuStreamWaitValue32 unavailable");
    wait = reinterpret_cast<WaitFn>(fn);
  }
  if (!flag) return fail(IVRQ_EINVAL, "ivrq_stream_wait_flag: null flag");
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, const_cast<uint32_t*>(flag), 0) != cudaSuccess) {
    cudaGetLastError();
    return fail(IVRQ_EINVAL, "ivrq_stream_wait_flag: flag is not in page-locked host memory");
  }
  if (wait(reinterpret_cast<CUstream>(as_stream(stream)), reinterpret_cast<CUdeviceptr>(dptr), value,
           CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
    return fail(IVRQ_EUNSUP, "ivrq_stream_wait_flag: stream wait rejected by the driver");
  return IVRQ_OK;
}

namespace {
// A host batch copied into page-locked memory by native threads, piece by piece.  The batch is cut
// into (piece, part) tasks queued piece-major on a persistent worker pool; a task copies its rows
// and then raises its piece's flag word by one (release), so flags[p] == nparts once piece p is
// staged.  No Python (and no GIL) is on the publish path: a stream waiting on the flags can never
// wait on the interpreter.  The workers live for the process (threads that exit per call unmap
// their stacks, and the TLB shootdowns measurably slowed the DMA reading the staged rows).
// Copy with non-temporal stores, then drain them.  The DMA that reads the staged rows must not find
// them dirty in the cores' private caches (snooping them back ran the H2D copy of the last-staged
// rows at ~1/3 of the rate of rows already written back).
void stream_copy(char* dst, const char* src, size_t bytes) {
#if defined(__x86_64__)
  size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head > bytes) head = bytes;
  if (head) std::memcpy(dst, src, head);
  dst += head;
  src += head;
  bytes -= head;
  size_t i = 0;
  for (; i + 64 <= bytes; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), e);
  }
  if (i < bytes) std::memcpy(dst + i, src + i, bytes - i);
  _mm_sfence();
#else
  std::memcpy(dst, src, bytes);
#endif
}

struct StageJob {
  std::atomic<int64_t> left{0};
  std::mutex mu;
  std::condition_variable cv;
};
struct StageTask {
  StageJob* job;
  char* dst;
  const char* src;
  size_t bytes;
  uint32_t* flag;
};
struct StagePool {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<StageTask> q;
  int workers = 0;
  void grow(int n) {  // under mu
    for (; workers < n; ++workers) {
      std::thread([this]() { run(); }).detach();
    }
  }
  void run() {
    for (;;) {
      StageTask t;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [this]() { return !q.empty(); });
        t = q.front();
        q.pop_front();
      }
      if (t.bytes) stream_copy(t.dst, t.src, t.bytes);
      __atomic_fetch_add(t.flag, 1u, __ATOMIC_SEQ_CST);
      {  // under the job's lock: ivrq_stage_join frees the job as soon as it sees left == 0
        std::lock_guard<std::mutex> lk(t.job->mu);
        if (t.job->left.fetch_sub(1) == 1) t.job->cv.notify_all();
      }
    }
  }
};
StagePool* g_stage_pool = nullptr;
void stage_pool_after_fork() { g_stage_pool = new StagePool(); }  // the child has none of the workers
StagePool& stage_pool() {
  static std::once_flag once;
  std::call_once(once, []() {
    g_stage_pool = new StagePool();  // never destroyed: the detached workers outlive main()
    pthread_atfork(nullptr, nullptr, stage_pool_after_fork);
  });
  return *g_stage_pool;
}
}  // namespace

extern "C" int ivrq_stage_rows(void* dst, const void* src, int64_t rows, int64_t row_bytes, int32_t npieces,
                               int32_t nthreads, uint32_t* flags, void** handle) {
  if (!handle) return fail(IVRQ_EINVAL, "ivrq_stage_rows: null handle");
  *handle = nullptr;
  if (rows < 0 || row_bytes <= 0 || npieces < 1 || nthreads < 1 || nthreads > 256 || !flags ||
      (rows > 0 && (!dst || !src)))
    return fail(IVRQ_EINVAL, "ivrq_stage_rows: bad arguments");
  for (int p = 0; p < npieces; ++p) __atomic_store_n(flags + p, 0u, __ATOMIC_RELEASE);
  auto* job = new StageJob();
  job->left = (int64_t)npieces * nthreads;
  char* d = static_cast<char*>(dst);
  const char* sp = static_cast<const char*>(src);
  StagePool& pool = stage_pool();
  {
    std::lock_guard<std::mutex> lk(pool.mu);
    try {
      pool.grow(nthreads);
    } catch (...) {
      if (pool.workers == 0) {
        delete job;
        return fail(IVRQ_ECUDA, "ivrq_stage_rows: could not start the staging threads");
      }
    }
    for (int p = 0; p < npieces; ++p) {
      const int64_t x = rows * p / npieces, y = rows * (p + 1) / npieces;
      for (int t = 0; t < nthreads; ++t) {
        const int64_t u = x + (y - x) * t / nthreads, v = x + (y - x) * (t + 1) / nthreads;
        pool.q.push_back({job, d + u * row_bytes, sp + u * row_bytes, (size_t)((v - u) * row_bytes), flags + p});
      }
    }
  }
  pool.cv.notify_all();
  *handle = job;
  return IVRQ_OK;
}

extern "C" int ivrq_stage_wait(const uint32_t* flags, int32_t piece, int32_t nthreads) {
  // host-side wait for one piece (used when the driver has no stream memory operations)
  while (__atomic_load_n(flags + piece, __ATOMIC_ACQUIRE) < (uint32_t)nthreads) std::this_thread::yield();
  return IVRQ_OK;
}

extern "C" int ivrq_stage_join(void* handle) {
  auto* job = static_cast<StageJob*>(handle);
  if (!job) return IVRQ_OK;
  {
    std::unique_lock<std::mutex> lk(job->mu);
    job->cv.wait(lk, [job]() { return job->left.load() == 0; });
  }
  delete job;
  return IVRQ_OK;
}

extern "C" int ivrq_device_sm_count(int device, int* out) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return fail(IVRQ_ECUDA, std::string("ivrq_device_sm_count: ") + cudaGetErrorString(e));
  *out = v;
  return IVRQ_OK;
}

extern "C" int ivrq_row_sqnorms(const void* x, int x_is_f64, int64_t n, int32_t d, double* out,
                                void* stream) {
  if (n < 0 || d < 0) return fail(IVRQ_EINVAL, "ivrq_row_sqnorms: negative size");
  if (n == 0) return IVRQ_OK;
  dim3 grid((unsigned)ceil_div(n, rowchain::ROWS));
  if (x_is_f64)
    row_sqnorm_kernel<double><<<grid, rowchain::THREADS, 0, as_stream(stream)>>>((const double*)x, n, d, out);
  else
    row_sqnorm_kernel<float><<<grid, rowchain::THREADS, 0, as_stream(stream)>>>((const float*)x, n, d, out);
  return check_launch("ivrq_row_sqnorms");
}

#include "ivrq_gemm.cuh"

namespace ivrq {
struct StoreOutF64 {
  double* out;
  int64_t ld;
  __device__ __forceinline__ void operator()(int64_t r, int64_t c, double v) const { out[r * ld + c] = v; }
};
template <typename TA, typename TB>
static int matmul_nt_t(const void* a, const void* b, int64_t m, int64_t n, int32_t k, double* out, cudaStream_t s) {
  gemm::RowMajor<TA> la{(const TA*)a, m, k};
  gemm::RowMajor<TB> lb{(const TB*)b, n, k};
  StoreOutF64 epi{out, n};
  return gemm::launch_gemm(la, m, lb, n, k, epi, s, "ivrq_matmul_nt");
}
}  // namespace ivrq

extern "C" int ivrq_matmul_nt(const void* a, int a_is_f64, const void* b, int b_is_f64, int64_t m, int64_t n,
                              int32_t k, double* out, void* stream) {
  if (m < 0 || n < 0 || k <= 0) return fail(IVRQ_EINVAL, "ivrq_matmul_nt: bad sizes");
  cudaStream_t s = as_stream(stream);
  if (a_is_f64 && b_is_f64) return matmul_nt_t<double, double>(a, b, m, n, k, out, s);
  if (a_is_f64) return matmul_nt_t<double, float>(a, b, m, n, k, out, s);
  if (b_is_f64) return matmul_nt_t<float, double>(a, b, m, n, k, out, s);
  return matmul_nt_t<float, float>(a, b, m, n, k, out, s);
}
