// Error state, device queries and the einsum-order row norms.
#include "ivrq_common.cuh"

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

// Row-wise einsum("ij,ij->i") with each row staged through shared memory so
// global loads stay coalesced; one thread owns one row's 2-lane chain.
template <typename T>
__global__ void row_sqnorm_kernel(const T* __restrict__ x, int64_t n, int d, double* __restrict__ out) {
  constexpr int ROWS = 64;
  constexpr int CH = 64;  // dims per chunk (multiple of 8 keeps einsum blocks whole)
  __shared__ double tile[ROWS][CH + 1];
  const int64_t row0 = (int64_t)blockIdx.x * ROWS;
  const int r = threadIdx.x;  // blockDim.x == ROWS
  EinsumAcc acc;
  for (int c0 = 0; c0 < d; c0 += CH) {
    const int cw = min(CH, d - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < ROWS * CH; idx += blockDim.x) {
      int rr = idx / CH, cc = idx % CH;
      int64_t gr = row0 + rr;
      double v = 0.0;
      if (gr < n && cc < cw) v = (double)x[gr * d + c0 + cc];
      tile[rr][cc] = v;
    }
    __syncthreads();
    if (row0 + r < n) {
      int i = 0;
      for (; i + 8 <= cw; i += 8) {
        double p[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          double v = tile[r][i + k];
          p[k] = dmul(v, v);
        }
        acc.block8(p);
      }
      for (; i < cw; i += 2) {
        double v0 = tile[r][i];
        bool has1 = (i + 1) < cw;
        double v1 = has1 ? tile[r][i + 1] : 0.0;
        acc.pair(dmul(v0, v0), dmul(v1, v1), has1);
      }
    }
  }
  if (row0 + r < n) out[row0 + r] = acc.result();
}

}  // namespace ivrq

using namespace ivrq;

extern "C" int ivrq_abi_version(void) { return IVRQ_ABI_VERSION; }

extern "C" const char* ivrq_last_error(void) { return g_last_error.c_str(); }

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
  dim3 grid((unsigned)ceil_div(n, 64));
  if (x_is_f64)
    row_sqnorm_kernel<double><<<grid, 64, 0, as_stream(stream)>>>((const double*)x, n, d, out);
  else
    row_sqnorm_kernel<float><<<grid, 64, 0, as_stream(stream)>>>((const float*)x, n, d, out);
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
