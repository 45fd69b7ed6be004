// Stand-alone check of the tcgen05 kind::i8 primitives in ivrq_tc.cuh:
// D[128 x N] = A[128 x K] (u8) * B[N x K]^T (s8), int32, against the CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/tcp tools/tc_probe.cu && /tmp/tcp
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cudaTypedefs.h>

#include "../paper_2602_23999_b200/csrc/ivrq_tc.cuh"

namespace ivrq {
namespace tc {
bool make_tmap_u8_sw128(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t row_stride,
                        uint32_t box_inner, uint32_t box_outer) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn) return false;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_stride};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace tc
}  // namespace ivrq

using namespace ivrq;

constexpr int M = 128;

template <int N, int K>
__global__ void __launch_bounds__(128) probe(const uint8_t* A, const int8_t* B, int* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint8_t* sa = sm;
  int8_t* sb = reinterpret_cast<int8_t*>(sm + M * K);
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, wid = tid >> 5;
  for (int i = tid; i < M * K; i += 128) sa[tc::kmajor_offset(i / K, i % K, M)] = A[i];
  for (int i = tid; i < N * K; i += 128) sb[tc::kmajor_offset(i / K, i % K, N)] = B[i];
  if (wid == 0) tc::tmem_alloc(&taddr_s, N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_smem_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t taddr = taddr_s;
  if (tid == 0) {
    constexpr uint32_t idesc = tc::idesc_i8(M, N, false, true);
    for (int s = 0; s < K / 32; ++s) {
      const uint64_t ad = tc::smem_desc(sa + 2 * s * M * 16, M * 16, 128);
      const uint64_t bd = tc::smem_desc(sb + 2 * s * N * 16, N * 16, 128);
      tc::mma_i8(taddr, ad, bd, idesc, s > 0);
    }
    tc::commit(&bar);
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(taddr + ((uint32_t)(wid * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(wid * 32 + (tid & 31)) * N + c0 + j] = (int)v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(taddr, N < 32 ? 32 : N);
}

// TMA (128B swizzle) + SW128 descriptors: A [128 x K] u8, B [N x K] s8 row-major in global
template <int N, int K>
__global__ void __launch_bounds__(128) probe_tma(const __grid_constant__ CUtensorMap ma,
                                                  const __grid_constant__ CUtensorMap mb, int* D) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;                                        // [K/128][128 rows x 128 B]
  int8_t* sb = reinterpret_cast<int8_t*>(sm + (K / 128) * M * 128);  // [K/128][N rows x 128 B]
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, wid = tid >> 5;
  if (wid == 0) tc::tmem_alloc(&taddr_s, N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    tc::mbar_expect_tx(&bar, (K / 128) * (M + N) * 128);
    for (int c = 0; c < K / 128; ++c) {
      tc::tma_load_2d(sa + c * M * 128, &ma, c * 128, 0, &bar);
      for (int r0 = 0; r0 < N; r0 += 128) tc::tma_load_2d(sb + c * N * 128 + r0 * 128, &mb, c * 128, r0, &bar);
    }
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  const uint32_t taddr = taddr_s;
  if (tid == 0) {
    constexpr uint32_t idesc = tc::idesc_i8(M, N, false, true);
    for (int s = 0; s < K / 32; ++s) {
      const int c = s / 4, off = (s % 4) * 32;
      const uint64_t ad = tc::smem_desc_sw128(sa + c * M * 128 + off);
      const uint64_t bd = tc::smem_desc_sw128(sb + c * N * 128 + off);
      tc::mma_i8(taddr, ad, bd, idesc, s > 0);
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(taddr + ((uint32_t)(wid * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(wid * 32 + (tid & 31)) * N + c0 + j] = (int)v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(taddr, N < 32 ? 32 : N);
}

template <int N, int K>
int run_tma() {
  std::vector<uint8_t> A(M * K);
  std::vector<int8_t> B(N * K);
  srand(7);
  for (auto& x : A) x = rand() & 255;
  for (auto& x : B) x = (int8_t)(rand() & 255);
  uint8_t* dA;
  int8_t* dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  CUtensorMap ma, mb;
  if (!tc::make_tmap_u8_sw128(&ma, dA, K, M, K, 128, 128) || !tc::make_tmap_u8_sw128(&mb, dB, K, N, K, 128, N < 128 ? N : 128)) {
    printf("tensor map encode failed\n");
    return 1;
  }
  const int smem = (K / 128) * (M + N) * 128 + 1024;
  cudaFuncSetAttribute(probe_tma<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_tma<N, K><<<1, 128, smem>>>(ma, mb, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("TMA N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> D(M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long long s = 0;
      for (int k = 0; k < K; ++k) s += (long long)A[i * K + k] * B[j * K + k];
      if (s != D[i * N + j]) {
        if (bad < 5) printf("  mismatch (%d,%d): gpu %d cpu %lld\n", i, j, D[i * N + j], s);
        ++bad;
      }
    }
  printf("TMA/SW128 N=%d K=%d: %d mismatches of %d\n", N, K, bad, M * N);
  return bad != 0;
}

// TS form: A (128 x K, u8) TMA-loaded (SW128) then tcgen05.cp'd into TMEM, B (N x K, s8) from smem
template <int N, int K>
__global__ void __launch_bounds__(128) probe_ts(const __grid_constant__ CUtensorMap ma,
                                                 const __grid_constant__ CUtensorMap mb, int* D) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sa = sm;
  int8_t* sb = reinterpret_cast<int8_t*>(sm + (K / 128) * M * 128);
  __shared__ uint64_t bar, mbar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, wid = tid >> 5;
  constexpr int ACOLS = K / 4;  // A in TMEM: K bytes per lane
  constexpr int NC = (ACOLS + N) <= 32 ? 32 : (ACOLS + N) <= 64 ? 64 : (ACOLS + N) <= 128 ? 128 : (ACOLS + N) <= 256 ? 256 : 512;
  if (wid == 0) tc::tmem_alloc(&taddr_s, NC);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&mbar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    tc::mbar_expect_tx(&bar, (K / 128) * (M + N) * 128);
    for (int c = 0; c < K / 128; ++c) {
      tc::tma_load_2d(sa + c * M * 128, &ma, c * 128, 0, &bar);
      for (int r0 = 0; r0 < N; r0 += 128) tc::tma_load_2d(sb + c * N * 128 + r0 * 128, &mb, c * 128, r0, &bar);
    }
  }
  tc::mbar_wait(&bar, 0);
  tc::fence_after_sync();
  const uint32_t taddr = taddr_s;
  const uint32_t ta = taddr + N;  // A columns after the accumulator
  if (tid == 0) {
    for (int s = 0; s < K / 32; ++s) {
      const int c = s / 4, off = (s % 4) * 32;
      tc::tmem_cp_128x256b(ta + 8 * s, tc::smem_desc_sw128(sa + c * M * 128 + off));
    }
    constexpr uint32_t idesc = tc::idesc_i8(M, N, false, true);
    for (int s = 0; s < K / 32; ++s) {
      const int c = s / 4, off = (s % 4) * 32;
      tc::mma_i8_ts(taddr, ta + 8 * s, tc::smem_desc_sw128(sb + c * N * 128 + off), idesc, s > 0);
    }
    tc::commit(&mbar);
  }
  tc::mbar_wait(&mbar, 0);
  tc::fence_after_sync();
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    tc::tmem_ld32(taddr + ((uint32_t)(wid * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int j = 0; j < 32; ++j) D[(wid * 32 + (tid & 31)) * N + c0 + j] = (int)v[j];
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(taddr, NC);
}

template <int N, int K>
int run_ts() {
  std::vector<uint8_t> A(M * K);
  std::vector<int8_t> B(N * K);
  srand(11);
  for (auto& x : A) x = rand() & 255;
  for (auto& x : B) x = (int8_t)(rand() & 255);
  uint8_t* dA;
  int8_t* dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  CUtensorMap ma, mb;
  tc::make_tmap_u8_sw128(&ma, dA, K, M, K, 128, 128);
  tc::make_tmap_u8_sw128(&mb, dB, K, N, K, 128, N < 128 ? N : 128);
  const int smem = (K / 128) * (M + N) * 128 + 1024;
  cudaFuncSetAttribute(probe_ts<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe_ts<N, K><<<1, 128, smem>>>(ma, mb, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("TS N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> Dh(M * N);
  cudaMemcpy(Dh.data(), dD, Dh.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long long sacc = 0;
      for (int k = 0; k < K; ++k) sacc += (long long)A[i * K + k] * B[j * K + k];
      if (sacc != Dh[i * N + j]) {
        if (bad < 5) printf("  mismatch (%d,%d): gpu %d cpu %lld\n", i, j, Dh[i * N + j], sacc);
        ++bad;
      }
    }
  printf("TS (A in TMEM via tcgen05.cp) N=%d K=%d: %d mismatches of %d\n", N, K, bad, M * N);
  return bad != 0;
}

// throughput: every SM issues REPS x (K/32) MMAs (M=128, N, K=32) from smem into one accumulator
template <int N>
__global__ void __launch_bounds__(128) mma_rate(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, wid = tid >> 5;
  for (int i = tid; i < (128 + N) * 128; i += 128) sm[i] = (unsigned char)(i * 7);
  if (wid == 0) tc::tmem_alloc(&taddr_s, N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_smem_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_i8(M, N, false, true);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int s2 = 0; s2 < 4; ++s2)
        tc::mma_i8(taddr_s, tc::smem_desc_sw128(sm + 32 * s2), tc::smem_desc_sw128(sm + 128 * 128 + 32 * s2), idesc,
                   r | s2);
    const long long t1 = clock64();
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    const long long t2 = clock64();
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = t2 - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(taddr_s, N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
}

// same, but A cycles through 6 distinct 16 KB stage tiles and B walks 6 distinct 128-byte K chunks
// (the refine kernel's smem footprint), optionally with TMA refilling the A stages concurrently
template <int N>
__global__ void __launch_bounds__(384) mma_rate_stream(long long* out, int reps, const __grid_constant__ CUtensorMap ma,
                                                       int with_tma) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = sm;                 // 6 x 16 KB
  constexpr int SB = N <= 128 ? 6 : 2;   // B chunks resident (smem budget)
  unsigned char* sb = sm + 6 * 128 * 128; // SB x N x 128
  __shared__ uint64_t bar, tbar, cbar, tbar2;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, wid = tid >> 5;
  for (int i = tid; i < (6 * 128 + SB * N) * 128; i += blockDim.x) sm[i] = (unsigned char)(i * 7);
  if (wid == 0) tc::tmem_alloc(&taddr_s, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::mbar_init(&tbar, 1);
    tc::mbar_init(&cbar, 1);
    tc::mbar_init(&tbar2, 1);
    tc::mbar_arrive(&tbar2);  // phase 0 completes
    tc::fence_mbar_init();
  }
  tc::fence_smem_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_i8(M, N, false, true);
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int st = r % 6;
      if (with_tma & 8) tc::fence_after_sync();  // the refine kernel's per-stage fence
      if (with_tma & 16) tc::mbar_wait(&tbar2, 0);  // a (satisfied) barrier wait per stage
      for (int s2 = 0; s2 < 4; ++s2)
        tc::mma_i8(taddr_s, tc::smem_desc_sw128(sa + st * 16384 + 32 * s2),
                   tc::smem_desc_sw128(sb + (st % SB) * N * 128 + 32 * s2), idesc, r | s2);
      if (with_tma & 2) tc::commit(&cbar);  // a commit per stage, as in the refine kernel
    }
    const long long t1 = clock64();
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[2 * blockIdx.x] = t1 - t0;
    out[2 * blockIdx.x + 1] = clock64() - t0;
  } else if (wid >= 2 && (with_tma & 32)) {
    // epilogue-like load: tcgen05.ld of 32 columns, int64 assembly and float64 arithmetic, global stores
    const int q4 = wid & 3;
    double acc = 1.0;
    for (int r = 0; r < reps / 2; ++r) {
      uint32_t v[32];
      tc::tmem_ld32(taddr_s + ((uint32_t)(q4 * 32) << 16) + 256 + (r % 4) * 32, v);
      tc::tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const long long hi = (long long)(int)v[4 * j] * 2097152LL + (long long)(int)v[4 * j + 1] * 16384LL +
                             (long long)(int)v[4 * j + 2] * 128LL + (int)v[4 * j + 3];
        acc = __dadd_rn(__dmul_rn((double)hi, 0x1p-30), __dmul_rn(acc, 0.999));
      }
    }
    if (acc == 12345.0) out[0] = (long long)acc;
  } else if (wid >= 2 && (with_tma & 4)) {
    // concurrent TMEM reads of another accumulator region (the epilogue's tcgen05.ld)
    const int q4 = wid & 3;
    for (int r = 0; r < reps / 8; ++r) {
      uint32_t v[32];
      tc::tmem_ld32(taddr_s + ((uint32_t)(q4 * 32) << 16) + 256 + (r % 4) * 32, v);
      tc::tmem_ld_wait();
      if (v[0] == 0xdeadbeef) out[0] = v[1];
    }
  } else if (tid == 32 && (with_tma & 1)) {
    // keep TMA writing 16 KB tiles into a stage (the data race with the MMA is irrelevant for timing)
    for (int r = 0; r < reps / 4; ++r) {
      tc::mbar_expect_tx(&tbar, 16384);
      tc::tma_load_2d(sa + (r % 6) * 16384, &ma, 0, (r * 128) % 4096, &tbar);
      tc::mbar_wait(&tbar, r & 1);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(taddr_s, 512);
}

// MMA rate with the B operand's 8-row atoms spread SBO bytes apart (the refine kernel keeps each
// query's K chunks together, so one chunk's atoms are nkc KB apart)
template <int N>
__global__ void __launch_bounds__(128) mma_rate_sbo(long long* out, int reps, int sbo) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char* sa = sm;            // 3 x 16 KB A stages
  unsigned char* sb = sm + 3 * 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t taddr_s;
  const int tid = threadIdx.x, wid = tid >> 5;
  // pseudo-random operand bytes (rcodes / digit slices look random to the multiplier array)
  for (int i = tid; i < 3 * 16384 + (N / 8) * sbo; i += 128) {
    uint32_t h = (uint32_t)i * 2654435761u;
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    sm[i] = (unsigned char)(sbo < 0 ? 0 : (h >> 24));
  }
  if (wid == 0) tc::tmem_alloc(&taddr_s, 512);
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_mbar_init();
  }
  tc::fence_smem_async();
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if (tid == 0) {
    const uint32_t idesc = tc::idesc_i8(M, N, false, true);
    const int nkc = sbo / 1024;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const int kc = r % nkc;
      for (int s2 = 0; s2 < 4; ++s2)
        tc::mma_i8(taddr_s + (r & 1) * 256, tc::smem_desc_sw128(sa + (r % 3) * 16384 + 32 * s2),
                   tc::smem_desc_sw128_sbo(sb + kc * 1024 + 32 * s2, sbo), idesc, r | s2);
    }
    tc::commit(&bar);
    tc::mbar_wait(&bar, 0);
    out[2 * blockIdx.x + 1] = clock64() - t0;
  }
  tc::fence_before_sync();
  __syncthreads();
  if (wid == 0) tc::tmem_dealloc(taddr_s, 512);
}

template <int N>
void rate_sbo(int sbo) {
  const int reps = 2000, blocks = 148;
  long long* d;
  cudaMalloc(&d, blocks * 16);
  const int smem = 3 * 16384 + (N / 8) * sbo + 1024;
  cudaFuncSetAttribute(mma_rate_sbo<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate_sbo<N><<<blocks, 128, smem>>>(d, reps, sbo);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(2 * blocks);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  printf("B atoms %d B apart N=%d: %.1f clk/MMA (%s)\n", sbo, N, h[1] / (4.0 * reps), cudaGetErrorString(e));
  cudaFree(d);
}

template <int N>
void rate_stream(int with_tma) {
  const int reps = 2000, blocks = 148;
  long long* d;
  cudaMalloc(&d, blocks * 16);
  uint8_t* src;
  cudaMalloc(&src, 4096 * 128);
  cudaMemset(src, 1, 4096 * 128);
  CUtensorMap ma;
  tc::make_tmap_u8_sw128(&ma, src, 128, 4096, 128, 128, 128);
  const int smem = (6 * 128 + (N <= 128 ? 6 : 2) * N) * 128 + 1024;
  cudaFuncSetAttribute(mma_rate_stream<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate_stream<N><<<blocks, (with_tma & 32) ? 384 : 128, smem>>>(d, reps, ma, with_tma);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<long long> h(2 * blocks);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  const double n_mma = 4.0 * reps;
  printf("streamed operands N=%d tma=%d: %.1f clk/MMA (%s)\n", N, with_tma, h[1] / n_mma, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(src);
}

template <int N>
double rate() {
  const int reps = 2000, blocks = 148;
  long long* d;
  cudaMalloc(&d, blocks * 16);
  const int smem = (128 + N) * 128 + 1024;
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  mma_rate<N><<<blocks, 128, smem>>>(d, reps);
  cudaDeviceSynchronize();
  std::vector<long long> h(2 * blocks);
  cudaMemcpy(h.data(), d, h.size() * 8, cudaMemcpyDeviceToHost);
  const double n_mma = 4.0 * reps;
  const double mac = 128.0 * N * 32 / (h[1] / n_mma);
  printf("int8 MMA M=128 N=%d K=32: issue %.1f clk/MMA, complete %.1f clk/MMA -> %.0f MAC/clk/SM\n", N,
         h[0] / n_mma, h[1] / n_mma, mac);
  cudaFree(d);
  return mac;
}

template <int N, int K>
int run() {
  std::vector<uint8_t> A(M * K);
  std::vector<int8_t> B(N * K);
  srand(1);
  for (auto& x : A) x = rand() & 255;
  for (auto& x : B) x = (int8_t)(rand() & 255);
  uint8_t* dA;
  int8_t* dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  const int smem = M * K + N * K;
  cudaFuncSetAttribute(probe<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<N, K><<<1, 128, smem>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d K=%d: CUDA error %s\n", N, K, cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> D(M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long long s = 0;
      for (int k = 0; k < K; ++k) s += (long long)A[i * K + k] * B[j * K + k];
      if (s != D[i * N + j]) {
        if (bad < 5) printf("  mismatch (%d,%d): gpu %d cpu %lld\n", i, j, D[i * N + j], s);
        ++bad;
      }
    }
  printf("N=%d K=%d: %d mismatches of %d\n", N, K, bad, M * N);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad != 0;
}

int main() {
  int rc = 0;
  rc |= run<32, 64>();
  rc |= run<128, 256>();
  rc |= run<256, 128>();
  rc |= run_tma<128, 256>();
  rc |= run_tma<64, 384>();
  rc |= run_tma<256, 128>();
  rc |= run_ts<128, 256>();
  rc |= run_ts<64, 128>();
  rate_stream<128>(0);
  rate_stream<128>(1);
  rate_stream<128>(2);
  rate_stream<128>(4);
  rate_stream<128>(7);
  rate_stream<128>(8);
  rate_stream<128>(16);
  rate_stream<128>(2 | 8 | 16);
  rate_stream<64>(0);
  rate_sbo<224>(1024);
  rate_sbo<224>(2048);
  rate_sbo<224>(4096);
  rate_sbo<224>(6144);
  rate_sbo<128>(6144);
  rate_sbo<64>(6144);
  rate_stream<224>(0);
  rate_stream<224>(2 | 8 | 16);
  rate_stream<128>(32);
  rate_stream<128>(32 | 1);
  rate_stream<208>(0);
  rate_stream<208>(32);
  rate_stream<208>(32 | 1 | 2 | 8 | 16);
  rate<64>();
  rate<128>();
  rate<224>();
  const double mac = rate<256>();
  // dense int8 peak of the part: MAC/clk/SM x 2 x SMs x max SM clock (the resident-operand rate)
  int dev = 0, sms = 0, khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  printf("{\"tops\": %.1f, \"mac_per_clk_per_sm\": %.0f, \"sms\": %d, \"sm_clock_mhz\": %.0f, "
         "\"how\": \"tools/tc_probe.cu: 148 CTAs x 8000 back-to-back tcgen05.mma.cta_group::1.kind::i8 M=128 N=256 K=32 "
         "from resident shared-memory operands, clock64 issue-to-commit\"}\n",
         2.0 * mac * sms * khz * 1e3 / 1e12, mac, sms, khz / 1e3);
  return rc;
}
