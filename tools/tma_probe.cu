// TMA streaming throughput on one B200: how fast can one producer thread per SM
// fill a ring of 16 KB shared-memory stages?  (tc_refine_kernel's A operand.)
//
//   mode 0: 2-D box 128 rows x 128 B, 128B swizzle, rows 768 B apart (the rcode layout)
//   mode 1: 1-D bulk copy of 16 KB contiguous bytes
//   mode 2: 2-D box 128 rows x 128 B, 128B swizzle, rows 128 B apart (pre-tiled layout)
//   mode 3: mode 0 issued as 4 boxes of 32 rows
// `window` = bytes each CTA cycles over (small: L2-resident, large: DRAM).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2602_23999_b200/csrc \
//        tools/tma_probe.cu paper_2602_23999_b200/csrc/ivrq_core.cu -lcuda -o tools/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include <vector>

#include "ivrq_tc.cuh"

using namespace ivrq;

constexpr int STAGE = 16384;

__global__ void __launch_bounds__(64) stream_kernel(const __grid_constant__ CUtensorMap m768,
                                                    const __grid_constant__ CUtensorMap m128,
                                                    const __grid_constant__ CUtensorMap m768s, const uint8_t* buf,
                                                    int mode, int ns, int loads, long long window_rows) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[16], empty[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < ns; ++i) {
      tc::mbar_init(&full[i], 1);
      tc::mbar_init(&empty[i], 1);
    }
    tc::fence_mbar_init();
  }
  __syncthreads();
  // this CTA's row window (768-byte rows for modes 0/3; 16 KB chunks for 1/2)
  const long long base_row = (long long)blockIdx.x * window_rows;
  if (tid == 0) {
    for (int i = 0; i < loads; ++i) {
      const int st = i % ns;
      tc::mbar_wait(&empty[st], ((i / ns) & 1) ^ 1);
      tc::mbar_expect_tx(&full[st], STAGE);
      unsigned char* dst = sm + st * STAGE;
      const long long tile = i / 6, kc = i % 6;  // 6 K chunks of 128 B per 768-byte row
      const long long r0 = base_row + (tile * 128) % window_rows;
      if (mode == 0) {
        tc::tma_load_2d(dst, &m768, (int)(kc * 128), (int)r0, &full[st]);
      } else if (mode == 3) {
        for (int p = 0; p < 4; ++p) tc::tma_load_2d(dst + p * 4096, &m768s, (int)(kc * 128), (int)(r0 + 32 * p), &full[st]);
      } else {
        // contiguous 16 KB chunks: chunk index walks the window (same bytes per CTA as mode 0)
        const long long chunk = (base_row * 768 / STAGE) + (i % (window_rows * 768 / STAGE));
        if (mode == 1)
          tc::bulk_load(dst, buf + chunk * STAGE, STAGE, &full[st], 0x1000000000000000ull /*evict normal*/);
        else
          tc::tma_load_2d(dst, &m128, 0, (int)(chunk * 128), &full[st]);
      }
    }
  } else if (tid == 32) {
    for (int i = 0; i < loads; ++i) {
      const int st = i % ns;
      tc::mbar_wait(&full[st], (i / ns) & 1);
      tc::mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long total_rows = 1400000;  // ~1.07 GB of 768-byte rows
  uint8_t* buf;
  cudaMalloc(&buf, total_rows * 768 + (1 << 20));
  cudaMemset(buf, 1, total_rows * 768);
  CUtensorMap m768, m128, m768s;
  tc::make_tmap_u8_sw128(&m768, buf, 768, total_rows, 768, 128, 128);
  tc::make_tmap_u8_sw128(&m128, buf, 128, total_rows * 6, 128, 128, 128);
  tc::make_tmap_u8_sw128(&m768s, buf, 768, total_rows, 768, 128, 32);
  const int loads = 3000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const long long windows[2] = {128 * 8, total_rows / sms / 128 * 128};  // 768 KB (L2) | ~7 MB per CTA (DRAM)
  const char* names[4] = {"2D 128x128B pitch768", "1D bulk 16KB", "2D 128x128B pitch128", "2D 4x(32x128B) pitch768"};
  for (int w = 0; w < 2; ++w)
    for (int mode = 0; mode < 4; ++mode)
      for (int ns : {3, 6, 12}) {
        const int smem = ns * STAGE + 1024;
        cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        stream_kernel<<<sms, 64, smem>>>(m768, m128, m768s, buf, mode, ns, loads, windows[w]);  // warm
        cudaEventRecord(e0);
        stream_kernel<<<sms, 64, smem>>>(m768, m128, m768s, buf, mode, ns, loads, windows[w]);
        cudaEventRecord(e1);
        cudaError_t e = cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = (double)sms * loads * STAGE;
        printf("%-26s window %s stages %2d: %7.1f GB/s  (%.3f ms) %s\n", names[mode], w ? "DRAM" : "L2  ", ns,
               bytes / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(e));
      }
  return 0;
}
