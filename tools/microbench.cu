// Throughput microbenchmarks on sm_100a: POPC, DFMA, DADD, I2F.F64 and legacy
// mma.sync int8 (IMMA), to size the scan kernel's compute ceilings.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench.cu && /tmp/mb
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

constexpr int ITERS = 4096;

__global__ void k_popc(uint32_t* out, uint32_t seed) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, acc = 0;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      acc += __popc(a0 ^ j) + __popc(a1 ^ j) + __popc(a2 ^ j) + __popc(a3 ^ j);
    }
    a0 += acc;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void k_dfma(double* out, double seed) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + j + threadIdx.x;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 0.999999, 1e-9);
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_i2f(double* out, uint32_t seed) {
  uint32_t u = seed ^ threadIdx.x;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] += (double)(u + j);
    u = u * 1664525u + 1013904223u;
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += s[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

__global__ void k_imma(int* out, int seed) {
  int a0 = seed ^ threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  int c[4][4] = {};
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
          : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main1() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  double thr = (double)blocks * threads;
  float ms = time_it([&] { k_popc<<<blocks, threads>>>((uint32_t*)buf, 7); });
  double ops = thr * ITERS * 32;
  printf("POPC      %8.2f Tops/s  = %6.1f /clk/SM (clk %d MHz)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  ms = time_it([&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0); });
  ops = thr * ITERS * 8;
  printf("DFMA      %8.2f Tops/s  = %6.1f /clk/SM\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_it([&] { k_i2f<<<blocks, threads>>>((double*)buf, 3); });
  ops = thr * ITERS * 8;
  printf("I2F.F64   %8.2f Tops/s  = %6.1f /clk/SM (with DADD)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_it([&] { k_imma<<<blocks, threads>>>((int*)buf, 3); });
  ops = thr / 32 * (ITERS / 4) * 4 * (16.0 * 8 * 32);
  printf("IMMA s8   %8.2f TMAC/s  = %6.1f MAC/clk/SM (mma.sync m16n8k32)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

// fp64 tensor core (DMMA) rates: m8n8k4 and m16n8k16
__global__ void k_dmma884(double* out, double seed) {
  double a = seed + threadIdx.x, b = seed * 0.5;
  double c[4][2] = {};
  for (int i = 0; i < ITERS / 4; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dmma16816(double* out, double seed) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = seed * i;
  double c[2][4] = {};
  for (int i = 0; i < ITERS / 16; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
          "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
          : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
          : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
            "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 2; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main2() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256;
  void* buf;
  cudaMalloc(&buf, (size_t)blocks * threads * 8);
  double warps = (double)blocks * threads / 32;
  float ms = time_it([&] { k_dmma884<<<blocks, threads>>>((double*)buf, 1.0); });
  double macs = warps * (ITERS / 4) * 4 * (8.0 * 8 * 4);
  printf("DMMA 884  %8.2f TMAC/s = %6.1f MAC/clk/SM\n", macs / ms / 1e9, macs / (ms * 1e-3) / sms / (clk * 1e3));
  ms = time_it([&] { k_dmma16816<<<blocks, threads>>>((double*)buf, 1.0); });
  macs = warps * (ITERS / 16) * 2 * (16.0 * 8 * 16);
  printf("DMMA16816 %8.2f TMAC/s = %6.1f MAC/clk/SM\n", macs / ms / 1e9, macs / (ms * 1e-3) / sms / (clk * 1e3));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
int main() { main1(); return main2(); }
