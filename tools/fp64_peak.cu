// Microbenchmark: FP64 pipe peak on B200 (DFMA vs DMMA), FP32 FFMA, and a
// double2 streaming copy. Used to fix the FP64 roofline denominator that
// MEASURED_PEAKS.json does not carry. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void ffma_kernel(float* out, int iters, float a, float b) {
  float acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3f + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fmaf(acc[c], a, b);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678f) out[0] = s;
}

// m8n8k4 f64 mma: 8*8*4 = 256 FMA per warp-instruction
template <int CHAINS>
__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = k; c[k][1] = -k; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1];
  if (s == 12345.678) out[0] = s;
}

// m16n8k16 f64 mma (sm_90+): 16*8*16 = 2048 FMA per warp-instruction
template <int CHAINS>
__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 0.5 + i;
  double c[CHAINS][4];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) { c[k][0] = k; c[k][1] = -k; c[k][2] = 0; c[k][3] = 1; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, "
                   "{%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[k][0]), "+d"(c[k][1]), "+d"(c[k][2]), "+d"(c[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void copy_kernel(const double2* __restrict__ in, double2* __restrict__ out, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) out[i] = in[i];
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d smem/block optin %zu L2 %d MB clock(kHz) %d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.l2CacheSize >> 20, p.clockRate);
  double* dout; CK(cudaMalloc(&dout, 64));
  float* fout; CK(cudaMalloc(&fout, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 2; ++rep) {
    // DFMA
    {
      const int threads = 512, blocks = sms * 4, iters = 20000; const int CH = 8;
      dfma_kernel<CH><<<blocks, threads>>>(dout, 100, 1.0000001, 1e-9);
      cudaEventRecord(e0);
      dfma_kernel<CH><<<blocks, threads>>>(dout, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * CH * iters * (double)threads * blocks;
      printf("DFMA  : %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    }
    {
      const int threads = 512, blocks = sms * 4, iters = 20000; const int CH = 8;
      ffma_kernel<CH><<<blocks, threads>>>(fout, 100, 1.0000001f, 1e-9f);
      cudaEventRecord(e0);
      ffma_kernel<CH><<<blocks, threads>>>(fout, iters, 1.0000001f, 1e-9f);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * CH * iters * (double)threads * blocks;
      printf("FFMA  : %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    }
    {
      const int threads = 256, blocks = sms * 4, iters = 4000; const int CH = 4;
      dmma884_kernel<CH><<<blocks, threads>>>(dout, 10);
      cudaEventRecord(e0);
      dmma884_kernel<CH><<<blocks, threads>>>(dout, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * CH * iters * (double)(threads / 32) * blocks;
      printf("DMMA m8n8k4  : %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    }
    {
      const int threads = 256, blocks = sms * 4, iters = 1000; const int CH = 4;
      dmma16816_kernel<CH><<<blocks, threads>>>(dout, 10);
      cudaEventRecord(e0);
      dmma16816_kernel<CH><<<blocks, threads>>>(dout, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 2048 * CH * iters * (double)(threads / 32) * blocks;
      printf("DMMA m16n8k16: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    }
    {
      size_t n = (size_t)1 << 27;  // 2 GiB of double2
      double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
      cudaMemset(a, 0, n * 16);
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) copy_kernel<<<sms * 8, 512>>>(a, b, n);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("copy  : %.1f GB/s\n", 5.0 * 2 * n * 16 / ms / 1e6);
      cudaFree(a); cudaFree(b);
    }
  }
  CK(cudaGetLastError());
  return 0;
}
