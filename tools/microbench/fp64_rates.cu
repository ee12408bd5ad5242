// FP64 throughput on this GPU: DFMA (CUDA cores) vs DMMA (mma.sync m8n8k4 f64 tensor path),
// and the two mixed.  Used to decide where the block contractions belong (profiles/NOTES.md).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double));
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    for (int warps : {4, 8, 16}) {
      const int blocks = 148 * 4, threads = warps * 32 / 4 * 4 / 4 * 4 / 4;  // warps per block = warps/4
      const int tpb = warps * 32 / 4 * 1;
      cudaEventRecord(t0);
      dfma_kernel<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(t1);
      cudaEventSynchronize(t1);
      float ms;
      cudaEventElapsedTime(&ms, t0, t1);
      const double flops = 2.0 * 8 * iters * double(blocks) * tpb;
      printf("DFMA  %2d warps/SM: %.1f TFLOP/s\n", warps, flops / ms / 1e9);
      cudaEventRecord(t0);
      dmma_kernel<<<blocks, tpb>>>(out, iters);
      cudaEventRecord(t1);
      cudaEventSynchronize(t1);
      cudaEventElapsedTime(&ms, t0, t1);
      const double mflops = 2.0 * 256 * 4 * iters * double(blocks) * tpb / 32;
      printf("DMMA  %2d warps/SM: %.1f TFLOP/s\n", warps, mflops / ms / 1e9);
      (void)threads;
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
