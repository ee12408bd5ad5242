// FP64 latency / per-SMSP issue spacing on this GPU (clock64 around dependent and
// independent chains, one CTA on one SM):
//   * DFMA dependent-chain latency, DMMA (mma.sync m8n8k4 f64) dependent-chain latency;
//   * DMMA throughput of one SMSP (1..4 warps per SMSP, independent accumulators).
// Used to size the ILP of the block-row kernel's tensor-core passes (profiles/NOTES.md).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dfma_chain(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c = 0.9999999;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a = fma(a, b, c);
  }
  const long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

template <int CHAINS>
__global__ void dmma_chains(double* out, long long* cyc, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  double d[CHAINS][2];
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) d[k][0] = d[k][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < CHAINS; ++k) dmma(d[k][0], d[k][1], a, b);
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < CHAINS; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[threadIdx.x >> 5] = t1 - t0;
}

// Half the warps run independent DFMA chains, half DMMA chains: do the two share a pipe?
__global__ void mixed(double* out, long long* cyc, int iters, int mode) {
  const int w = threadIdx.x >> 5;
  const bool dmma_warp = mode == 2 ? ((w >> 2) & 1) : mode == 1;  // mode 2: one of each per SMSP
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  double d[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  __syncthreads();
  const long long t0 = clock64();
  if (dmma_warp) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) dmma(d[k][0], d[k][1], a[k], b);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
    }
  }
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1] + a[k] + a[k + 4];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if ((threadIdx.x & 31) == 0) cyc[w] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMalloc(&cyc, 64 * sizeof(long long));
  long long h[64];
  const int iters = 4096;
  dfma_chain<<<1, 32>>>(out, cyc, iters);
  cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", double(h[0]) / (iters * 16.0));
#define RUN(CH, WARPS)                                                                        \
  dmma_chains<CH><<<1, 32 * (WARPS)>>>(out, cyc, iters);                                     \
  cudaMemcpy(h, cyc, 8 * (WARPS), cudaMemcpyDeviceToHost);                                   \
  {                                                                                         \
    long long mx = 0;                                                                         \
    for (int w = 0; w < (WARPS); ++w) mx = h[w] > mx ? h[w] : mx;                             \
    const double per = double(mx) / (iters * double(CH));                                     \
    printf("DMMA chains=%d warps/CTA=%d: %.2f cycles per DMMA per warp, SM: %.2f DMMA/cycle\n", \
           CH, WARPS, per, (WARPS) / per);                                                    \
  }
  RUN(1, 1)
  RUN(2, 1)
  RUN(4, 1)
  RUN(8, 1)
  RUN(4, 4)
  RUN(8, 4)
  RUN(4, 8)
  RUN(4, 16)
  RUN(8, 16)
  for (int mode = 0; mode < 3; ++mode) {
    mixed<<<1, mode == 2 ? 256 : 128>>>(out, cyc, iters, mode);
    cudaMemcpy(h, cyc, 8 * 8, cudaMemcpyDeviceToHost);
    printf("mixed mode %d (0 all DFMA, 1 all DMMA, 2 alternate):", mode);
    for (int w = 0; w < 8; ++w) printf(" %.2f", double(h[w]) / iters);
    printf("  cycles per iteration per warp (DFMA iter = 8 DFMA, DMMA iter = 4 DMMA)\n");
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
