// The persistent P1 kernel's output stream alone (config 4 sizes, no arithmetic): 148 CTAs x
// 12 warps, warp gw handles chunks gw + j * 1776 of 32 elements; per chunk it writes the chunk's
// value range (32 rows x 4 blocks x 9 doubles, 16-byte stores from lanes in turn), the RHS slice
// (3 x 8-byte stores per lane), block columns (4 x 4-byte per lane) and row pointers.  Compared
// with plain coalesced 16-byte stores of the same bytes.  Tools only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_p1 write_p1.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st2(double* g, double a, double b) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};\n" :: "l"(g), "d"(a), "d"(b) : "memory");
}

__global__ void __launch_bounds__(384, 1) p1_pattern(double* val, double* rhs, int* col, int* rp, int n_elem,
                                                     int rhs_mode) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gw = blockIdx.x * 12 + warp, n_gw = gridDim.x * 12;
  const int n_chunks = (n_elem + 31) / 32;
  for (int c = gw; c < n_chunks; c += n_gw) {
    const int e = c * 32 + lane;
    // row pointers and block columns (4 blocks per row)
    rp[e + 1] = 4 * (e + 1);
#pragma unroll
    for (int b = 0; b < 4; ++b) col[4 * e + b] = e + b;
    // RHS
    if (rhs_mode == 0) {
#pragma unroll
      for (int i = 0; i < 3; ++i) rhs[3LL * e + i] = 1.0 + i;
    } else {
      double* r = rhs + 3LL * c * 32;
      for (int k = lane; k < 48; k += 32) st2(r + 2 * k, 1.0, 2.0);
    }
    // value range of the chunk: 32 x 36 doubles, 16-byte stores
    double* dst = val + (long long)c * 32 * 36;
#pragma unroll 4
    for (int k = lane; k < 576; k += 32) st2(dst + 2 * k, 1.0, 2.0);
  }
}

__global__ void coalesced(double* out, long long n2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    st2(out + 2 * i, 1.0, 2.0);
}

int main() {
  const int n_elem = 8388608;
  double *val, *rhs;
  int *col, *rp;
  cudaMalloc(&val, (size_t)n_elem * 36 * 8);
  cudaMalloc(&rhs, (size_t)n_elem * 3 * 8);
  cudaMalloc(&col, (size_t)n_elem * 4 * 4);
  cudaMalloc(&rp, (size_t)(n_elem + 1) * 4);
  float* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = (double)n_elem * (36 * 8 + 3 * 8 + 4 * 4 + 4);
  for (int kind = 0; kind < 3; ++kind) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaMemset(flush, it, 256 << 20);
      cudaEventRecord(a);
      if (kind == 0) coalesced<<<148 * 8, 512>>>(val, (long long)(bytes / 16));
      else p1_pattern<<<148, 384>>>(val, rhs, col, rp, n_elem, kind - 1);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-22s %.4f ms  %.1f GB/s  (%.0f MB written)\n",
           kind == 0 ? "coalesced 16B" : (kind == 1 ? "P1 pattern, rhs 8B" : "P1 pattern, rhs 16B"), best,
           bytes / best / 1e6, bytes / 1e6);
  }
  return 0;
}
