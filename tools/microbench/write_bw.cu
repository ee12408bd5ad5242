// Write-only HBM bandwidth on this part: (a) coalesced 16-byte stores, (b) the block-row
// kernel's fragment pattern (8 element blocks x 64 contiguous bytes per store instruction,
// blocks of N2 doubles, 4 blocks per element row), both with and without the L2 evict-first
// hint.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_bw write_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st2(double* g, double a, double b, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n"
               :: "l"(g), "d"(a), "d"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ unsigned long long pol_of(int ef) {
  unsigned long long p;
  if (ef) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  else asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

__global__ void coalesced(double* out, long long n2, int ef) {
  const unsigned long long pol = pol_of(ef);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x)
    st2(out + 2 * i, 1.0, 2.0, pol);
}

// one warp = 32 elements; element e owns 4 blocks of N2 = 36 doubles (288 B) at e*4*36;
// the warp writes block b of its elements: lane (g, t), m-tile m, n-tile nt -> row 8m+g,
// entries 8nt+2t, +1 (entries >= 36 skipped)
__global__ void fragment(double* out, int n_elem, int ef) {
  const unsigned long long pol = pol_of(ef);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int e0 = warp * 32;
  if (e0 >= n_elem) return;
  for (int b = 0; b < 4; ++b)
    for (int nt = 0; nt < 5; ++nt)
      for (int m = 0; m < 4; ++m) {
        const int e = e0 + 8 * m + g, n0 = 8 * nt + 2 * t;
        if (e < n_elem && n0 < 36) st2(out + (long long)e * 144 + b * 36 + n0, 1.0, 2.0, pol);
      }
}

__device__ __forceinline__ void st4(double* g, double a, double b, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.f64 [%0], {%1, %2, %3, %4}, %5;\n"
               :: "l"(g), "d"(a), "d"(b), "d"(a), "d"(b), "l"(pol) : "memory");
}
// as `fragment`, but each lane stores 32 bytes (256-bit STG): lane (g, t) of n-tile pair
// (2p, 2p+1) writes entries 16p + 4t .. +3 of row g -- 8 rows x 128 bytes per instruction
__global__ void fragment32(double* out, int n_elem, int ef) {
  const unsigned long long pol = pol_of(ef);
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int e0 = warp * 32;
  if (e0 >= n_elem) return;
  for (int b = 0; b < 4; ++b)
    for (int np = 0; np < 3; ++np)
      for (int m = 0; m < 4; ++m) {
        const int e = e0 + 8 * m + g, n0 = 16 * np + 4 * t;
        if (e < n_elem && n0 < 36) st4(out + (long long)e * 144 + b * 36 + n0, 1.0, 2.0, pol);
      }
}

int main() {
  const int n_elem = 3 * 131072;            // the config-2 batch: 3 x 131072 element rows
  const long long n = (long long)n_elem * 144;
  double* out;
  cudaMalloc(&out, n * sizeof(double));
  float* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int ef = 0; ef < 2; ++ef) {
    for (int kind = 0; kind < 3; ++kind) {
      float best = 1e9;
      for (int it = 0; it < 10; ++it) {
        cudaMemset(flush, it, 256 << 20);
        cudaEventRecord(a);
        if (kind == 0) coalesced<<<148 * 16, 256>>>(out, n / 2, ef);
        else if (kind == 1) fragment<<<(n_elem + 127) / 128, 128>>>(out, n_elem, ef);
        else fragment32<<<(n_elem + 127) / 128, 128>>>(out, n_elem, ef);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("%-10s evict_first=%d: %.4f ms, %.1f GB/s (%.0f MB)\n", kind == 0 ? "coalesced" : (kind == 1 ? "fragment" : "fragment32"),
             ef, best, n * 8.0 / best / 1e6, n * 8.0 / 1e6);
    }
  }
  return 0;
}
