// Config 5's value stream alone (524288 elements x 4 blocks of 225 doubles, 3.77 GB): (a) the
// block-row kernel's fragment stores -- lane (g, t) of m-tile m writes entries 8 nt + 2t, +1 of
// element 8m + g's block, as two 8-byte stores because the odd block size leaves every other
// block 8-byte aligned only; (b) the same fragments re-paired across the quad so every pair is
// 16-byte aligned (one 16-byte store, 8-byte stores only at block ends); (c) coalesced 16-byte
// stores of the same bytes.  Tools only.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/write_p4 write_p4.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st1(double* g, double a, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;\n" :: "l"(g), "d"(a), "l"(pol) : "memory");
}
__device__ __forceinline__ void st2(double* g, double a, double b, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" :: "l"(g), "d"(a), "d"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ unsigned long long pol_ef() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
constexpr int N2 = 225, NT = 29;

__global__ void frag8(double* out, int n_elem) {
  const unsigned long long pol = pol_ef();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int e0 = warp * 32;
  if (e0 >= n_elem) return;
  for (int b = 0; b < 4; ++b)
    for (int nt = 0; nt < NT; ++nt)
      for (int m = 0; m < 4; ++m) {
        const int n0 = 8 * nt + 2 * t;
        double* blk = out + ((long long)(e0 + 8 * m + g) * 4 + b) * N2;
        if (n0 < N2) st1(blk + n0, 1.0, pol);
        if (n0 + 1 < N2) st1(blk + n0 + 1, 2.0, pol);
      }
}

// re-paired: for a block whose start is 16-byte aligned, pairs (2k, 2k+1) as in the fragment;
// for an 8-byte-aligned block, lane t stores (n0 + 1, n0 + 2) with n0 + 2 from the next lane
// (the quad's last lane takes the next n-tile's first entry), entry 0 alone
__global__ void frag16(double* out, int n_elem) {
  const unsigned long long pol = pol_ef();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int e0 = warp * 32;
  if (e0 >= n_elem) return;
  for (int b = 0; b < 4; ++b)
    for (int m = 0; m < 4; ++m) {
      double* blk = out + ((long long)(e0 + 8 * m + g) * 4 + b) * N2;
      const bool odd = (reinterpret_cast<unsigned long long>(blk) & 15) != 0;
      double carry = 0.0;
      for (int nt = 0; nt < NT; ++nt) {
        const int n0 = 8 * nt + 2 * t;
        const double d0 = 1.0, d1 = 2.0;
        if (!odd) {
          if (n0 + 1 < N2) st2(blk + n0, d0, d1, pol);
          else if (n0 < N2) st1(blk + n0, d0, pol);
        } else {
          const double next0 = __shfl_down_sync(0xffffffffu, d0, 1, 4);
          const double first = __shfl_sync(0xffffffffu, d0, (lane & ~3), 32);
          (void)first;
          if (nt == 0 && t == 0) st1(blk, d0, pol);
          if (t < 3) {
            if (n0 + 2 < N2) st2(blk + n0 + 1, d1, next0, pol);
            else if (n0 + 1 < N2) st1(blk + n0 + 1, d1, pol);
          } else {
            carry = d1;  // entry 8 nt + 7 pairs with the next n-tile's entry 8 (nt + 1)
            if (nt + 1 < NT && n0 + 2 < N2) st2(blk + n0 + 1, carry, 1.0, pol);
            else if (n0 + 1 < N2) st1(blk + n0 + 1, carry, pol);
          }
        }
      }
    }
}

__global__ void coalesced(double* out, long long n2) {
  const unsigned long long pol = pol_ef();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2; i += (long long)gridDim.x * blockDim.x)
    st2(out + 2 * i, 1.0, 2.0, pol);
}

int main() {
  const int n_elem = 524288;
  const long long n = (long long)n_elem * 4 * N2;
  double* out;
  cudaMalloc(&out, n * 8);
  float* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int kind = 0; kind < 3; ++kind) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaMemset(flush, it, 256 << 20);
      cudaEventRecord(a);
      if (kind == 0) frag8<<<n_elem / 64, 64>>>(out, n_elem);
      else if (kind == 1) frag16<<<n_elem / 64, 64>>>(out, n_elem);
      else coalesced<<<148 * 8, 512>>>(out, n / 2);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("%-26s %.4f ms  %.1f GB/s  (%.0f MB)\n",
           kind == 0 ? "fragments, 8-byte stores" : (kind == 1 ? "fragments, 16-byte pairs" : "coalesced 16-byte"), best,
           n * 8.0 / best / 1e6, n * 8.0 / 1e6);
  }
  return 0;
}
