// Event-timed cost of one launch of an empty kernel, as bench.py times the block-row kernel
// (event, launch, event on one stream): parameter-block size, dynamic shared memory and grid
// size.  Used to attribute the fixed per-assembly cost (profiles/NOTES.md).
#include <cstdio>
#include <cuda_runtime.h>

template <int BYTES>
struct Blob {
  double x[BYTES / 8];
};

template <int BYTES>
__global__ void empty_kernel(const __grid_constant__ Blob<BYTES> b, double* out) {
  extern __shared__ double sm[];
  if (threadIdx.x == 0 && b.x[0] == 12345.0) out[blockIdx.x] = sm[0];
}

template <int BYTES>
float time_one(int grid, int threads, size_t smem, double* out, cudaStream_t s) {
  static Blob<BYTES> b;
  b.x[0] = 1.0;
  cudaFuncSetAttribute(empty_kernel<BYTES>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9, sum = 0;
  const int reps = 50;
  for (int r = 0; r < reps + 5; ++r) {
    cudaEventRecord(e0, s);
    empty_kernel<BYTES><<<grid, threads, smem, s>>>(b, out);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r >= 5) {
      sum += ms;
      best = ms < best ? ms : best;
    }
  }
  printf("param %6d B grid %6d x %4d smem %6zu: mean %.2f us  best %.2f us\n", BYTES, grid, threads,
         smem, 1000 * sum / reps, 1000 * best);
  return sum / reps;
}

int main() {
  double* out;
  cudaMalloc(&out, 1 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  time_one<64>(1024, 128, 0, out, s);
  time_one<64>(1024, 128, 52 * 1024, out, s);
  time_one<8192>(1024, 128, 0, out, s);
  time_one<8192>(1024, 128, 52 * 1024, out, s);
  time_one<30000>(1024, 128, 52 * 1024, out, s);
  time_one<64>(148, 128, 0, out, s);
  time_one<64>(296, 512, 52 * 1024, out, s);
  time_one<8192>(148, 512, 0, out, s);
  time_one<64>(16384, 128, 0, out, s);
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
