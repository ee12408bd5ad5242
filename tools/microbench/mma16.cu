#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
  double a[8], b[4], d[4][4];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-6;
  for (int c = 0; c < 4; ++c) for (int i = 0; i < 4; ++i) d[c][i] = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  long long t1 = clock64();
  double s = 0; for (int c = 0; c < 4; ++c) for (int i = 0; i < 4; ++i) s += d[c][i];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 64);
  const int iters = 2048;
  for (int w : {1, 4}) {
    k<<<1, 32 * w>>>(o, c, iters); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("m16n8k16 f64: warps %d: %.2f cycles per mma per warp (= %.2f per m8n8k4 equivalent)\n", w, double(h) / (iters * 4), double(h) / (iters * 4) / 8);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
