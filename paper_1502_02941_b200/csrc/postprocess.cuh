// postprocess.cuh -- element-local quadrature kernels after the solve (included by
// dg_assembly.cu):
//   * l2_error (postprocess.cpp:14-50): ||u_h - u||_L2 with the sharper rule of
//     ReferenceElement(k, max(2k+3, volume degree + 1)) and max_element_diameter (mesh.cpp:259);
//   * project (postprocess.cpp:56-81): coef_ej = sum_q w_q f(x_q) phi_qj (orthonormal basis);
//   * eval_solution (postprocess.cpp:83-93): u_h at reference points of given elements.
// One thread per element (per point for eval).  The per-element arithmetic follows the
// reference's expressions and order (unfused), so project is bitwise the reference's for
// polynomial data; l2_error sums per-element partials and then reduces them in a fixed tree
// order (deterministic; the reference accumulates serially).
#pragma once

namespace dgb {
namespace post {

constexpr int kThreads = 256;

// Dubiner basis values of degree K at (x, y) (the basis of host_reference.cpp / reference.cpp:20-84).
template <int K>
__device__ __forceinline__ void dubiner_values(double x, double y, double* val) {
  const double u = 2.0 * x + y - 1.0, t = 1.0 - y, z = 2.0 * y - 1.0;
  double f[K + 1];
  f[0] = 1.0;
  if (K >= 1) f[1] = u;
#pragma unroll
  for (int m = 1; m < K; ++m) {
    const double a = 2.0 * m + 1.0;
    f[m + 1] = (a * u * f[m] - m * t * t * f[m - 1]) / (m + 1);
  }
#pragma unroll
  for (int m = 0; m <= K; ++m) {
    const double al = 2.0 * m + 1.0;
    double gm2 = 0.0, gm1 = 1.0;
#pragma unroll
    for (int n = 0; m + n <= K; ++n) {
      double g;
      if (n == 0) {
        g = 1.0;
      } else if (n == 1) {
        g = 0.5 * ((al + 2.0) * z + al);
      } else {
        const double c0 = 2.0 * n * (n + al) * (2.0 * n + al - 2.0);
        const double c1 = 2.0 * n + al - 1.0;
        const double c2 = (2.0 * n + al) * (2.0 * n + al - 2.0);
        const double c3 = 2.0 * (n + al - 1.0) * (n - 1.0) * (2.0 * n + al);
        g = (c1 * ((c2 * z + al * al) * gm1) - c3 * gm2) / c0;
      }
      if (n >= 1) gm2 = gm1;
      gm1 = g;
      const double c = sqrt(2.0 * (2.0 * m + 1.0) * (m + n + 1.0));
      const int d = m + n, j = d * (d + 1) / 2 + n;
      val[j] = c * f[m] * g;
    }
  }
}

struct PostParams {
  const double* nodes;
  const int32_t* elements;
  const double* coef;
  const double* phi;  // [nq][nl] of the plan's rule
  const double* vx;
  const double* vy;
  const double* vw;
  dgb_scalar_field field;  // exact solution (l2_error) or projected field (project)
  double* out;             // l2: per-block partials [gridDim][2]; project: coef [E][nl]
  int32_t n_elements;
  int32_t nq;
};

__device__ __forceinline__ double block_reduce_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  return sh[0];
}

__device__ __forceinline__ double block_reduce_max(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  return sh[0];
}

// Per-block partial (sum of element err2, max longest edge).
template <int NL>
__global__ void __launch_bounds__(kThreads) l2_error_kernel(const __grid_constant__ PostParams P) {
  __shared__ double sh[kThreads];
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  double err2 = 0.0, diam = 0.0;
  if (e < P.n_elements) {
    int v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * e + k);
    double2 p[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) p[k] = __ldg(reinterpret_cast<const double2*>(P.nodes) + v[k]);
    const double B00 = __dsub_rn(p[1].x, p[0].x), B01 = __dsub_rn(p[2].x, p[0].x);
    const double B10 = __dsub_rn(p[1].y, p[0].y), B11 = __dsub_rn(p[2].y, p[0].y);
    const double det = __dsub_rn(__dmul_rn(B00, B11), __dmul_rn(B01, B10));
    double c[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) c[j] = __ldg(P.coef + static_cast<long long>(e) * NL + j);
    for (int q = 0; q < P.nq; ++q) {
      const double xq = __ldg(P.vx + q), yq = __ldg(P.vy + q);
      const double px = __dadd_rn(__dadd_rn(p[0].x, __dmul_rn(B00, xq)), __dmul_rn(B01, yq));
      const double py = __dadd_rn(__dadd_rn(p[0].y, __dmul_rn(B10, xq)), __dmul_rn(B11, yq));
      const double ue = scalar_point(P.field, px, py);
      double uh = 0.0;
#pragma unroll
      for (int j = 0; j < NL; ++j) uh = __dadd_rn(uh, __dmul_rn(c[j], __ldg(P.phi + q * NL + j)));
      const double diff = __dsub_rn(uh, ue);
      err2 = __dadd_rn(err2, __dmul_rn(__dmul_rn(__dmul_rn(det, __ldg(P.vw + q)), diff), diff));
    }
    // longest_edge (mesh.cpp:39-47)
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const double2 a = p[(l + 1) % 3], b = p[(l + 2) % 3];
      diam = fmax(diam, hypot_dd(__dsub_rn(b.x, a.x), __dsub_rn(b.y, a.y)));
    }
  }
  const double s = block_reduce_sum(err2, sh);
  __syncthreads();
  const double m = block_reduce_max(diam, sh);
  if (threadIdx.x == 0) {
    P.out[2 * blockIdx.x] = s;
    P.out[2 * blockIdx.x + 1] = m;
  }
}

// out[0] = sum of partial sums (fixed tree order), out[1] = max.
__global__ void l2_finish_kernel(const double* partial, int nb, double* out) {
  __shared__ double sh[kThreads];
  double s = 0.0, m = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    s += partial[2 * b];
    m = fmax(m, partial[2 * b + 1]);
  }
  const double ts = block_reduce_sum(s, sh);
  __syncthreads();
  const double tm = block_reduce_max(m, sh);
  if (threadIdx.x == 0) {
    out[0] = ts;
    out[1] = tm;
  }
}

// coef[e][j] = sum_q (w_q f(x_q)) phi_qj in q order (postprocess.cpp:64-79)
template <int NL>
__global__ void __launch_bounds__(kThreads) project_kernel(const __grid_constant__ PostParams P) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= P.n_elements) return;
  int v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * e + k);
  double2 p[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) p[k] = __ldg(reinterpret_cast<const double2*>(P.nodes) + v[k]);
  const double B00 = __dsub_rn(p[1].x, p[0].x), B01 = __dsub_rn(p[2].x, p[0].x);
  const double B10 = __dsub_rn(p[1].y, p[0].y), B11 = __dsub_rn(p[2].y, p[0].y);
  double acc[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j) acc[j] = 0.0;
  for (int q = 0; q < P.nq; ++q) {
    const double xq = __ldg(P.vx + q), yq = __ldg(P.vy + q);
    const double px = __dadd_rn(__dadd_rn(p[0].x, __dmul_rn(B00, xq)), __dmul_rn(B01, yq));
    const double py = __dadd_rn(__dadd_rn(p[0].y, __dmul_rn(B10, xq)), __dmul_rn(B11, yq));
    const double wf = __dmul_rn(__ldg(P.vw + q), scalar_point(P.field, px, py));
#pragma unroll
    for (int j = 0; j < NL; ++j) acc[j] = __dadd_rn(acc[j], __dmul_rn(wf, __ldg(P.phi + q * NL + j)));
  }
#pragma unroll
  for (int j = 0; j < NL; ++j) P.out[static_cast<long long>(e) * NL + j] = acc[j];
}

// values[i] = sum_j coef[element_i][j] phi_j(xhat_i, yhat_i) (postprocess.cpp:83-93)
template <int K>
__global__ void __launch_bounds__(kThreads) eval_kernel(const double* __restrict__ coef,
                                                        int n_elements, long long n,
                                                        const int32_t* __restrict__ elements,
                                                        const double* __restrict__ xh,
                                                        const double* __restrict__ yh,
                                                        double* __restrict__ values,
                                                        unsigned long long* bad) {
  constexpr int NL = (K + 1) * (K + 2) / 2;
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int e = elements[i];
  if (e < 0 || e >= n_elements) {
    atomicMin(bad, static_cast<unsigned long long>(i));
    values[i] = nan("");
    return;
  }
  double phi[NL];
  dubiner_values<K>(xh[i], yh[i], phi);
  double v = 0.0;
#pragma unroll
  for (int j = 0; j < NL; ++j) v = __dadd_rn(v, __dmul_rn(coef[static_cast<long long>(e) * NL + j], phi[j]));
  values[i] = v;
}

}  // namespace post
}  // namespace dgb
