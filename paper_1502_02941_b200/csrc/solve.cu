// solve.cu -- the solve of the assembled system and the Newton driver on the device
// (SURVEY.md §8(f) rank 2).
//
// The reference factorises K with Eigen's SparseLU (direct_solve, sparse.cpp:154-217) and
// drives Newton with it (newton_solve, nonlinear.cpp:109-176).  Eigen is not part of the
// reference tree and not in this image; on the B200 the BSR system stays on the device and is
// solved by restarted GMRES(m), right-preconditioned with block Jacobi (the inverses of the
// nl x nl diagonal blocks, one thread per block row).  A solve is accepted under the
// reference's own contract ||A x - b||_2 <= 1e-10 (||A||_F ||x||_2 + ||b||_2), checked on the
// true residual, with the reference's error codes.
//
// Every reduction is deterministic: per-block partial sums in a fixed order, then one block
// sums the partials in a fixed order (no atomics), so a solve is bitwise reproducible.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <set>
#include <vector>

#include "common.hpp"

namespace dgb {
void cuda_check(cudaError_t err, const char* what);
}

namespace {

using dgb::cuda_check;

constexpr int kThreads = 256;
constexpr int kRedBlocks = 296;  // 2 per SM: partial sums of one reduction
constexpr int kMaxRestart = 200;
constexpr long long kGraphMaxN = 1 << 18;  // unknowns: below this a GMRES step is launch-bound

// ------------------------------------------------------------------------------ kernels
// Inverse of block row e's diagonal block (Gauss-Jordan, partial pivoting).  A zero pivot
// records the scalar row (min over rows) in *fail.
template <int NL>
__global__ void diag_inverse_kernel(const int32_t* __restrict__ row_ptr,
                                    const int32_t* __restrict__ col,
                                    const double* __restrict__ val, int E, double* dinv,
                                    unsigned long long* fail) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int b = -1;
  for (int k = row_ptr[e]; k < row_ptr[e + 1]; ++k) {
    if (col[k] == e) b = k;
  }
  double a[NL][NL], inv[NL][NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) {
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      a[i][j] = b >= 0 ? val[static_cast<long long>(b) * NL * NL + i * NL + j] : 0.0;
      inv[i][j] = i == j ? 1.0 : 0.0;
    }
  }
  for (int c = 0; c < NL; ++c) {
    int p = c;
    double best = fabs(a[c][c]);
    for (int r = c + 1; r < NL; ++r) {
      if (fabs(a[r][c]) > best) {
        best = fabs(a[r][c]);
        p = r;
      }
    }
    if (best == 0.0) {
      atomicMin(fail, static_cast<unsigned long long>(e) * NL + c);
      return;
    }
    if (p != c) {
      for (int j = 0; j < NL; ++j) {
        double t = a[c][j]; a[c][j] = a[p][j]; a[p][j] = t;
        t = inv[c][j]; inv[c][j] = inv[p][j]; inv[p][j] = t;
      }
    }
    const double rp = 1.0 / a[c][c];
    for (int j = 0; j < NL; ++j) {
      a[c][j] *= rp;
      inv[c][j] *= rp;
    }
    for (int r = 0; r < NL; ++r) {
      if (r == c) continue;
      const double f = a[r][c];
      if (f == 0.0) continue;
      for (int j = 0; j < NL; ++j) {
        a[r][j] -= f * a[c][j];
        inv[r][j] -= f * inv[c][j];
      }
    }
  }
  double* out = dinv + static_cast<long long>(e) * NL * NL;
#pragma unroll
  for (int i = 0; i < NL; ++i) {
#pragma unroll
    for (int j = 0; j < NL; ++j) out[i * NL + j] = inv[i][j];
  }
}

// y = blockdiag(D) x, one thread per scalar row.
template <int NL>
__global__ void block_apply_kernel(const double* __restrict__ d, const double* __restrict__ x,
                                   double* __restrict__ y, long long n) {
  const long long r = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const long long e = r / NL;
  const int i = static_cast<int>(r - e * NL);
  const double* row = d + e * NL * NL + i * NL;
  const double* xs = x + e * NL;
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < NL; ++j) s = fma(row[j], xs[j], s);
  y[r] = s;
}

// One colour of the symmetric block Gauss-Seidel sweep (right preconditioner y = M^-1 x with
// M = (D + L) D^-1 (D + U), L / U the blocks whose column has an earlier / later colour).
// FORWARD: t_e = D_e^-1 (x_e - sum_{colour(j) < c} K_ej t_j); BACKWARD (colours descending):
// y_e = t_e - D_e^-1 sum_{colour(j) > c} K_ej y_j.  Rows of one colour share no block, so every
// row of the colour is updated in parallel (one thread per block row).
template <int NL, bool FORWARD>
__global__ void sgs_colour_kernel(const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                  const double* __restrict__ val, const double* __restrict__ dinv,
                                  const int32_t* __restrict__ colour, const int32_t* __restrict__ order,
                                  int begin, int end, int c, const double* __restrict__ x,
                                  const double* __restrict__ t, double* __restrict__ out) {
  const int idx = begin + blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= end) return;
  const int e = order[idx];
  double acc[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) acc[i] = 0.0;
  for (int b = row_ptr[e]; b < row_ptr[e + 1]; ++b) {
    const int j = col[b];
    const int cj = colour[j];
    if (FORWARD ? cj >= c : cj <= c) continue;  // the diagonal block (cj == c) included
    const double* blk = val + static_cast<long long>(b) * NL * NL;
    const double* vj = out + static_cast<long long>(j) * NL;  // t (forward) / y (backward)
#pragma unroll
    for (int i = 0; i < NL; ++i) {
      double sacc = 0.0;
#pragma unroll
      for (int k = 0; k < NL; ++k) sacc = fma(blk[i * NL + k], vj[k], sacc);
      acc[i] += sacc;
    }
  }
  const double* d = dinv + static_cast<long long>(e) * NL * NL;
  const long long o = static_cast<long long>(e) * NL;
#pragma unroll
  for (int i = 0; i < NL; ++i) {
    double r = 0.0;
#pragma unroll
    for (int k = 0; k < NL; ++k) {
      const double rhs = FORWARD ? x[o + k] - acc[k] : acc[k];
      r = fma(d[i * NL + k], rhs, r);
    }
    out[o + i] = FORWARD ? r : t[o + i] - r;
  }
}

__device__ __forceinline__ double block_sum(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
    __syncthreads();
  }
  const double r = sh[0];
  __syncthreads();
  return r;
}

// partial[j * gridDim.x + bx] = sum over this block's rows of V_j[i] * w[i]  (grid.y = j)
__global__ void multidot_partial_kernel(const double* __restrict__ V, long long ldv,
                                        const double* __restrict__ w, long long n,
                                        double* __restrict__ partial) {
  __shared__ double sh[kThreads];
  const int j = blockIdx.y;
  const double* v = V + j * ldv;
  double s = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    s = fma(v[i], w[i], s);
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) partial[j * gridDim.x + blockIdx.x] = s;
}

// out[j] = sum_b partial[j * nb + b] in a fixed order (one block per j)
__global__ void sum_partials_kernel(const double* __restrict__ partial, int nb,
                                    double* __restrict__ out) {
  __shared__ double sh[kThreads];
  double s = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) s += partial[blockIdx.x * nb + b];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

// w -= sum_{j<k} h[j] V_j   (h on the device)
__global__ void subtract_combo_kernel(double* __restrict__ w, const double* __restrict__ V,
                                      long long ldv, const double* __restrict__ h, int k,
                                      long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = w[i];
  for (int j = 0; j < k; ++j) s = fma(-h[j], V[j * ldv + i], s);
  w[i] = s;
}

// u = sum_{j<k} y[j] V_j
__global__ void combo_kernel(double* __restrict__ u, const double* __restrict__ V, long long ldv,
                             const double* __restrict__ y, int k, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int j = 0; j < k; ++j) s = fma(y[j], V[j * ldv + i], s);
  u[i] = s;
}

__global__ void scale_kernel(double* __restrict__ dst, const double* __restrict__ src, double a,
                             long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = a * src[i];
}

__global__ void axpy_kernel(double* __restrict__ y, double a, const double* __restrict__ x,
                            long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = fma(a, x[i], y[i]);
}

// r = b - r  (r holds A x on entry)
__global__ void residual_kernel(double* __restrict__ r, const double* __restrict__ b, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) r[i] = b[i] - r[i];
}

__global__ void absmax_partial_kernel(const double* __restrict__ x, long long n,
                                      double* __restrict__ partial) {
  __shared__ double sh[kThreads];
  double m = 0.0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    m = fmax(m, fabs(x[i]));
  }
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = sh[0];
}

// J values = K values, then each block row's diagonal block += HJ block (Newton Jacobian).
template <int NL>
__global__ void add_block_diagonal_kernel(const int32_t* __restrict__ row_ptr,
                                          const int32_t* __restrict__ col,
                                          const double* __restrict__ kval,
                                          const double* __restrict__ hj, double* __restrict__ jval,
                                          int E) {
  const int e = blockIdx.x;
  if (e >= E) return;
  constexpr int N2 = NL * NL;
  for (int b = row_ptr[e]; b < row_ptr[e + 1]; ++b) {
    const bool diag = col[b] == e;
    for (int t = threadIdx.x; t < N2; t += blockDim.x) {
      const long long o = static_cast<long long>(b) * N2 + t;
      jval[o] = diag ? kval[o] + hj[static_cast<long long>(e) * N2 + t] : kval[o];
    }
  }
}

// res = res + h - f   (res holds K u on entry)
__global__ void newton_residual_kernel(double* __restrict__ res, const double* __restrict__ h,
                                       const double* __restrict__ f, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) res[i] += h[i] - f[i];
}

// h[j] += d[j], j < k (the second CGS pass into the Hessenberg column)
__global__ void add_small_kernel(double* __restrict__ h, const double* __restrict__ d, int k) {
  const int j = threadIdx.x;
  if (j < k) h[j] += d[j];
}

// h_{k+1,k} = ||w||, v_{k+1} = w / ||w|| (zero on a happy breakdown); nrm2 = w . w on the device
__global__ void normalize_kernel(double* __restrict__ v, const double* __restrict__ w,
                                 const double* __restrict__ nrm2, double* __restrict__ hsub,
                                 long long n) {
  const double hn = sqrt(*nrm2);
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i == 0) *hsub = hn;
  if (i < n) v[i] = hn > 0.0 ? w[i] * (1.0 / hn) : 0.0;
}

// Givens rotations of Hessenberg column k (column-major, leading dimension ld) and the
// right-hand side g; one thread.  res = |g[k+1]| (the GMRES residual estimate).
__global__ void givens_kernel(double* __restrict__ H, int ld, double* __restrict__ cs,
                              double* __restrict__ sn, double* __restrict__ g, int k,
                              double* __restrict__ res) {
  double* hk = H + static_cast<long long>(k) * ld;
  for (int j = 0; j < k; ++j) {
    const double t = cs[j] * hk[j] + sn[j] * hk[j + 1];
    hk[j + 1] = -sn[j] * hk[j] + cs[j] * hk[j + 1];
    hk[j] = t;
  }
  const double rr = hypot(hk[k], hk[k + 1]);
  cs[k] = rr > 0 ? hk[k] / rr : 1.0;
  sn[k] = rr > 0 ? hk[k + 1] / rr : 0.0;
  hk[k] = rr;
  hk[k + 1] = 0.0;
  g[k + 1] = -sn[k] * g[k];
  g[k] = cs[k] * g[k];
  *res = fabs(g[k + 1]);
}

__global__ void set_scalar_kernel(double* p, double v) { *p = v; }

unsigned grid_for(long long n) { return static_cast<unsigned>((n + kThreads - 1) / kThreads); }

// ------------------------------------------------------------------------------ host side
// Stream-ordered allocations from the device's default memory pool, kept cached across solves
// (the pool's release threshold is raised once), so a repeated solve allocates nothing new.
cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t st = nullptr;
  return st;
}

void keep_pool_cached() {  // per device (each has its own default pool)
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!done.insert(dev).second) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}

struct DevBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t bytes) : s(alloc_stream()) {
    keep_pool_cached();
    cuda_check(cudaMallocAsync(&p, std::max<size_t>(bytes, 16), s), "cudaMallocAsync(solve)");
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { if (p) cudaFreeAsync(p, s); }
  template <typename T> T* as() const { return static_cast<T*>(p); }
};

// Pinned host scratch (one per thread, grown on demand): no cudaMallocHost per solve.  A nested
// user (a Newton reducer alive during its inner solves) gets a private buffer.
struct PinnedPool {
  double* buf = nullptr;
  size_t cap = 0;
  int users = 0;
};
PinnedPool& pinned_pool() {
  static thread_local PinnedPool pp;
  return pp;
}
struct PinnedBuf {
  double* p = nullptr;
  bool own = false;
  explicit PinnedBuf(size_t n) {
    PinnedPool& pp = pinned_pool();
    n = std::max<size_t>(n, 1);
    if (pp.users == 0) {
      if (pp.cap < n) {
        if (pp.buf) cudaFreeHost(pp.buf);
        pp.buf = nullptr;
        pp.cap = 0;
        cuda_check(cudaMallocHost(&pp.buf, n * sizeof(double)), "cudaMallocHost");
        pp.cap = n;
      }
      p = pp.buf;
    } else {
      cuda_check(cudaMallocHost(&p, n * sizeof(double)), "cudaMallocHost");
      own = true;
    }
    ++pp.users;
  }
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() {
    if (own) cudaFreeHost(p);
    --pinned_pool().users;
  }
};

// The operator pieces one solve needs, for block size NL.
struct BsrOps {
  const dgb_bsr* a;
  int nl;
  long long n;
  cudaStream_t s;

  void spmv(const double* x, double* y) const { dgb::launch_bsr_spmv(a, x, y, s); }
  // symmetric block Gauss-Seidel in colour order: forward colours 0..C-1 into t, backward
  // colours C-1..0 into y
  template <int NL>
  void sgs_t(const double* dinv, const int32_t* colour, const int32_t* order,
             const std::vector<int>& cstart, const double* x, double* t, double* y) const {
    const int C = static_cast<int>(cstart.size()) - 1;
    for (int c = 0; c < C; ++c) {
      const int cnt = cstart[c + 1] - cstart[c];
      if (cnt > 0) sgs_colour_kernel<NL, true><<<(cnt + 127) / 128, 128, 0, s>>>(
          a->row_ptr, a->col, a->val, dinv, colour, order, cstart[c], cstart[c + 1], c, x, nullptr, t);
    }
    for (int c = C - 1; c >= 0; --c) {
      const int cnt = cstart[c + 1] - cstart[c];
      if (cnt > 0) sgs_colour_kernel<NL, false><<<(cnt + 127) / 128, 128, 0, s>>>(
          a->row_ptr, a->col, a->val, dinv, colour, order, cstart[c], cstart[c + 1], c, nullptr, t, y);
    }
  }
  void sgs(const double* dinv, const int32_t* colour, const int32_t* order,
           const std::vector<int>& cstart, const double* x, double* t, double* y) const {
    switch (nl) {
      case 3: sgs_t<3>(dinv, colour, order, cstart, x, t, y); break;
      case 6: sgs_t<6>(dinv, colour, order, cstart, x, t, y); break;
      case 10: sgs_t<10>(dinv, colour, order, cstart, x, t, y); break;
      case 15: sgs_t<15>(dinv, colour, order, cstart, x, t, y); break;
      default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported block size", nl);
    }
    cuda_check(cudaGetLastError(), "sgs_colour_kernel");
  }
  void precond(const double* dinv, const double* x, double* y) const {
    switch (nl) {
      case 3: block_apply_kernel<3><<<grid_for(n), kThreads, 0, s>>>(dinv, x, y, n); break;
      case 6: block_apply_kernel<6><<<grid_for(n), kThreads, 0, s>>>(dinv, x, y, n); break;
      case 10: block_apply_kernel<10><<<grid_for(n), kThreads, 0, s>>>(dinv, x, y, n); break;
      case 15: block_apply_kernel<15><<<grid_for(n), kThreads, 0, s>>>(dinv, x, y, n); break;
      default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported block size", nl);
    }
    cuda_check(cudaGetLastError(), "block_apply_kernel");
  }
  void diag_inverse(double* dinv, unsigned long long* fail) const {
    const int E = a->n_block_rows;
    const unsigned g = static_cast<unsigned>((E + 127) / 128);
    switch (nl) {
      case 3: diag_inverse_kernel<3><<<g, 128, 0, s>>>(a->row_ptr, a->col, a->val, E, dinv, fail); break;
      case 6: diag_inverse_kernel<6><<<g, 128, 0, s>>>(a->row_ptr, a->col, a->val, E, dinv, fail); break;
      case 10: diag_inverse_kernel<10><<<g, 128, 0, s>>>(a->row_ptr, a->col, a->val, E, dinv, fail); break;
      case 15: diag_inverse_kernel<15><<<g, 128, 0, s>>>(a->row_ptr, a->col, a->val, E, dinv, fail); break;
      default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported block size", nl);
    }
    cuda_check(cudaGetLastError(), "diag_inverse_kernel");
  }
};

// Deterministic reductions with one host round trip each.
struct Reducer {
  cudaStream_t s;
  DevBuf partial, out;
  PinnedBuf host;
  explicit Reducer(cudaStream_t st)
      : s(st), partial(sizeof(double) * kRedBlocks * (kMaxRestart + 1)),
        out(sizeof(double) * (kMaxRestart + 1)), host(kMaxRestart + 1) {}
  // h[j] = V_j . w for j < k; returns a host pointer (valid until the next call)
  // partial-sum blocks: 2 per SM, fewer for short vectors (a block per 256 rows at most)
  static int blocks_for(long long n) {
    return static_cast<int>(std::min<long long>(kRedBlocks, (n + kThreads - 1) / kThreads));
  }
  const double* dots(const double* V, long long ldv, int k, const double* w, long long n) {
    const int nb = blocks_for(n);
    multidot_partial_kernel<<<dim3(nb, k), kThreads, 0, s>>>(V, ldv, w, n, partial.as<double>());
    sum_partials_kernel<<<k, kThreads, 0, s>>>(partial.as<double>(), nb, out.as<double>());
    cuda_check(cudaGetLastError(), "multidot");
    cuda_check(cudaMemcpyAsync(host.p, out.p, sizeof(double) * k, cudaMemcpyDeviceToHost, s), "D2H(dots)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(dots)");
    return host.p;
  }
  double dot(const double* a, const double* b, long long n) { return dots(a, 0, 1, b, n)[0]; }
  // the same, left on the device: out[j] = V_j . w (no host round trip)
  void dots_device(const double* V, long long ldv, int k, const double* w, long long n, double* out) {
    const int nb = blocks_for(n);
    multidot_partial_kernel<<<dim3(nb, k), kThreads, 0, s>>>(V, ldv, w, n, partial.as<double>());
    sum_partials_kernel<<<k, kThreads, 0, s>>>(partial.as<double>(), nb, out);
    cuda_check(cudaGetLastError(), "multidot");
  }
  double absmax(const double* x, long long n) {
    const int nb = blocks_for(n);
    absmax_partial_kernel<<<nb, kThreads, 0, s>>>(x, n, partial.as<double>());
    cuda_check(cudaGetLastError(), "absmax");
    std::vector<double> hp(nb);
    cuda_check(cudaMemcpyAsync(hp.data(), partial.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, s), "D2H(absmax)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(absmax)");
    double m = 0.0;
    for (double v : hp) m = std::max(m, v);
    return m;
  }
};

void check_bsr(const dgb_bsr* a) {
  if (!a || !a->row_ptr || !a->col || !a->val) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null BSR");
  if (a->n_block_rows < 0 || a->block_dim <= 0) throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "BSR dimensions");
}

dgb_solve_options resolve(const dgb_solve_options* opt) {
  dgb_solve_options o;
  dgb_solve_options_default(&o);
  if (opt) {
    if (opt->tolerance_scale > 0) o.tolerance_scale = opt->tolerance_scale;
    if (opt->max_iterations > 0) o.max_iterations = opt->max_iterations;
    if (opt->restart > 0) o.restart = std::min(opt->restart, kMaxRestart);
    if (opt->preconditioner == DGB_PRECOND_BLOCK_JACOBI || opt->preconditioner == DGB_PRECOND_BLOCK_SGS) {
      o.preconditioner = opt->preconditioner;
    }
  }
  return o;
}

// GMRES(m), right preconditioning (block Jacobi, or one symmetric block Gauss-Seidel sweep in
// multicolour order), classical Gram-Schmidt with one re-orthogonalisation (CGS2).  Returns the contract check on the true residual.
// A library-owned blocking stream that stands in for the legacy default stream (which cannot
// be captured into a graph).  Blocking streams are ordered with the legacy stream both ways,
// so callers on stream 0 see the usual semantics.
cudaStream_t solve_stream_for(cudaStream_t s) {
  if (s != nullptr && s != cudaStreamLegacy) return s;
  static thread_local cudaStream_t own[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return s;
  if (!own[dev]) cuda_check(cudaStreamCreate(&own[dev]), "cudaStreamCreate(solve)");
  return own[dev];
}

void gmres_solve(const dgb_bsr* a, const double* b, double* x, const dgb_solve_options& o,
                 dgb_solve_info* info, cudaStream_t s_in) {
  const cudaStream_t s = solve_stream_for(s_in);
  const int nl = a->block_dim, E = a->n_block_rows;
  const long long n = static_cast<long long>(E) * nl;
  alloc_stream() = s;
  BsrOps A{a, nl, n, s};
  Reducer R(s);
  dgb_solve_info inf{};
  if (n == 0) {
    if (info) *info = inf;
    return;
  }
  const int m = o.restart;
  DevBuf dinv(sizeof(double) * n * nl), fail(sizeof(unsigned long long));
  DevBuf V(sizeof(double) * n * (m + 1)), z(sizeof(double) * n), w(sizeof(double) * n),
      r(sizeof(double) * n), hdev(sizeof(double) * (m + 1));
  DevBuf Hd(sizeof(double) * (m + 1) * m), gd(sizeof(double) * (m + 1)), csd(sizeof(double) * m),
      snd(sizeof(double) * m), nrm(sizeof(double)), resd(sizeof(double));
  PinnedBuf est(1);
  constexpr int kCheck = 4;
  cuda_check(cudaMemsetAsync(fail.p, 0xFF, sizeof(unsigned long long), s), "memset(fail)");
  A.diag_inverse(dinv.as<double>(), fail.as<unsigned long long>());
  unsigned long long bad = 0;
  cuda_check(cudaMemcpyAsync(&bad, fail.p, sizeof bad, cudaMemcpyDeviceToHost, s), "D2H(fail)");
  cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(dinv)");
  if (bad != ~0ull) {
    throw dgb::Error(DGB_STATUS_SINGULAR_MATRIX, "block-Jacobi factorization failed: zero pivot in a diagonal block",
                     static_cast<long long>(bad));
  }
  // multicolour order for the block SGS preconditioner: a greedy colouring of the BSR graph on
  // the host (the block columns of row e are its neighbours; <= 4 colours on a triangle mesh)
  const bool sgs = o.preconditioner == DGB_PRECOND_BLOCK_SGS;
  std::vector<int> cstart;
  DevBuf colour_d(sgs ? sizeof(int32_t) * E : 1), order_d(sgs ? sizeof(int32_t) * E : 1),
      tbuf(sgs ? sizeof(double) * n : 1);
  if (sgs) {
    std::vector<int32_t> rp(E + 1), cl(static_cast<size_t>(a->nnzb)), colour(E, -1), order(E);
    cuda_check(cudaMemcpyAsync(rp.data(), a->row_ptr, sizeof(int32_t) * (E + 1), cudaMemcpyDeviceToHost, s), "D2H(rp)");
    cuda_check(cudaMemcpyAsync(cl.data(), a->col, sizeof(int32_t) * a->nnzb, cudaMemcpyDeviceToHost, s), "D2H(col)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(pattern)");
    int n_col = 0;
    for (int e = 0; e < E; ++e) {
      unsigned used = 0;  // colours of already-coloured neighbours (< 32)
      for (int b = rp[e]; b < rp[e + 1]; ++b) {
        const int j = cl[b];
        if (j != e && j >= 0 && j < E && colour[j] >= 0 && colour[j] < 32) used |= 1u << colour[j];
      }
      int c = 0;
      while (c < 31 && (used >> c & 1u)) ++c;
      colour[e] = c;
      n_col = std::max(n_col, c + 1);
    }
    cstart.assign(n_col + 1, 0);
    for (int e = 0; e < E; ++e) ++cstart[colour[e] + 1];
    for (int c = 0; c < n_col; ++c) cstart[c + 1] += cstart[c];
    std::vector<int> fill(cstart.begin(), cstart.end() - 1);
    for (int e = 0; e < E; ++e) order[fill[colour[e]]++] = e;
    cuda_check(cudaMemcpyAsync(colour_d.p, colour.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, s), "H2D(colour)");
    cuda_check(cudaMemcpyAsync(order_d.p, order.data(), sizeof(int32_t) * E, cudaMemcpyHostToDevice, s), "H2D(order)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(colour)");
  }
  auto precond = [&](const double* xin, double* yout) {
    if (sgs) {
      A.sgs(dinv.as<double>(), colour_d.as<int32_t>(), order_d.as<int32_t>(), cstart, xin,
            tbuf.as<double>(), yout);
    } else {
      A.precond(dinv.as<double>(), xin, yout);
    }
  };
  const long long nvals = a->nnzb * static_cast<long long>(nl) * nl;
  const double a_fro = std::sqrt(R.dot(a->val, a->val, nvals));
  const double b_norm = std::sqrt(R.dot(b, b, n));
  double* Vp = V.as<double>();
  auto residual = [&]() {  // r = b - A x, returns ||r||_2
    A.spmv(x, r.as<double>());
    residual_kernel<<<grid_for(n), kThreads, 0, s>>>(r.as<double>(), b, n);
    cuda_check(cudaGetLastError(), "residual_kernel");
    return std::sqrt(R.dot(r.as<double>(), r.as<double>(), n));
  };
  double beta = residual();
  double x_norm = std::sqrt(R.dot(x, x, n));
  std::vector<double> H(static_cast<size_t>(m + 1) * m), g(m + 1), y(m);
  int its = 0, restarts = 0;
  // Arnoldi step k on the device: Hessenberg column k, rotations and g live in HBM
  auto arnoldi_step = [&](int k) {
    double* vk = Vp + static_cast<long long>(k) * n;
    double* vn = Vp + static_cast<long long>(k + 1) * n;
    double* hk = Hd.as<double>() + static_cast<long long>(k) * (m + 1);
    precond(vk, z.as<double>());
    A.spmv(z.as<double>(), w.as<double>());
    R.dots_device(Vp, n, k + 1, w.as<double>(), n, hk);                          // CGS pass 1
    subtract_combo_kernel<<<grid_for(n), kThreads, 0, s>>>(w.as<double>(), Vp, n, hk, k + 1, n);
    R.dots_device(Vp, n, k + 1, w.as<double>(), n, hdev.as<double>());           // CGS pass 2
    subtract_combo_kernel<<<grid_for(n), kThreads, 0, s>>>(w.as<double>(), Vp, n, hdev.as<double>(), k + 1, n);
    add_small_kernel<<<1, kMaxRestart + 1, 0, s>>>(hk, hdev.as<double>(), k + 1);
    R.dots_device(w.as<double>(), 0, 1, w.as<double>(), n, nrm.as<double>());
    normalize_kernel<<<grid_for(n), kThreads, 0, s>>>(vn, w.as<double>(), nrm.as<double>(), hk + k + 1, n);
    givens_kernel<<<1, 1, 0, s>>>(Hd.as<double>(), m + 1, csd.as<double>(), snd.as<double>(),
                                  gd.as<double>(), k, resd.as<double>());
    cuda_check(cudaGetLastError(), "arnoldi step");
  };
  // CUDA graphs for launch-bound (small) systems, on a capturable (non-legacy) stream
  const bool use_graph = n <= kGraphMaxN && s != nullptr && s != cudaStreamLegacy;
  cudaGraph_t cycle_graph = nullptr;
  cudaGraphExec_t cycle_exec = nullptr;
  struct GraphGuard {
    cudaGraph_t* g;
    cudaGraphExec_t* e;
    ~GraphGuard() {
      if (*e) cudaGraphExecDestroy(*e);
      if (*g) cudaGraphDestroy(*g);
    }
  } graph_guard{&cycle_graph, &cycle_exec};
  while (true) {
    const double bound = 1e-10 * (a_fro * x_norm + b_norm);
    const double target = o.tolerance_scale * bound;
    if (beta <= target || its >= o.max_iterations) break;
    scale_kernel<<<grid_for(n), kThreads, 0, s>>>(Vp, r.as<double>(), 1.0 / beta, n);
    // the host reads the residual estimate every kCheck steps (extra steps past convergence
    // only lower it)
    cuda_check(cudaMemsetAsync(gd.p, 0, sizeof(double) * (m + 1), s), "memset(g)");
    set_scalar_kernel<<<1, 1, 0, s>>>(gd.as<double>(), beta);
    int k = 0;
    bool done = false;
    if (use_graph && its + m <= o.max_iterations) {
      // small system: the m Arnoldi steps (13 launches each) as one CUDA graph, captured on
      // the first cycle and replayed; the residual estimate is read once per cycle (extra
      // steps past convergence only lower it)
      if (!cycle_exec) {
        cuda_check(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
        for (int kk = 0; kk < m; ++kk) arnoldi_step(kk);
        cuda_check(cudaStreamEndCapture(s, &cycle_graph), "cudaStreamEndCapture");
        cuda_check(cudaGraphInstantiate(&cycle_exec, cycle_graph, 0), "cudaGraphInstantiate");
      }
      cuda_check(cudaGraphLaunch(cycle_exec, s), "cudaGraphLaunch");
      k = m;
      its += m;
    } else {
      for (; k < m && its < o.max_iterations && !done; ++k) {
        ++its;
        arnoldi_step(k);
        if ((k + 1) % kCheck == 0 || k + 1 == m || its >= o.max_iterations) {
          cuda_check(cudaMemcpyAsync(est.p, resd.p, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H(res)");
          cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(res)");
          done = *est.p <= target;
        }
      }
    }
    // y = H(0:k, 0:k)^-1 g (host, one copy per cycle), then x += M^-1 (V y)
    cuda_check(cudaMemcpyAsync(H.data(), Hd.p, sizeof(double) * (m + 1) * k, cudaMemcpyDeviceToHost, s), "D2H(H)");
    cuda_check(cudaMemcpyAsync(g.data(), gd.p, sizeof(double) * (m + 1), cudaMemcpyDeviceToHost, s), "D2H(g)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(H)");
    for (int i = k - 1; i >= 0; --i) {
      double t = g[i];
      for (int j = i + 1; j < k; ++j) t -= H[static_cast<size_t>(j) * (m + 1) + i] * y[j];
      const double d = H[static_cast<size_t>(i) * (m + 1) + i];
      y[i] = d != 0.0 ? t / d : 0.0;
    }
    cuda_check(cudaMemcpyAsync(hdev.p, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s), "H2D(y)");
    combo_kernel<<<grid_for(n), kThreads, 0, s>>>(w.as<double>(), Vp, n, hdev.as<double>(), k, n);
    precond(w.as<double>(), z.as<double>());
    axpy_kernel<<<grid_for(n), kThreads, 0, s>>>(x, 1.0, z.as<double>(), n);
    cuda_check(cudaGetLastError(), "gmres update");
    ++restarts;
    beta = residual();
    x_norm = std::sqrt(R.dot(x, x, n));
  }
  // the reference's acceptance test (sparse.cpp:201-214) on the true residual
  beta = residual();
  x_norm = std::sqrt(R.dot(x, x, n));
  inf.defect_norm2 = beta;
  inf.defect_norm_inf = R.absmax(r.as<double>(), n);
  inf.bound = 1e-10 * (a_fro * x_norm + b_norm);
  inf.iterations = its;
  inf.restarts = restarts;
  if (info) *info = inf;
  if (inf.defect_norm2 > inf.bound) {
    throw dgb::Error(DGB_STATUS_SOLVE_ACCURACY, "iterative solve defect exceeds accuracy bound", its);
  }
}

}  // namespace

extern "C" {

void dgb_solve_options_default(dgb_solve_options* opt) {
  if (!opt) return;
  opt->tolerance_scale = 0.1;
  opt->max_iterations = 20000;
  opt->restart = 30;
  opt->preconditioner = DGB_PRECOND_BLOCK_SGS;
  opt->pad_ = 0;
}

void dgb_newton_config_default(dgb_newton_config* cfg) {
  if (!cfg) return;
  cfg->max_iterations = 50;
  cfg->use_legacy_check = 0;
  cfg->residual_tolerance = 1e-10;
  cfg->step_tolerance = 1e-12;
  cfg->legacy_check = 0.0;
}

int dgb_solve(const dgb_bsr* a, const double* b, double* x, const dgb_solve_options* opt,
              dgb_solve_info* info, void* stream) {
  return dgb::guarded([&] {
    check_bsr(a);
    if (!b || !x) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null vector");
    gmres_solve(a, b, x, resolve(opt), info, static_cast<cudaStream_t>(stream));
  });
}

int dgb_newton_solve(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_bsr* k,
                     const double* f, const dgb_reaction* reaction,
                     const dgb_newton_config* config, const dgb_solve_options* inner,
                     double* coef, dgb_newton_report* report, void* stream) {
  return dgb::guarded([&] {
    check_bsr(k);
    if (!plan || !mesh || !f || !reaction || !coef) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    }
    dgb_newton_config cfg;
    dgb_newton_config_default(&cfg);
    if (config) cfg = *config;
    const dgb_solve_options o = resolve(inner);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int nl = k->block_dim, E = k->n_block_rows;
    if (E != mesh->n_elements) throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "system / mesh size mismatch");
    const long long n = static_cast<long long>(E) * nl, nvals = k->nnzb * static_cast<long long>(nl) * nl;
    alloc_stream() = s;
    DevBuf h(sizeof(double) * n), res(sizeof(double) * n), neg(sizeof(double) * n), step(sizeof(double) * n),
        jw(sizeof(double) * n), hjv(sizeof(double) * E * nl * nl), hjr(sizeof(int32_t) * (E + 1)),
        hjc(sizeof(int32_t) * std::max(E, 1)), jval(sizeof(double) * nvals);
    dgb_bsr hj{E, nl, E, hjr.as<int32_t>(), hjc.as<int32_t>(), hjv.as<double>()};
    dgb_bsr J = *k;
    J.val = jval.as<double>();
    BsrOps K{k, nl, n, s}, JO{&J, nl, n, s};
    Reducer R(s);
    // Res = K u + H(u) - F, and HJ(u) (nonlinear.cpp:126-137)
    auto evaluate = [&](double* out) {
      const int rc = dgb_assemble_nonlinear(plan, mesh, coef, n, reaction, h.as<double>(), &hj, s);
      if (rc != DGB_OK) throw dgb::Error(rc, dgb_last_error_message(), dgb_last_error_detail());
      K.spmv(coef, out);
      newton_residual_kernel<<<grid_for(n), kThreads, 0, s>>>(out, h.as<double>(), f, n);
      cuda_check(cudaGetLastError(), "newton_residual_kernel");
    };
    dgb_newton_report rep{};
    rep.residual_history = report ? report->residual_history : nullptr;
    evaluate(res.as<double>());
    for (int it = 0; it < cfg.max_iterations; ++it) {
      switch (nl) {  // J = K + HJ
        case 3: add_block_diagonal_kernel<3><<<E, 64, 0, s>>>(k->row_ptr, k->col, k->val, hjv.as<double>(), J.val, E); break;
        case 6: add_block_diagonal_kernel<6><<<E, 64, 0, s>>>(k->row_ptr, k->col, k->val, hjv.as<double>(), J.val, E); break;
        case 10: add_block_diagonal_kernel<10><<<E, 128, 0, s>>>(k->row_ptr, k->col, k->val, hjv.as<double>(), J.val, E); break;
        case 15: add_block_diagonal_kernel<15><<<E, 256, 0, s>>>(k->row_ptr, k->col, k->val, hjv.as<double>(), J.val, E); break;
        default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported block size", nl);
      }
      cuda_check(cudaGetLastError(), "add_block_diagonal_kernel");
      scale_kernel<<<grid_for(n), kThreads, 0, s>>>(neg.as<double>(), res.as<double>(), -1.0, n);
      cuda_check(cudaMemsetAsync(step.p, 0, sizeof(double) * n, s), "memset(step)");
      dgb_solve_info si{};
      gmres_solve(&J, neg.as<double>(), step.as<double>(), o, &si, s);
      rep.linear_iterations += si.iterations;
      axpy_kernel<<<grid_for(n), kThreads, 0, s>>>(coef, 1.0, step.as<double>(), n);
      cuda_check(cudaGetLastError(), "axpy_kernel");
      rep.iterations = it + 1;
      // post-step residual (what the tolerance is tested against); res keeps the old one
      evaluate(jw.as<double>());
      const double res_norm = std::sqrt(R.dot(jw.as<double>(), jw.as<double>(), n));
      if (rep.residual_history) rep.residual_history[it] = res_norm;
      rep.final_residual = res_norm;
      const double step_norm = std::sqrt(R.dot(step.as<double>(), step.as<double>(), n));
      if (res_norm <= cfg.residual_tolerance || step_norm <= cfg.step_tolerance) {
        rep.converged = 1;
        break;
      }
      if (cfg.use_legacy_check) {  // ||J w + Res||_2 < legacy_check (nonlinear.cpp:160-170)
        JO.spmv(step.as<double>(), neg.as<double>());
        axpy_kernel<<<grid_for(n), kThreads, 0, s>>>(neg.as<double>(), 1.0, res.as<double>(), n);
        cuda_check(cudaGetLastError(), "axpy_kernel");
        if (std::sqrt(R.dot(neg.as<double>(), neg.as<double>(), n)) < cfg.legacy_check) {
          rep.converged = 1;
          break;
        }
      }
      cuda_check(cudaMemcpyAsync(res.p, jw.p, sizeof(double) * n, cudaMemcpyDeviceToDevice, s), "copy(res)");
    }
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(newton)");
    if (report) *report = rep;
  });
}

}  // extern "C"
