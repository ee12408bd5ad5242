// spmv_lab.cu -- experiment harness for the BSR SpMV (tools only; not product code).
// v2: the first two-stage kernel; v3: the three-stage kernel with staged x gathers.
#include <cuda_runtime.h>
#include <cstdint>
#include <algorithm>
#include "../paper_1502_02941_b200/csrc/common.hpp"
namespace v2 {

__device__ __forceinline__ void cp16(void* sm, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp8(void* sm, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cp4(void* sm, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void wait_prev() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

constexpr int kMaxPerRow = 4;  // staged capacity in blocks per row (DG: 1 + interior edges <= 4)

template <int NL, int T>
struct Cfg {
  static constexpr int R = T / NL;                   // block rows per tile
  static constexpr int N2 = NL * NL;
  static constexpr int kMaxBlocks = kMaxPerRow * R;  // staged blocks per tile
  static constexpr int kVal = kMaxBlocks * N2 + 2;   // doubles per stage (+1 alignment slack, even)
  static constexpr int kCol = (kMaxBlocks + 3) & ~3;  // ints per stage
  static constexpr size_t kStageBytes = sizeof(double) * kVal + sizeof(int) * kCol;
  static constexpr size_t kBytes = 2 * kStageBytes;
};

// One scalar row: sum over the row's blocks (ascending block column, as the reference's CSR
// row runs over ascending columns) of K(e, i, :) . x(col).  `v` points at the row's first
// block's row i, stride N2 between blocks; `c` at the row's first block column.
template <int NL>
__device__ __forceinline__ double row_dot(const double* v, const int* c, int nb,
                                          const double* __restrict__ x) {
  double acc = 0.0;
#pragma unroll
  for (int b = 0; b < kMaxPerRow; ++b) {
    if (b < nb) {
      const double* xb = x + static_cast<long long>(c[b]) * NL;
#pragma unroll
      for (int j = 0; j < NL; ++j) acc = fma(v[b * NL * NL + j], __ldg(xb + j), acc);
    }
  }
  for (int b = kMaxPerRow; b < nb; ++b) {  // only rows with more than kMaxPerRow blocks
    const double* xb = x + static_cast<long long>(c[b]) * NL;
#pragma unroll
    for (int j = 0; j < NL; ++j) acc = fma(v[b * NL * NL + j], __ldg(xb + j), acc);
  }
  return acc;
}

template <int NL, int T>
__global__ void __launch_bounds__(T) bsr_spmv_kernel(int32_t n_rows, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col,
                                                     const double* __restrict__ val,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ y, int aligned) {
  using C = Cfg<NL, T>;
  constexpr int R = C::R, N2 = C::N2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n_tiles = (n_rows + R - 1) / R;
  const int tid = threadIdx.x;
  auto sval = [&](int s) { return reinterpret_cast<double*>(smem_raw + s * C::kStageBytes); };
  auto scol = [&](int s) {
    return reinterpret_cast<int*>(smem_raw + s * C::kStageBytes + sizeof(double) * C::kVal);
  };

  // Issue tile t's copies into stage s (every thread commits one group, staged or not).
  // Returns whether the tile is staged (uniform over the CTA).
  auto issue = [&](int t, int s) -> bool {
    bool staged = false;
    if (t < n_tiles && aligned) {
      const int r0 = t * R, r1 = min(r0 + R, n_rows);
      const long long b0 = __ldg(row_ptr + r0), b1 = __ldg(row_ptr + r1);
      if (b1 - b0 <= C::kMaxBlocks) {
        staged = true;
        // values [b0 N2, b1 N2) from the 16-byte boundary at or below the start; an odd last
        // double goes alone (never read past the array)
        const long long v0 = b0 * N2, v1 = b1 * N2, va = v0 & ~1ll;
        const int npair = static_cast<int>((v1 - va + 1) >> 1);
        double* sv = sval(s);
        for (int k = tid; k < npair; k += T) {
          const long long g = va + 2 * k;
          if (g + 1 < v1) cp16(sv + 2 * k, val + g);
          else cp8(sv + 2 * k, val + g);
        }
        int* sc = scol(s);
        for (int k = tid; k < b1 - b0; k += T) cp4(sc + k, col + b0 + k);
      }
    }
    commit();
    return staged;
  };

  int t = blockIdx.x, s = 0;
  bool staged = issue(t, 0);
  for (; t < n_tiles; t += gridDim.x, s ^= 1) {
    const bool staged_next = issue(t + gridDim.x, s ^ 1);
    wait_prev();  // this thread's copies of tile t have landed
    __syncthreads();  // ... and everyone else's
    const int r0 = t * R, r1 = min(r0 + R, n_rows);
    const int el = tid / NL, i = tid - el * NL;
    if (el < R && r0 + el < r1) {
      const int e = r0 + el;
      const int bs = __ldg(row_ptr + e), be = __ldg(row_ptr + e + 1);
      double acc;
      if (staged) {
        const int b0 = __ldg(row_ptr + r0);
        const int off = static_cast<int>((static_cast<long long>(b0) * N2) & 1);
        acc = row_dot<NL>(sval(s) + off + static_cast<long long>(bs - b0) * N2 + i * NL,
                          scol(s) + (bs - b0), be - bs, x);
      } else {
        acc = row_dot<NL>(val + static_cast<long long>(bs) * N2 + i * NL, col + bs, be - bs, x);
      }
      y[static_cast<long long>(e) * NL + i] = acc;
    }
    __syncthreads();  // stage s is refilled by the next-but-one issue
    staged = staged_next;
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

}
namespace v3 {

__device__ __forceinline__ unsigned long long evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
// streamed once (values, block columns, row pointer): 16 / 4-byte copies, L2 evict-first so the
// stream does not push the gathered x out of L2
__device__ __forceinline__ void cp16s(void* sm, const void* g, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp8s(void* sm, const void* g, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp4s(void* sm, const void* g, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(s), "l"(g), "l"(pol)
               : "memory");
}
// gathered (x, read by up to 4 block rows in any order): default L2 priority
__device__ __forceinline__ void cp8(void* sm, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

constexpr int kMaxPerRow = 4;  // staged capacity in blocks per row (DG: 1 + interior edges <= 4)
constexpr int kStages = 3;

template <int NL, int T>
struct Cfg {
  static constexpr int R = T / NL;                    // block rows per tile
  static constexpr int N2 = NL * NL;
  static constexpr int kMaxBlocks = kMaxPerRow * R;   // staged blocks per tile
  static constexpr int kVal = kMaxBlocks * N2 + 2;    // doubles (+1 alignment slack, even)
  static constexpr int kX = kMaxBlocks * NL;          // gathered x doubles
  static constexpr int kCol = (kMaxBlocks + 3) & ~3;  // block columns
  static constexpr int kRp = (R + 1 + 3) & ~3;        // row pointers of the tile
  static constexpr size_t kStageBytes = sizeof(double) * (kVal + kX) + sizeof(int) * (kCol + kRp);
  static constexpr size_t kBytes = kStages * kStageBytes;
};

// One scalar row from global memory (tiles beyond the staged capacity, unaligned values).
template <int NL>
__device__ __forceinline__ double row_dot_global(const double* v, const int* c, int nb,
                                                 const double* __restrict__ x) {
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) {
    const double* xb = x + static_cast<long long>(__ldg(c + b)) * NL;
#pragma unroll
    for (int j = 0; j < NL; ++j) acc = fma(__ldg(v + b * NL * NL + j), __ldg(xb + j), acc);
  }
  return acc;
}

// Three-stage pipeline over the CTA's tiles (k = 0, 1, ...; stage k % 3):
//   V(k): row pointers, values and block columns of tile k      (needs row_ptr only)
//   X(k): the x blocks named by tile k's block columns           (needs V(k) landed)
// Iteration k commits V(k+2), waits for V(k+1) and X(k), commits X(k+1), then computes tile k
// from shared memory alone.  Every thread commits every group (possibly empty), so the
// per-thread group counts line up and `wait_group 1` means "all but the newest".
template <int NL, int T>
__global__ void __launch_bounds__(T) bsr_spmv_kernel(int32_t n_rows, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col,
                                                     const double* __restrict__ val,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ y, int aligned) {
  using C = Cfg<NL, T>;
  constexpr int R = C::R, N2 = C::N2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n_tiles = (n_rows + R - 1) / R;
  const int tid = threadIdx.x;
  const unsigned long long pol = evict_first();
  auto base = [&](int s) { return smem_raw + s * C::kStageBytes; };
  auto sval = [&](int s) { return reinterpret_cast<double*>(base(s)); };
  auto sx = [&](int s) { return reinterpret_cast<double*>(base(s)) + C::kVal; };
  auto scol = [&](int s) { return reinterpret_cast<int*>(sx(s) + C::kX); };
  auto srp = [&](int s) { return scol(s) + C::kCol; };
  auto tile_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };

  // V(k) into stage s; returns whether tile k is staged (uniform over the CTA)
  auto issue_v = [&](int k, int s) -> bool {
    const int t = tile_of(k);
    bool staged = false;
    if (t < n_tiles && aligned) {
      const int r0 = t * R, r1 = min(r0 + R, n_rows);
      const long long b0 = __ldg(row_ptr + r0), b1 = __ldg(row_ptr + r1);
      if (b1 - b0 <= C::kMaxBlocks) {
        staged = true;
        const long long v0 = b0 * N2, v1 = b1 * N2, va = v0 & ~1ll;
        const int npair = static_cast<int>((v1 - va + 1) >> 1);
        double* sv = sval(s);
        for (int k2 = tid; k2 < npair; k2 += T) {
          const long long g = va + 2 * k2;
          if (g + 1 < v1) cp16s(sv + 2 * k2, val + g, pol);
          else cp8s(sv + 2 * k2, val + g, pol);
        }
        int* sc = scol(s);
        for (int k2 = tid; k2 < b1 - b0; k2 += T) cp4s(sc + k2, col + b0 + k2, pol);
        int* sr = srp(s);
        for (int k2 = tid; k2 <= r1 - r0; k2 += T) cp4s(sr + k2, row_ptr + r0 + k2, pol);
      }
    }
    commit();
    return staged;
  };
  // X(k) into stage s (V(k) has landed and is visible)
  auto issue_x = [&](int k, int s, bool staged) {
    const int t = tile_of(k);
    if (staged && t < n_tiles) {
      const int r0 = t * R, r1 = min(r0 + R, n_rows);
      const int* sr = srp(s);
      const int nb = sr[r1 - r0] - sr[0];
      const int* sc = scol(s);
      double* xs = sx(s);
      for (int k2 = tid; k2 < nb * NL; k2 += T) {
        const int b = k2 / NL, j = k2 - b * NL;
        cp8(xs + k2, x + static_cast<long long>(sc[b]) * NL + j);
      }
    }
    commit();
  };

  if (static_cast<int>(blockIdx.x) >= n_tiles) return;
  bool st0 = issue_v(0, 0);
  bool st1 = issue_v(1, 1);
  wait_1();
  __syncthreads();
  issue_x(0, 0, st0);
  for (int k = 0; tile_of(k) < n_tiles; ++k) {
    const int s = k % kStages;
    const bool st2 = issue_v(k + 2, (k + 2) % kStages);
    wait_1();           // V(k+1) and X(k) have landed (V(k+2) may be in flight)
    __syncthreads();
    issue_x(k + 1, (k + 1) % kStages, st1);
    const int t = tile_of(k);
    const int r0 = t * R, r1 = min(r0 + R, n_rows);
    const int el = tid / NL, i = tid - el * NL;
    if (el < R && r0 + el < r1) {
      const int e = r0 + el;
      double acc = 0.0;
      if (st0) {
        const int* sr = srp(s);
        const int b0 = sr[0], bs = sr[el] - b0, be = sr[el + 1] - b0;
        const int off = static_cast<int>((static_cast<long long>(b0) * N2) & 1);
        const double* v = sval(s) + off + i * NL;
        const double* xs = sx(s);
#pragma unroll
        for (int b = 0; b < kMaxPerRow; ++b) {
          if (bs + b < be) {
#pragma unroll
            for (int j = 0; j < NL; ++j) acc = fma(v[(bs + b) * N2 + j], xs[(bs + b) * NL + j], acc);
          }
        }
        for (int b = bs + kMaxPerRow; b < be; ++b) {  // rows above kMaxPerRow blocks
#pragma unroll
          for (int j = 0; j < NL; ++j) acc = fma(v[b * N2 + j], xs[b * NL + j], acc);
        }
      } else {
        const int bs = __ldg(row_ptr + e), be = __ldg(row_ptr + e + 1);
        acc = row_dot_global<NL>(val + static_cast<long long>(bs) * N2 + i * NL, col + bs, be - bs, x);
      }
      y[static_cast<long long>(e) * NL + i] = acc;
    }
    __syncthreads();    // stage s is refilled by V(k+3)
    st0 = st1;
    st1 = st2;
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

}

namespace v4 {

__device__ __forceinline__ unsigned long long evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
// streamed once (values, block columns, row pointer): 16 / 4-byte copies, L2 evict-first so the
// stream does not push the gathered x out of L2
__device__ __forceinline__ void cp16s(void* sm, const void* g, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp8s(void* sm, const void* g, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(s), "l"(g), "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp4s(void* sm, const void* g, unsigned long long pol) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;\n" ::"r"(s), "l"(g), "l"(pol)
               : "memory");
}
// gathered (x, read by up to 4 block rows in any order): default L2 priority
__device__ __forceinline__ void cp8(void* sm, const void* g) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(sm));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

constexpr int kMaxPerRow = 4;  // staged capacity in blocks per row (DG: 1 + interior edges <= 4)

template <int NL, int T, int S = 4>
struct Cfg {
  static constexpr int kStages = S;
  static constexpr int R = T / NL;                    // block rows per tile
  static constexpr int N2 = NL * NL;
  static constexpr int kMaxBlocks = kMaxPerRow * R;   // staged blocks per tile
  static constexpr int kVal = kMaxBlocks * N2 + 2;    // doubles (+1 alignment slack, even)
  static constexpr int kX = kMaxBlocks * NL;          // gathered x doubles
  static constexpr int kCol = (kMaxBlocks + 3) & ~3;  // block columns
  static constexpr int kRp = (R + 1 + 3) & ~3;        // row pointers of the tile
  static constexpr size_t kStageBytes = sizeof(double) * (kVal + kX) + sizeof(int) * (kCol + kRp);
  static constexpr size_t kBytes = S * kStageBytes;
};

// One scalar row from global memory (tiles beyond the staged capacity, unaligned values).
template <int NL>
__device__ __forceinline__ double row_dot_global(const double* v, const int* c, int nb,
                                                 const double* __restrict__ x) {
  double acc = 0.0;
  for (int b = 0; b < nb; ++b) {
    const double* xb = x + static_cast<long long>(__ldg(c + b)) * NL;
#pragma unroll
    for (int j = 0; j < NL; ++j) acc = fma(__ldg(v + b * NL * NL + j), __ldg(xb + j), acc);
  }
  return acc;
}

// S-stage pipeline over the CTA's tiles (k = 0, 1, ...; stage k % S):
//   V(k): row pointers, values and block columns of tile k      (needs row_ptr only)
//   X(k): the x blocks named by tile k's block columns           (needs V(k) landed)
// Iteration k commits V(k+S-1), waits for V(k+S-2) and X(k), commits X(k+S-2), then computes
// tile k from shared memory alone: the random x gathers have S-2 iterations to land, the value
// stream S-1.  Every thread commits every group (possibly empty), so the per-thread group
// counts line up and `wait_group n` means "all but the n newest".
template <int NL, int T, int S = 4>
__global__ void __launch_bounds__(T) bsr_spmv_kernel(int32_t n_rows, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col,
                                                     const double* __restrict__ val,
                                                     const double* __restrict__ x,
                                                     double* __restrict__ y, int aligned, int accumulate = 0) {
  using C = Cfg<NL, T, S>;
  static_assert(S >= 3, "at least three stages");
  constexpr int R = C::R, N2 = C::N2;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int n_tiles = (n_rows + R - 1) / R;
  const int tid = threadIdx.x;
  const unsigned long long pol = evict_first();
  auto base = [&](int s) { return smem_raw + s * C::kStageBytes; };
  auto sval = [&](int s) { return reinterpret_cast<double*>(base(s)); };
  auto sx = [&](int s) { return reinterpret_cast<double*>(base(s)) + C::kVal; };
  auto scol = [&](int s) { return reinterpret_cast<int*>(sx(s) + C::kX); };
  auto srp = [&](int s) { return scol(s) + C::kCol; };
  auto tile_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };

  // V(k) into stage s; returns whether tile k is staged (uniform over the CTA)
  auto issue_v = [&](int k, int s) -> bool {
    const int t = tile_of(k);
    bool staged = false;
    if (t < n_tiles && aligned) {
      const int r0 = t * R, r1 = min(r0 + R, n_rows);
      const long long b0 = __ldg(row_ptr + r0), b1 = __ldg(row_ptr + r1);
      if (b1 - b0 <= C::kMaxBlocks) {
        staged = true;
        const long long v0 = b0 * N2, v1 = b1 * N2, va = v0 & ~1ll;
        const int npair = static_cast<int>((v1 - va + 1) >> 1);
        double* sv = sval(s);
        for (int k2 = tid; k2 < npair; k2 += T) {
          const long long g = va + 2 * k2;
          if (g + 1 < v1) cp16s(sv + 2 * k2, val + g, pol);
          else cp8s(sv + 2 * k2, val + g, pol);
        }
        int* sc = scol(s);
        for (int k2 = tid; k2 < b1 - b0; k2 += T) cp4s(sc + k2, col + b0 + k2, pol);
        int* sr = srp(s);
        for (int k2 = tid; k2 <= r1 - r0; k2 += T) cp4s(sr + k2, row_ptr + r0 + k2, pol);
      }
    }
    commit();
    return staged;
  };
  // X(k) into stage s (V(k) has landed and is visible)
  auto issue_x = [&](int k, int s, bool staged) {
    const int t = tile_of(k);
    if (staged && t < n_tiles) {
      const int r0 = t * R, r1 = min(r0 + R, n_rows);
      const int* sr = srp(s);
      const int nb = sr[r1 - r0] - sr[0];
      const int* sc = scol(s);
      double* xs = sx(s);
      for (int k2 = tid; k2 < nb * NL; k2 += T) {
        const int b = k2 / NL, j = k2 - b * NL;
        cp8(xs + k2, x + static_cast<long long>(sc[b]) * NL + j);
      }
    }
    commit();
  };

  if (static_cast<int>(blockIdx.x) >= n_tiles) return;
  unsigned staged = 0;  // bit (k % S): tile k is staged
#pragma unroll
  for (int j = 0; j < S - 1; ++j) staged |= issue_v(j, j) ? 1u << j : 0u;
#pragma unroll
  for (int j = 0; j < S - 2; ++j) {
    wait_group<S - 2>();  // V(j) has landed
    __syncthreads();
    issue_x(j, j, (staged >> j) & 1u);
  }
  for (int k = 0; tile_of(k) < n_tiles; ++k) {
    const int s = k % S;
    {
      const int sv = (k + S - 1) % S;
      staged = (staged & ~(1u << sv)) | (issue_v(k + S - 1, sv) ? 1u << sv : 0u);
    }
    wait_group<(S == 3 ? 1 : 2)>();  // V(k+S-2) and X(k) have landed
    __syncthreads();
    {
      const int sx2 = (k + S - 2) % S;
      issue_x(k + S - 2, sx2, (staged >> sx2) & 1u);
    }
    const int t = tile_of(k);
    const int r0 = t * R, r1 = min(r0 + R, n_rows);
    const int el = tid / NL, i = tid - el * NL;
    if (el < R && r0 + el < r1) {
      const int e = r0 + el;
      double acc = accumulate ? y[static_cast<long long>(e) * NL + i] : 0.0;
      if ((staged >> s) & 1u) {
        const int* sr = srp(s);
        const int b0 = sr[0], bs = sr[el] - b0, be = sr[el + 1] - b0;
        const int off = static_cast<int>((static_cast<long long>(b0) * N2) & 1);
        const double* v = sval(s) + off + i * NL;
        const double* xs = sx(s);
#pragma unroll
        for (int b = 0; b < kMaxPerRow; ++b) {
          if (bs + b < be) {
#pragma unroll
            for (int j = 0; j < NL; ++j) acc = fma(v[(bs + b) * N2 + j], xs[(bs + b) * NL + j], acc);
          }
        }
        for (int b = bs + kMaxPerRow; b < be; ++b) {  // rows above kMaxPerRow blocks
#pragma unroll
          for (int j = 0; j < NL; ++j) acc = fma(v[b * N2 + j], xs[b * NL + j], acc);
        }
      } else {
        const int bs = __ldg(row_ptr + e), be = __ldg(row_ptr + e + 1);
        acc = row_dot_global<NL>(val + static_cast<long long>(bs) * N2 + i * NL, col + bs, be - bs, x);
      }
      y[static_cast<long long>(e) * NL + i] = acc;
    }
    __syncthreads();    // stage s is refilled by V(k+S)
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}

}
extern "C" int lab_spmv_acc(int threads, int nrows, const int* rp, const int* col,
                        const double* val, const double* x, double* y, int accumulate, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  using C = v4::Cfg<3, 128, 3>;
  auto k = v4::bsr_spmv_kernel<3, 128, 3>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kBytes);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 128, C::kBytes);
  long long nt = (nrows + C::R - 1) / C::R;
  int grid = (int)std::min<long long>(nt, (long long)sms * std::max(per, 1));
  k<<<grid, 128, C::kBytes, s>>>(nrows, rp, col, val, x, y, 1, accumulate);
  return per;
}

extern "C" int lab_spmv(int variant, int threads, int nrows, const int* rp, const int* col,
                        const double* val, const double* x, double* y, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int aligned = (reinterpret_cast<uintptr_t>(val) & 15) == 0;
#define RUN(NS, T)                                                                              \
  {                                                                                             \
    using C = NS::Cfg<3, T>;                                                                    \
    auto k = NS::bsr_spmv_kernel<3, T>;                                                         \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kBytes);       \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, T, C::kBytes);                      \
    long long nt = (nrows + C::R - 1) / C::R;                                                   \
    int grid = (int)std::min<long long>(nt, (long long)sms * std::max(per, 1));                 \
    k<<<grid, T, C::kBytes, s>>>(nrows, rp, col, val, x, y, aligned);                           \
  }
#define RUN4(T, S)                                                                              \
  {                                                                                             \
    using C = v4::Cfg<3, T, S>;                                                                 \
    auto k = v4::bsr_spmv_kernel<3, T, S>;                                                      \
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kBytes);       \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, T, C::kBytes);                      \
    long long nt = (nrows + C::R - 1) / C::R;                                                   \
    int grid = (int)std::min<long long>(nt, (long long)sms * std::max(per, 1));                 \
    k<<<grid, T, C::kBytes, s>>>(nrows, rp, col, val, x, y, aligned, 0);                        \
  }
  if (variant == 2 && threads == 256) RUN(v2, 256)
  else if (variant == 2 && threads == 128) RUN(v2, 128)
  else if (variant == 2 && threads == 512) RUN(v2, 512)
  else if (variant == 3 && threads == 256) RUN(v3, 256)
  else if (variant == 3 && threads == 128) RUN(v3, 128)
  else if (variant == 3 && threads == 512) RUN(v3, 512)
  else if (variant == 43 && threads == 128) RUN4(128, 3)
  else if (variant == 44 && threads == 128) RUN4(128, 4)
  else if (variant == 45 && threads == 128) RUN4(128, 5)
  else if (variant == 46 && threads == 128) RUN4(128, 6)
  else if (variant == 44 && threads == 256) RUN4(256, 4)
  else if (variant == 45 && threads == 256) RUN4(256, 5)
  else if (variant == 44 && threads == 64) RUN4(64, 4)
  else if (variant == 46 && threads == 64) RUN4(64, 6)
  else return -1;
  return per;
}
