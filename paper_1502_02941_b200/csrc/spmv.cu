// spmv.cu -- y = K x for the assembled BSR (the reference's `matvec`, sparse.cpp:116-129, on
// the CSR that `stiffness()` returns; here on its 1:1 block form).  Used by dgb_spmv (the
// C-ABI A*x check and config 4's 100 products) and by the Krylov solve (solve.cu).
//
// The product is a stream over the values (8 nl^2 bytes per block, >80% of the bytes) plus a
// gather of x by block column.  Design:
//
// * Tiles of R = T / nl consecutive block rows.  A tile's blocks are one contiguous range
//   [row_ptr[r0], row_ptr[r0 + R]) of `val` and `col`, so the CTA stages them in shared memory
//   with 16-byte cp.async copies (LDGSTS: fully coalesced, no registers held in flight).  The
//   per-thread reads of a scalar row (nl doubles at stride nl^2 per block) then come from
//   shared memory instead of touching a different 32-byte sector per lane.
// * Two stages: tile t + grid's copies are in flight while tile t computes; CTAs are persistent
//   over tiles (grid = SMs x resident CTAs), so the HBM stream does not drain between tiles.
// * Thread (row e, i) of a tile computes y[e nl + i]: consecutive threads write consecutive
//   y entries (coalesced stores); the nl threads of a block row read the same x block
//   (one L1 line, broadcast).
// * A tile whose block range exceeds the staged capacity (more than kMaxPerRow blocks per row
//   on average -- never for an assembled DG matrix, which has <= 4) is computed straight from
//   global memory, so any valid BSR is accepted.  So is a `val` that is not 16-byte aligned
//   (every tile then takes the global path).
//
// Bytes per product: 8 nl^2 nnzb + 4 nnzb + 4 (n_rows + 1) + 16 nl n_rows.

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "common.hpp"

namespace dgb {

void cuda_check(cudaError_t err, const char* what);  // dg_assembly.cu
void ensure_dynamic_smem(const void* fn, size_t bytes, const char* what);
namespace spmv {

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

template <int NL, int T>
void launch(const dgb_bsr* a, const double* x, double* y, cudaStream_t s) {
  using C = Cfg<NL, T>;
  if (a->n_block_rows <= 0) return;
  int dev = 0, sms = 0, per_sm = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  ensure_dynamic_smem(reinterpret_cast<const void*>(bsr_spmv_kernel<NL, T>), C::kBytes,
                      "cudaFuncSetAttribute(spmv)");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsr_spmv_kernel<NL, T>, T, C::kBytes),
             "occupancy(spmv)");
  const long long n_tiles = (static_cast<long long>(a->n_block_rows) + C::R - 1) / C::R;
  const int grid = static_cast<int>(std::min<long long>(n_tiles, static_cast<long long>(sms) * std::max(per_sm, 1)));
  const int aligned = (reinterpret_cast<uintptr_t>(a->val) & 15) == 0;
  bsr_spmv_kernel<NL, T><<<grid, T, C::kBytes, s>>>(a->n_block_rows, a->row_ptr, a->col, a->val, x, y, aligned);
}

}  // namespace spmv

void launch_bsr_spmv(const dgb_bsr* a, const double* x, double* y, cudaStream_t s) {
  switch (a->block_dim) {
    case 3: spmv::launch<3, 256>(a, x, y, s); break;
    case 6: spmv::launch<6, 256>(a, x, y, s); break;
    case 10: spmv::launch<10, 128>(a, x, y, s); break;
    case 15: spmv::launch<15, 128>(a, x, y, s); break;
    default: throw Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported block size", a->block_dim);
  }
  cuda_check(cudaGetLastError(), "bsr_spmv_kernel");
}

}  // namespace dgb
