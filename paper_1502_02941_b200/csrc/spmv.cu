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
// * A pipeline of S stages: the value stream of a tile is issued S-1 tiles ahead and the x
//   gathers it names S-2 tiles ahead (cp.async into shared memory), so the compute step reads
//   shared memory only; CTAs are persistent over tiles (grid = SMs x resident CTAs).
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
                                                     double* __restrict__ y, int aligned) {
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
      double acc = 0.0;
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

template <int NL, int T, int S>
void launch(const dgb_bsr* a, const double* x, double* y, cudaStream_t s) {
  using C = Cfg<NL, T, S>;
  if (a->n_block_rows <= 0) return;
  int dev = 0, sms = 0, per_sm = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  ensure_dynamic_smem(reinterpret_cast<const void*>(bsr_spmv_kernel<NL, T, S>), C::kBytes,
                      "cudaFuncSetAttribute(spmv)");
  cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev), "sm count");
  cuda_check(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bsr_spmv_kernel<NL, T, S>, T, C::kBytes),
             "occupancy(spmv)");
  const long long n_tiles = (static_cast<long long>(a->n_block_rows) + C::R - 1) / C::R;
  const int grid = static_cast<int>(std::min<long long>(n_tiles, static_cast<long long>(sms) * std::max(per_sm, 1)));
  const int aligned = (reinterpret_cast<uintptr_t>(a->val) & 15) == 0;
  bsr_spmv_kernel<NL, T, S><<<grid, T, C::kBytes, s>>>(a->n_block_rows, a->row_ptr, a->col, a->val, x, y, aligned);
}

}  // namespace spmv

void launch_bsr_spmv(const dgb_bsr* a, const double* x, double* y, cudaStream_t s) {
  // 128-thread CTAs, three stages: measured best on config 4 (tools/spmv_lab.py; deeper
  // pipelines, larger CTAs, L2 persistence on x and column-split passes were all slower)
  switch (a->block_dim) {
    case 3: spmv::launch<3, 128, 3>(a, x, y, s); break;
    case 6: spmv::launch<6, 128, 3>(a, x, y, s); break;
    case 10: spmv::launch<10, 128, 3>(a, x, y, s); break;
    case 15: spmv::launch<15, 128, 3>(a, x, y, s); break;
    default: throw Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported block size", a->block_dim);
  }
  cuda_check(cudaGetLastError(), "bsr_spmv_kernel");
}

}  // namespace dgb
