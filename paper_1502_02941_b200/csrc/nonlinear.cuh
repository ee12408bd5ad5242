// nonlinear.cuh -- nonlinear reaction vector H(u) and its block-diagonal Jacobian HJ(u)
// (included by dg_assembly.cu).  Replaces dgfem::assemble_nonlinear (nonlinear.cpp:11-107);
// SURVEY.md §8(f) rank 1.
//
// One thread per element for the pointwise part, one warp per 32 elements for HJ:
//  * thread: element_geometry's det (mesh.cpp:212-230, unfused), u_h at every volume point
//    (sum_j coef_j phi_qj in j order, unfused, nonlinear.cpp:41-47), r and r' with the
//    reference's expressions, then H_i = sum_q ((det w_q) r_q) phi_qi in q order, unfused --
//    the same operations in the same order as nonlinear.cpp:48-56, so H is bitwise the
//    reference's;
//  * warp: HJ[32 elements x nl^2] = S[32 x nq] . Phi[nq x nl^2] on the FP64 tensor cores
//    (mma.sync m8n8k4), with S_q = (det w_q) r'_q in shared memory and
//    Phi_q,(i,j) = phi_qj * phi_qi (the reference's rounded product, nonlinear.cpp:61) as a
//    fragment-ordered table; accumulator fragments are stored straight to the element's
//    block (8 elements x 64 contiguous bytes per store instruction).
//  H leaves through shared memory as one bulk copy per warp.
#pragma once

namespace dgb {
namespace nlr {

constexpr int kMaxQ = 64;   // volume points
constexpr int kCT = 36;     // S row stride (doubles): conflict-free A-fragment loads

__device__ __forceinline__ void reaction(int kind, double u, double& r, double& dr) {
  switch (kind) {
    case DGB_REACTION_LINEAR: r = u; dr = 1.0; return;
    case DGB_REACTION_SQUARE: r = __dmul_rn(u, u); dr = __dmul_rn(2.0, u); return;
    case DGB_REACTION_CUBIC:
      r = __dmul_rn(__dmul_rn(u, u), u);
      dr = __dmul_rn(__dmul_rn(3.0, u), u);
      return;
    default: r = 0.0; dr = 0.0; return;
  }
}

struct NlParams {
  const double* nodes;
  const int32_t* elements;
  const double2* geo;   // the plan's bound geometry record [chunk][8][32] (dg_assembly.cu), or null
  const double* coef;
  const double* phi;    // [nq][nl]
  const double* w;      // [nq]
  const double* bfrag;  // [ks][nt][lane]
  double* h;
  double* val;
  int32_t* row_ptr;
  int32_t* col;
  int32_t n_elements;
  int32_t nq;
  int32_t ks;           // ceil(nq / 4)
  int32_t kind;
};

template <int NL>
__global__ void __launch_bounds__(128) nonlinear_kernel(const __grid_constant__ NlParams P) {
  constexpr int N2 = NL * NL, NT = (N2 + 7) / 8;
  extern __shared__ double sm[];
  const int kpad = 4 * P.ks;
  double* sphi = sm;                                  // [nq][NL]
  double* sw = sphi + ((P.nq * NL + 1) & ~1);         // [nq]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* S = sw + ((P.nq + 1) & ~1) + warp * (kpad * kCT + 32 * NL);  // [k][kCT]
  double* sh = S + kpad * kCT;                                         // [32][NL] packed H
  for (int i = threadIdx.x; i < P.nq * NL; i += blockDim.x) sphi[i] = P.phi[i];
  for (int i = threadIdx.x; i < P.nq; i += blockDim.x) sw[i] = P.w[i];
  __syncthreads();

  const int e0 = blockIdx.x * blockDim.x + warp * 32;
  const int e = e0 + lane;
  const bool active = e < P.n_elements;
  const int ee = active ? e : P.n_elements - 1;
  if (e0 >= P.n_elements) return;  // whole warp past the end (warp-uniform)

  // element_geometry's det, unfused (mesh.cpp:212-230)
  double2 pv[3];
  if (P.geo) {
    // the vertices from the record bound with the mesh (copies of the nodes, coalesced): no
    // connectivity read, no random node gathers
    const double2* g = P.geo + static_cast<size_t>(e0 >> 5) * (v2::kGeoRows * 32) + lane;
#pragma unroll
    for (int k = 0; k < 3; ++k) pv[k] = __ldg(g + k * 32);
  } else {
    int v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * ee + k);
#pragma unroll
    for (int k = 0; k < 3; ++k) pv[k] = __ldg(reinterpret_cast<const double2*>(P.nodes) + v[k]);
  }
  const double B00 = __dsub_rn(pv[1].x, pv[0].x), B01 = __dsub_rn(pv[2].x, pv[0].x);
  const double B10 = __dsub_rn(pv[1].y, pv[0].y), B11 = __dsub_rn(pv[2].y, pv[0].y);
  const double det = __dsub_rn(__dmul_rn(B00, B11), __dmul_rn(B01, B10));

  double c[NL], H[NL];
#pragma unroll
  for (int j = 0; j < NL; ++j) {
    c[j] = __ldg(P.coef + static_cast<long long>(ee) * NL + j);
    H[j] = 0.0;
  }
#pragma unroll 1
  for (int q = 0; q < kpad; ++q) {
    if (q >= P.nq) {  // zero K padding of the A operand
      S[q * kCT + lane] = 0.0;
      continue;
    }
    double uh = 0.0;
#pragma unroll
    for (int j = 0; j < NL; ++j) uh = __dadd_rn(uh, __dmul_rn(c[j], sphi[q * NL + j]));
    double r, dr;
    reaction(P.kind, uh, r, dr);
    const double dw = __dmul_rn(det, sw[q]);
    const double s = __dmul_rn(dw, r);
#pragma unroll
    for (int i = 0; i < NL; ++i) H[i] = __dadd_rn(H[i], __dmul_rn(s, sphi[q * NL + i]));
    S[q * kCT + lane] = __dmul_rn(dw, dr);
  }

  // H: the warp's contiguous slice, one bulk copy
#pragma unroll
  for (int i = 0; i < NL; ++i) sh[lane * NL + i] = H[i];
  v2::fence_smem_to_async();  // every writer: its shared-memory stores -> the async (TMA) proxy
  if (active) {
    P.row_ptr[e + 1] = e + 1;
    P.col[e] = e;
    if (e == 0) P.row_ptr[0] = 0;
  }
  __syncwarp();
  {
    const int n_here = min(32, P.n_elements - e0);
    double* dst = P.h + static_cast<long long>(e0) * NL;
    const int bulk = (n_here * NL) & ~1;  // 16-byte multiple; warp slices start 16-B aligned
    if (lane == 0 && bulk > 0) v2::bulk_store(dst, sh, bulk * sizeof(double), false);
    for (int idx = bulk + lane; idx < n_here * NL; idx += 32) dst[idx] = sh[idx];
  }

  // HJ = S . Phi on the tensor cores; fragments stored straight to the element blocks
  const int g = lane >> 2, t = lane & 3;
  long long bm[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int em = e0 + 8 * m + g;
    bm[m] = em < P.n_elements ? static_cast<long long>(em) * N2 : -1LL;
  }
#pragma unroll 2
  for (int nt = 0; nt < NT; ++nt) {
    double d[4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m) d[m][0] = d[m][1] = 0.0;
    // k-steps in chunks of 4: the chunk's B fragments are loaded together, then the products
#pragma unroll 1
    for (int k0 = 0; k0 < P.ks; k0 += 4) {
      double b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        b[u] = k0 + u < P.ks ? __ldg(P.bfrag + (static_cast<long long>(k0 + u) * NT + nt) * 32 + lane) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < P.ks) {
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            v2::dmma_8x8x4(d[m][0], d[m][1], S[(4 * (k0 + u) + t) * kCT + 8 * m + g], b[u]);
          }
        }
      }
    }
    const int n0 = 8 * nt + 2 * t;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (bm[m] < 0) continue;
      double* dst = P.val + bm[m] + n0;
      if constexpr (N2 % 2 == 0) {
        if (n0 < N2) __stcs(reinterpret_cast<double2*>(dst), make_double2(d[m][0], d[m][1]));
      } else {
        if (n0 < N2) __stcs(dst, d[m][0]);
        if (n0 + 1 < N2) __stcs(dst + 1, d[m][1]);
      }
    }
  }
  if (lane == 0) v2::bulk_wait_all();
}

}  // namespace nlr
}  // namespace dgb
