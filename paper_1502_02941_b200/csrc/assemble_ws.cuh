// assemble_ws.cuh -- warp-specialised block-row kernel for the tensor-core P-form (constant
// velocity, bound mesh; config 2's kernel).  Included by dg_assembly.cu after assemble_v2.cuh.
//
// The monolithic kernel (assemble_v2.cuh) runs each warp through two phases back to back:
// the per-element pass (gathers, geometry, source and edge terms: FP64-latency-bound, the
// memory system idle) and the block products and fragment stores (HBM-write-bound).  With
// every warp of an SM in the same phase at the same time the two costs ADD (measured with the
// ablation option: 0.0625 ms without block stores + 0.075 ms of stores = 0.1377 ms for the
// config-2 batch).  Here they overlap: one persistent CTA per SM holds NP producer warps and NP
// consumer warps, paired.  Producer p runs the per-element pass of a 32-element chunk into a
// shared-memory slot (the DMMA A operand rows, the edge metadata, the row pointers) and writes
// the chunk's row_ptr, block columns and RHS; consumer p runs the products and stores of the
// previous chunk from the other slot.  Two slots per pair, handed over with mbarriers.
#pragma once

namespace dgb {
namespace v2 {

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" :: "r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" :: "r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" :: "r"(smem_addr(bar)), "r"(parity) : "memory");
}

template <int NL, int NQV, int NQE, int NPROD = 8, int NCONS = 8>
struct SmemWs {
  using SM = Smem<NL, NQV, NQE, 0>;
  static constexpr int NP = NPROD;               // producer warps per CTA
  static constexpr int NC = NCONS;               // consumer warps per CTA
  static constexpr int NS = NP + NC;             // chunk slots (ring)
  static constexpr int kThreads = 32 * (NP + NC);
  static constexpr int kInts = 3 * 32 + 48 + 64; // meta [3][32], row map [48], rp / diag slot
  static constexpr int kSlot = SM::kStash + kInts / 2;  // doubles
  static constexpr int kRhs = SM::kRhs;          // producer RHS staging [32][NL]
  static constexpr int kBars = NS * 2;           // full / empty per slot
  static constexpr size_t kBytes = sizeof(double) * (size_t(kBars) + NS * kSlot + NP * kRhs);
};

// Producer: the per-element pass of the chunk starting at e_first (relative to row_begin).
// Mirrors assemble_kernel phases A0-A2 (assemble_v2.cuh) for BK = 0 on a bound mesh.
template <int NL, int NQV, int NQE, bool FUSE>
__device__ __forceinline__ void ws_produce(const Params2<NL, NQV, NQE, false, full_tensors(NL, 0)>& P,
                                           int e_first, int lane, double* slot, double* srhs,
                                           int n_sets) {
  using L = Lay<NL, NQV, NQE, false, false>;
  using SM = Smem<NL, NQV, NQE, 0>;
  constexpr int CT = SM::kCT, OB = SM::kDRows;
  double* sk = slot;
  int* mk = reinterpret_cast<int*>(slot + SM::kStash);
  int* xfer = mk + 96 + 48;
  const double kappa = P.bt[0].kappa, sigma_i = P.bt[0].sigma_i, sigma_b = P.bt[0].sigma_b;
  const int e = P.row_begin + e_first + lane;
  const bool active = e < P.row_end;
  const int ee = active ? e : P.row_end - 1;
  const dgb_vector_field& bf = P.prob.advection;
  if constexpr (FUSE) {
#pragma unroll
    for (int i = 0; i < NL; ++i) srhs[lane * NL + i] = 0.0;  // Fk
  }

  int v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * ee + k);
  const int4 anb = __ldg(P.adj_nb + (ee - P.row_begin));
  const int4 aop = __ldg(P.adj_op + (ee - P.row_begin));
  double2 pv[3], po[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pv[k] = __ldg(reinterpret_cast<const double2*>(P.nodes) + v[k]);
  po[0] = __ldg(reinterpret_cast<const double2*>(P.nodes) + max(aop.x, 0));
  po[1] = __ldg(reinterpret_cast<const double2*>(P.nodes) + max(aop.y, 0));
  po[2] = __ldg(reinterpret_cast<const double2*>(P.nodes) + max(aop.z, 0));
  const double B00 = FSUB(pv[1].x, pv[0].x), B01 = FSUB(pv[2].x, pv[0].x);
  const double B10 = FSUB(pv[1].y, pv[0].y), B11 = FSUB(pv[2].y, pv[0].y);
  const double det = FSUB(FMUL(B00, B11), FMUL(B01, B10));
  const double rdet = rcp_nr(det);
  const double G00 = B11 * rdet, G01 = -B10 * rdet;
  const double G10 = -B01 * rdet, G11 = B00 * rdet;
  const double eps = scalar_element(P.prob.diffusion, ee);

  // RHS volume term
  double F[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) F[i] = 0.0;
  {
    source_points<NQV, false>(
        P.prob.source, ee, DGB_ABLATE(2),
        [&](int q, double& px, double& py) {
          // volume points only evaluate coefficients (no term selection): fused
          px = fma(B01, P.t.x[L::VY + q], fma(B00, P.t.x[L::VX + q], pv[0].x));
          py = fma(B11, P.t.x[L::VY + q], fma(B10, P.t.x[L::VX + q], pv[0].y));
        },
        [&](int q, double f, double, double) {
          const double c = det * P.t.x[L::VW + q] * f;
#pragma unroll
          for (int i = 0; i < NL; ++i) F[i] = fma(c, P.t.x[L::PHI + q * NL + i], F[i]);
        });
  }

  // per local edge: A-operand rows W0 W1 P (diagonal) and X Y0 Y1 Z0 Z1 (neighbour), boundary RHS
  int fcol[3] = {-1, -1, -1};
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int a = v[(l + 1) % 3], b = v[(l + 2) % 3];
    const int o = a < b ? 0 : 1;  // make_side orientation (assembly.cpp:125-126)
    const double2 A = o == 0 ? pv[(l + 1) % 3] : pv[(l + 2) % 3];
    const double2 Bn = o == 0 ? pv[(l + 2) % 3] : pv[(l + 1) % 3];
    const double dx = FSUB(Bn.x, A.x), dy = FSUB(Bn.y, A.y);
    // edge_geometry (mesh.cpp:232-257): length and its reciprocal from one rsqrt
    const double rh = rsqrt_nr(fma(dx, dx, dy * dy));
    const double h = fma(dx, dx, dy * dy) * rh;
    const double tx = dx * rh, ty = dy * rh;
    const double nx = o == 0 ? ty : -ty, ny = o == 0 ? -tx : tx;
    const double ge0 = G00 * nx + G10 * ny, ge1 = G01 * nx + G11 * ny;
    const int kind = (anb.w >> (4 * l)) & 3;
    const int lf = (anb.w >> (4 * l + 2)) & 3;
    const int f = l == 0 ? anb.x : (l == 1 ? anb.y : anb.z);
    double w0 = 0.0, w1 = 0.0, cp = 0.0, y0 = 0.0, y1 = 0.0, z0 = 0.0, z1 = 0.0, cx = 0.0;
    if (kind == DGB_EDGE_INTERIOR) {
      const double2 qo = l == 0 ? po[0] : (l == 1 ? po[1] : po[2]);
      const double2 qa = l == 0 ? pv[1] : (l == 1 ? pv[2] : pv[0]);
      const double2 qb = l == 0 ? pv[2] : (l == 1 ? pv[0] : pv[1]);
      const Geo gf = element_geo_coords(qo, qb, qa);  // rotated order (opposite, b, a)
      double eps_e = eps;
      if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
        const double ef = __ldg(P.prob.diffusion.per_element + f);
        eps_e = ee < f ? 0.5 * (eps + ef) : 0.5 * (ef + eps);
      }
      fcol[l] = f;
      const double base = 0.5 * h * eps_e;
      w0 = base * ge0;
      w1 = base * ge1;
      y0 = -base * (gf.G00 * nx + gf.G10 * ny);
      y1 = -base * (gf.G01 * nx + gf.G11 * ny);
      z0 = -1.0 * base * ge0;  // kappa lives in the B operand's Z rows
      z1 = -1.0 * base * ge1;
      const double sh = sigma_i * rh;
      const double fl = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
      const double up = fl < 0.0 ? FMUL(h, fl) : 0.0;
      cp = sh * (h * eps_e) - up;
      cx = up - sh * (h * eps_e);
    } else {
      double fls[NQE], gb[NQE];
      bool inflow = false;
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double tq = o == 0 ? P.t.x[L::ET + p] : 1.0 - P.t.x[L::ET + p];
        const double px = FADD(A.x, FMUL(tq, dx));
        const double py = FADD(A.y, FMUL(tq, dy));
        const double bx = bf.p[0], by = bf.p[1];
        fls[p] = FADD(FMUL(bx, nx), FMUL(by, ny));
        if (fls[p] < -1e-12 * fmax(1.0, hypot_dd(bx, by))) inflow = true;  // assembly.cpp:324-401
        gb[p] = scalar_point(kind == DGB_EDGE_NEUMANN ? P.prob.neumann : P.prob.dirichlet, px, py);
      }
      double cG[NQE], cH[NQE];
      if (kind == DGB_EDGE_NEUMANN) {
        const int edge = __ldg(P.element_edges + 3 * ee + l);
        if (inflow && !P.drop_neumann && active) {
          atomicMax(P.err_edge, (P.epoch << 32) | (0xFFFFFFFFull - static_cast<unsigned>(edge)));
        }
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          cG[p] = FMUL(FMUL(P.t.x[L::EW + p], h), gb[p]);  // neumann_rhs (assembly.cpp:427-442)
          cH[p] = 0.0;
        }
      } else {
        const double base = h * eps;
        w0 = base * ge0;
        w1 = base * ge1;
        const double sh = sigma_b * rh;
        cp = sh * (h * eps) - ((inflow && fls[0] < 0.0) ? FMUL(h, fls[0]) : 0.0);
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double w = FMUL(P.t.x[L::EW + p], h);
          const double win = (inflow && fls[p] < 0.0) ? -FMUL(w, fls[p]) : 0.0;
          const double wgd = w * gb[p];
          cG[p] = wgd * (sh * eps) + win * gb[p];
          cH[p] = FUSE ? wgd * eps : wgd * (kappa * eps);
        }
      }
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double h0 = cH[p] * ge0, h1 = cH[p] * ge1;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          if constexpr (FUSE) {
            F[i] = fma(cG[p], P.t.x[L::EPHI + (l * NQE + p) * NL + i], F[i]);
            srhs[lane * NL + i] =
                fma(h0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i],
                    fma(h1, P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], srhs[lane * NL + i]));
          } else {
            F[i] = fma(cG[p], P.t.x[L::EPHI + (l * NQE + p) * NL + i],
                       fma(h0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i],
                           fma(h1, P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], F[i])));
          }
        }
      }
    }
    sk[(6 + 2 * l) * CT + lane] = w0;
    sk[(7 + 2 * l) * CT + lane] = w1;
    sk[(12 + l) * CT + lane] = cp;
    double* so = sk + (OB + 5 * l) * CT + lane;
    so[0] = cx;
    so[CT] = y0;
    so[2 * CT] = y1;
    so[3 * CT] = z0;
    so[4 * CT] = z1;
    mk[l * 32 + lane] = kind | (lf << 2);
  }

  // sorted block columns -> slots (rank among the row's columns)
  int slot_of[4];
  {
    const int cx[4] = {ee, fcol[0], fcol[1], fcol[2]};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) r += (j != i && cx[j] >= 0 && cx[j] < cx[i]) ? 1 : 0;
      slot_of[i] = r;
    }
  }
  const int rp = __ldg(P.row_ptr_src + (ee - P.row_begin));
  if (active) {
    const int rp1 = __ldg(P.row_ptr_src + (ee - P.row_begin + 1));
#pragma unroll 1
    for (int s = 0; s < n_sets; ++s) {
      int32_t* rpo = P.bt[s].row_ptr;
      int32_t* co = P.bt[s].col;
      rpo[ee - P.row_begin + 1] = rp1;
      if (ee == P.row_begin) rpo[0] = 0;
      co[rp + slot_of[0]] = ee;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        if (fcol[l] >= 0) co[rp + slot_of[1 + l]] = fcol[l];
      }
    }
  }
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (fcol[l] >= 0) mk[l * 32 + lane] |= slot_of[1 + l] << 4;
  }
  xfer[lane] = active ? rp : -1;
  xfer[32 + lane] = slot_of[0];

  // RHS: per set F0 (+ kappa_s Fk), coalesced 16-byte stores of the chunk's contiguous slice
  const unsigned long long pol = output_policy(P.evict_first);
  {
    double fk[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) fk[i] = FUSE ? srhs[lane * NL + i] : 0.0;
    const int n_here = min(32, P.row_end - P.row_begin - e_first);
    const int n = n_here * NL;
#pragma unroll 1
    for (int s = 0; s < n_sets; ++s) {
      const double ks = P.bt[s].kappa;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NL; ++i) srhs[lane * NL + i] = FUSE ? fma(ks, fk[i], F[i]) : F[i];
      __syncwarp();
      double* dst = P.bt[s].rhs + static_cast<long long>(e_first) * NL;
      for (int idx = 2 * lane; idx + 1 < n; idx += 64) {
        store_pair(dst + idx, srhs[idx], srhs[idx + 1], pol);
      }
      if (n > 0 && (n & 1) && lane == 0) store_one(dst + n - 1, srhs[n - 1], pol);
    }
    __syncwarp();  // srhs is rewritten by the next chunk
  }

  // diagonal A rows: S0 S1 S2 M T0 T1 (W and P rows written above), zero K padding
  {
    const double alpha = scalar_element(P.prob.linear_reaction, ee);
    const double de = det * eps;
    sk[0 * CT + lane] = de * (G00 * G00 + G10 * G10);
    sk[1 * CT + lane] = de * (G00 * G01 + G10 * G11);
    sk[2 * CT + lane] = de * (G01 * G01 + G11 * G11);
    sk[3 * CT + lane] = det * alpha;
    sk[4 * CT + lane] = det * (G00 * bf.p[0] + G10 * bf.p[1]);
    sk[5 * CT + lane] = det * (G01 * bf.p[0] + G11 * bf.p[1]);
#pragma unroll
    for (int k = SM::kTerms; k < SM::kDRows; ++k) sk[k * CT + lane] = 0.0;
  }
}

// Consumer, diagonal block: D = C . B (SPLIT: + kappa_s C . Bq per set, see
// mma_block_store_split).  The next n-tile's B fragments are loaded while this one's products
// run, and all four m-tiles' products are issued before their stores.
template <int KS, int NT, int N2, bool SPLIT, class AF>
__device__ __forceinline__ void ws_diag(AF a_at, const double* __restrict__ frag, long long base,
                                        const MethodOut* bt, int n_sets, int lane,
                                        unsigned long long pol) {
  constexpr int NB = KS + (SPLIT ? 2 : 0);  // B fragments per n-tile
  const int g = lane >> 2, t = lane & 3;
  double af[4][KS];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) af[m][ks] = a_at(m, ks);
  }
  long long bm[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) bm[m] = __shfl_sync(0xffffffffu, base, 8 * m + g);
  const double* fq = frag + KS * NT * 32;
  auto load_b = [&](int nt, double (&b)[NB]) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) b[ks] = __ldg(frag + (ks * NT + nt) * 32 + lane);
    if constexpr (SPLIT) {
      b[KS] = __ldg(fq + nt * 32 + lane);
      b[KS + 1] = __ldg(fq + (NT + nt) * 32 + lane);
    }
  };
  double bn[NB];
  load_b(0, bn);
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    double bf[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) bf[i] = bn[i];
    if (nt + 1 < NT) load_b(nt + 1, bn);
    double d[4][2], q[4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      d[m][0] = d[m][1] = q[m][0] = q[m][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma_8x8x4(d[m][0], d[m][1], af[m][ks], bf[ks]);
      if constexpr (SPLIT) {
        dmma_8x8x4(q[m][0], q[m][1], af[m][1], bf[KS]);
        dmma_8x8x4(q[m][0], q[m][1], af[m][2], bf[KS + 1]);
      }
    }
    const int n0 = 8 * nt + 2 * t;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      if (bm[m] < 0) continue;
      if constexpr (SPLIT) {
#pragma unroll
        for (int s = 0; s < kMaxBatch; ++s) {
          if (s < n_sets) {
            const double k = bt[s].kappa;
            store_entries<N2>(bt[s].val + bm[m], n0, fma(k, q[m][0], d[m][0]),
                              fma(k, q[m][1], d[m][1]), pol);
          }
        }
      } else {
        store_entries<N2>(bt[0].val + bm[m], n0, d[m][0], d[m][1], pol);
      }
    }
  }
}

// Consumer: the block products and fragment stores of a produced chunk.
template <int NL, int NQV, int NQE, bool FUSE>
__device__ __forceinline__ void ws_consume(const Params2<NL, NQV, NQE, false, full_tensors(NL, 0)>& P, int lane,
                                           double* slot, int n_sets) {
  using SM = Smem<NL, NQV, NQE, 0>;
  constexpr int N2 = NL * NL, CT = SM::kCT, NT = SM::kNT;
  const double* sk = slot;
  int* mk = reinterpret_cast<int*>(slot + SM::kStash);
  const int* xfer = mk + 96 + 48;
  const int g = lane >> 2, t = lane & 3;
  const int rp = xfer[lane];
  const bool active = rp >= 0;
  const int diag_slot = xfer[32 + lane];
  const unsigned long long pol = output_policy(P.evict_first);
  const double* frag = P.bt[0].bfrag;

  if (!(DGB_ABLATE(8))) {
    const long long base = (active && !(DGB_ABLATE(1))) ? static_cast<long long>(rp + diag_slot) * N2 : -1LL;
    auto a_at = [&](int m, int ks) { return sk[(4 * ks + t) * CT + 8 * m + g]; };
    ws_diag<SM::kKS, NT, N2, FUSE>(a_at, frag, base, P.bt, n_sets, lane, pol);
  }

  int* pmap = mk + 96;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int meta = mk[l * 32 + lane];
    const bool has = (meta & 3) == DGB_EDGE_INTERIOR;
    if (!__any_sync(0xffffffffu, has)) continue;
    if (DGB_ABLATE(4)) continue;
    const int lf = (meta >> 2) & 3, bslot = meta >> 4;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned m0 = __ballot_sync(0xffffffffu, has && lf == 0);
    const unsigned m1 = __ballot_sync(0xffffffffu, has && lf == 1);
    const unsigned m2 = __ballot_sync(0xffffffffu, has && lf == 2);
    const int t1 = (__popc(m0) + 7) >> 3, t2 = t1 + ((__popc(m1) + 7) >> 3);
    const int ntiles = t2 + ((__popc(m2) + 7) >> 3);
    pmap[lane] = -1;
    if (lane < 16) pmap[32 + lane] = -1;
    __syncwarp();
    if (has) {
      const unsigned mv = lf == 0 ? m0 : (lf == 1 ? m1 : m2);
      const int tv = lf == 0 ? 0 : (lf == 1 ? t1 : t2);
      pmap[8 * tv + __popc(mv & lt)] = lane;
    }
    __syncwarp();
    const long long my_base = (active && has) ? static_cast<long long>(rp + bslot) * N2 : -1LL;
    const double* so = sk + (SM::kDRows + 5 * l) * CT;
    // k-step 0: X Y0 Y1 (FUSE: Z apart in k-step 1) / X Y0 Y1 Z0, k-step 1: Z1 (kappa-folded)
    auto rows = [&](int r, double& a0, double& a1, long long& bm) {
      const int src = pmap[8 * r + g];
      const int sl = src < 0 ? 0 : src;
      if constexpr (FUSE) {
        a0 = (src < 0 || t >= 3) ? 0.0 : so[t * CT + sl];
        a1 = (src < 0 || t >= 2) ? 0.0 : so[(3 + t) * CT + sl];
      } else {
        a0 = src < 0 ? 0.0 : so[t * CT + sl];
        a1 = (src < 0 || t >= 1) ? 0.0 : so[4 * CT + sl];
      }
      bm = __shfl_sync(0xffffffffu, my_base, sl);
      if (src < 0) bm = -1;
    };
    double a0, a1;
    long long bm;
    if (ntiles > 0) rows(0, a0, a1, bm);
#pragma unroll
    for (int v = 0; v < 3; ++v) {
      const int tb = v == 0 ? 0 : (v == 1 ? t1 : t2), te = v == 0 ? t1 : (v == 1 ? t2 : ntiles);
      if (tb == te) continue;
      const double* fr = frag + SM::kFragTile + (FUSE ? 2 * NT * 32 : 0) +
                         (l * 3 + v) * SM::kOffTile + lane;
      double bv[2][NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        bv[0][nt] = __ldg(fr + nt * 32);
        bv[1][nt] = __ldg(fr + (NT + nt) * 32);
      }
#pragma unroll 1
      for (int r = tb; r < te; ++r) {
        const double c0 = a0, c1 = a1;
        const long long cb = bm;
        if (r + 1 < ntiles) rows(r + 1, a0, a1, bm);
        // all n-tiles' products first (DMMA latency overlapped), then the stores
        double d[NT][2], z[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          d[nt][0] = d[nt][1] = z[nt][0] = z[nt][1] = 0.0;
          if constexpr (FUSE) {
            dmma_8x8x4(d[nt][0], d[nt][1], c0, bv[0][nt]);
            dmma_8x8x4(z[nt][0], z[nt][1], c1, bv[1][nt]);
          } else {
            dmma_8x8x4(d[nt][0], d[nt][1], c0, bv[0][nt]);
            dmma_8x8x4(d[nt][0], d[nt][1], c1, bv[1][nt]);
          }
        }
        if (cb >= 0 && !(DGB_ABLATE(1))) {
          if constexpr (FUSE) {
#pragma unroll
            for (int s = 0; s < kMaxBatch; ++s) {
              if (s < n_sets) {
                const double k = P.bt[s].kappa;
                double* dst = P.bt[s].val + cb;
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) {
                  store_entries<N2>(dst, 8 * nt + 2 * t, fma(k, z[nt][0], d[nt][0]),
                                    fma(k, z[nt][1], d[nt][1]), pol);
                }
              }
            }
          } else {
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              store_entries<N2>(P.bt[0].val + cb, 8 * nt + 2 * t, d[nt][0], d[nt][1], pol);
            }
          }
        }
      }
    }
    __syncwarp();  // the row map is rebuilt for the next l
  }
}

// Persistent warp-specialised kernel: one CTA per SM.  The CTA's chunks (32 elements each,
// chunk blockIdx.x + k gridDim.x for k = 0, 1, ..) go round-robin to its NP producer warps and
// NC consumer warps through a ring of NS slots: chunk k uses slot k % NS, round k / NS.
template <int NL, int NQV, int NQE, bool FUSE, int NPROD, int NCONS>
__global__ void __launch_bounds__(SmemWs<NL, NQV, NQE, NPROD, NCONS>::kThreads, 1)
    assemble_ws_kernel(const __grid_constant__ Params2<NL, NQV, NQE, false, full_tensors(NL, 0)> P) {
  using W = SmemWs<NL, NQV, NQE, NPROD, NCONS>;
  constexpr int NP = W::NP, NC = W::NC, NS = W::NS;
  extern __shared__ double smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);  // [NS][full, empty]
  double* slots = smem + W::kBars;
  double* rhs_st = slots + NS * W::kSlot;
  if (threadIdx.x < W::kBars) mbar_init(bars + threadIdx.x, 32);
  __syncthreads();
  if (DGB_ABLATE(16)) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp < NP;
  const int n_sets = FUSE ? P.n_batch : 1;
  const int n_rows = P.row_end - P.row_begin;
  const int n_chunks = (n_rows + 31) >> 5;
  const int n_local = n_chunks > static_cast<int>(blockIdx.x)
                          ? (n_chunks - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                          : 0;
  if (producer) {
    for (int k = warp; k < n_local; k += NP) {
      const int s = k % NS, r = k / NS;
      double* slot = slots + s * W::kSlot;
      if (r > 0) mbar_wait(bars + 2 * s + 1, (r - 1) & 1);  // empty: round r - 1 consumed
      const int c = blockIdx.x + k * gridDim.x;
      ws_produce<NL, NQV, NQE, FUSE>(P, c * 32, lane, slot, rhs_st + warp * W::kRhs, n_sets);
      mbar_arrive(bars + 2 * s);
    }
  } else {
    for (int k = warp - NP; k < n_local; k += NC) {
      const int s = k % NS, r = k / NS;
      mbar_wait(bars + 2 * s, r & 1);                       // full: round r produced
      ws_consume<NL, NQV, NQE, FUSE>(P, lane, slots + s * W::kSlot, n_sets);
      mbar_arrive(bars + 2 * s + 1);
    }
  }
}

}  // namespace v2
}  // namespace dgb
