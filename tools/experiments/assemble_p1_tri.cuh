// assemble_p1_tri.cuh -- the P1 block-row kernel with THREE lanes per element (bound mesh,
// constant velocity: configs 1 and 4), included by dg_assembly.cu after assemble_p1.cuh.
//
// The one-lane-per-element kernels (assemble_p1.cuh) run each element's whole block row as one
// long dependent instruction stream -- source at 6 points, volume terms, then three faces --
// and at the 166 registers that stream needs only 12 warps fit on an SM: ncu shows the FP64
// pipe half idle and `wait` (fixed-latency dependency) the top stall.  Here lane (j, l) of a
// warp's group j (lanes 3j .. 3j+2, ten elements per warp, lanes 30-31 idle) does element j's
// share l of the work:
//
//   * the source at points q = l, l + 3, ... (a partial RHS, summed over the group by shuffles);
//   * row l of the diagonal block's volume terms;
//   * local edge l: its geometry, its neighbour block (written whole by this lane) and, on the
//     boundary, its RHS terms; the edge's three diagonal-block coefficients (w0, w1, cp) go to
//     the row owners by shuffles, and every lane adds the face terms of edges 0, 1, 2 -- in that
//     order, as the one-lane kernel does -- to its own diagonal row.
//
// Every term is the same expression as in p1_row (assemble_p1.cuh); only the source's point
// sum and the RHS's edge sum are regrouped across lanes (they are within a few ulp of the
// one-lane sums).  Tensors indexed by the lane's role (row l, edge l, point q) come from a
// shared-memory copy of the parameter table, so no lane-divergent constant-bank access remains.
// The warp's ten block rows are one contiguous BSR range: staged in shared memory and copied
// out with 16-byte stores, as in the persistent one-lane kernel.
#pragma once

namespace dgb {
namespace v2 {

template <int NQV, int NQE>
struct SmemP1Tri {
  using L = Lay<3, NQV, NQE, false, true>;
  static constexpr int kTab = (L::TOTAL + 1) & ~1;               // parameter table copy
  static constexpr int kTr = (3 * NQE * 3 * 3 + 1) & ~1;          // neighbour trace table
  static constexpr int kStage = (10 * 4 * 9 + 2 + 1) & ~1;       // a warp's ten block rows
  static size_t bytes(int warps) { return sizeof(double) * (kTab + kTr + size_t(warps) * kStage); }
};

// Element j of group lanes 3j + r: value of lane (3j + r) for r = 0, 1, 2.
__device__ __forceinline__ double grp_shfl(double v, int base, int r) {
  return __shfl_sync(0xffffffffu, v, base + r);
}
__device__ __forceinline__ double2 grp_shfl2(double2 v, int base, int r) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, base + r), __shfl_sync(0xffffffffu, v.y, base + r));
}
template <class T>
__device__ __forceinline__ T sel3(int i, T a, T b, T c) {
  return i == 0 ? a : (i == 1 ? b : c);
}

template <int NQV, int NQE, int WARPS, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) assemble_p1_tri_kernel(
    const __grid_constant__ Params2<3, NQV, NQE, false, true> P) {
  constexpr int NL = 3, N2 = 9;
  using L = Lay<NL, NQV, NQE, false, true>;
  using SM = SmemP1Tri<NQV, NQE>;
  extern __shared__ double smem[];
  double* tab = smem;                 // P.t.x copy (lane-indexed tensors)
  double* tr = smem + SM::kTab;       // neighbour traces, rotated (p1_tables<.., true>)
  for (int i = threadIdx.x; i < L::TOTAL; i += blockDim.x) tab[i] = P.t.x[i];
  p1_tables<NQV, NQE, true>(P, tr);
  __syncthreads();

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mset = blockIdx.y;
  const int grp = lane / 3, l = lane - 3 * grp;   // element of the warp's chunk, role
  const int base = 3 * min(grp, 9);                // group's first lane (lanes 30-31 mirror group 9)
  const bool lane_ok = grp < 10;
  double* stw = smem + SM::kTab + SM::kTr + warp * SM::kStage;

  const double kappa = P.bt[mset].kappa, sigma_i = P.bt[mset].sigma_i, sigma_b = P.bt[mset].sigma_b;
  int32_t* const o_row_ptr = P.bt[mset].row_ptr;
  int32_t* const o_col = P.bt[mset].col;
  double* const o_val = P.bt[mset].val;
  double* const o_rhs = P.bt[mset].rhs;
  const dgb_vector_field& bf = P.prob.advection;
  const double2* nodes2 = reinterpret_cast<const double2*>(P.nodes);
  const unsigned long long pol_out = output_policy(P.evict_first);

  const int n_rows = P.row_end - P.row_begin;
  const int n_chunks = (n_rows + 9) / 10;
  const int gw = blockIdx.x * WARPS + warp, n_gw = gridDim.x * WARPS;

#pragma unroll 1
  for (int c = gw; c < n_chunks; c += n_gw) {
    const int e_first = c * 10;                                   // row offset of the chunk
    const int e = P.row_begin + e_first + min(grp, 9);
    const bool active = lane_ok && e < P.row_end;
    const int ee = min(e, P.row_end - 1);
    const int r = ee - P.row_begin;
    // ---- records (the group's three lanes read the same ones) and this lane's node gathers
    const int4 anb = __ldg(P.adj_nb + r);
    const int4 aop = __ldg(P.adj_op + r);
    int v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * ee + k);
    const int rp = __ldg(P.row_ptr_src + r), rp_next = __ldg(P.row_ptr_src + r + 1);
    const double2 my_pv = __ldg(nodes2 + sel3(l, v[0], v[1], v[2]));
    const double2 my_po = __ldg(nodes2 + max(sel3(l, aop.x, aop.y, aop.z), 0));
    double2 pv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) pv[k] = grp_shfl2(my_pv, base, k);

    // ---- neighbours, sorted block columns -> slots (as p1_row, bound) ---------------------
    int kindv[3], lfv[3], fv[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      kindv[k] = (anb.w >> (4 * k)) & 3;
      lfv[k] = (anb.w >> (4 * k + 2)) & 3;
      fv[k] = k == 0 ? anb.x : (k == 1 ? anb.y : anb.z);
      if (kindv[k] != DGB_EDGE_INTERIOR) fv[k] = -1;
    }
    int slot_of[4], nb = 1;
    {
      const int cx[4] = {ee, fv[0], fv[1], fv[2]};
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int rk = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) rk += (j != i && cx[j] >= 0 && cx[j] < cx[i]) ? 1 : 0;
        slot_of[i] = rk;
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) nb += fv[k] >= 0 ? 1 : 0;
    }
    if (active) {
      if (l == 0) {
        o_row_ptr[r + 1] = rp_next;
        if (r == 0) o_row_ptr[0] = 0;
        o_col[rp + slot_of[0]] = ee;
      }
      const int myf = sel3(l, fv[0], fv[1], fv[2]);
      if (myf >= 0) o_col[rp + sel3(l, slot_of[1], slot_of[2], slot_of[3])] = myf;
    }
    const int rp_first = __shfl_sync(0xffffffffu, rp, 0);
    const int rp_last = __reduce_max_sync(0xffffffffu, active ? rp + nb : 0);
    double* srow = stw + (rp_first & 1);  // same 16-byte phase as val + rp_first * N2
    double* const myrow = srow + (rp - rp_first) * N2;

    // ---- own geometry (every lane of the group, as p1_row) -------------------------------
    const double B00 = FSUB(pv[1].x, pv[0].x), B01 = FSUB(pv[2].x, pv[0].x);
    const double B10 = FSUB(pv[1].y, pv[0].y), B11 = FSUB(pv[2].y, pv[0].y);
    const double det = FSUB(FMUL(B00, B11), FMUL(B01, B10));
    const double rdet = rcp_nr(det);
    const double G00 = B11 * rdet, G01 = -B10 * rdet;
    const double G10 = -B01 * rdet, G11 = B00 * rdet;
    const double eps = scalar_element(P.prob.diffusion, ee);

    // ---- RHS: this lane's share of the volume points -------------------------------------
    double F[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) F[i] = 0.0;
    source_points<NQV, false>(
        P.prob.source, ee, false,
        [&](int q, double& px, double& py) {
          px = fma(B01, tab[L::VY + q], fma(B00, tab[L::VX + q], pv[0].x));
          py = fma(B11, tab[L::VY + q], fma(B10, tab[L::VX + q], pv[0].y));
        },
        [&](int q, double f, double, double) {
          const double cq = (det * tab[L::VW + q]) * f;
#pragma unroll
          for (int i = 0; i < NL; ++i) F[i] = fma(cq, tab[L::PHI + q * NL + i], F[i]);
        },
        l, 3);

    // ---- diagonal row l: volume terms ------------------------------------------------------
    double acc[NL];
    {
      const double alpha = scalar_element(P.prob.linear_reaction, ee);
      const double de = det * eps;
      const double cD0 = de * (G00 * G00 + G10 * G10);
      const double cD1 = de * (G00 * G01 + G10 * G11);
      const double cD2 = de * (G01 * G01 + G11 * G11);
      const double cR = det * alpha;
      const double cC0 = det * (G00 * bf.p[0] + G10 * bf.p[1]);
      const double cC1 = det * (G01 * bf.p[0] + G11 * bf.p[1]);
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int k = l * NL + j;
        double x = cD0 * tab[L::S + k];
        x = fma(cD1, tab[L::S + N2 + k], x);
        x = fma(cD2, tab[L::S + 2 * N2 + k], x);
        x = fma(cR, tab[L::M + k], x);
        x = fma(cC0, tab[L::T + k], x);
        x = fma(cC1, tab[L::T + N2 + k], x);
        acc[j] = x;
      }
    }

    // ---- local edge l (this lane) ----------------------------------------------------------
    double w0 = 0.0, w1 = 0.0, cp = 0.0;
    {
      const int ia = l == 0 ? 1 : (l == 1 ? 2 : 0), ib = l == 0 ? 2 : (l == 1 ? 0 : 1);
      const int a = sel3(ia, v[0], v[1], v[2]), b = sel3(ib, v[0], v[1], v[2]);
      const double2 pa = sel3(ia, pv[0], pv[1], pv[2]), pb = sel3(ib, pv[0], pv[1], pv[2]);
      const int o = a < b ? 0 : 1;  // make_side orientation (assembly.cpp:125-126)
      const double2 A = o == 0 ? pa : pb;
      const double2 Bn = o == 0 ? pb : pa;
      const double dx = FSUB(Bn.x, A.x), dy = FSUB(Bn.y, A.y);
      const double rh = rsqrt_nr(fma(dx, dx, dy * dy));
      const double h = fma(dx, dx, dy * dy) * rh;
      const double tx = dx * rh, ty = dy * rh;
      const double nx = o == 0 ? ty : -ty, ny = o == 0 ? -tx : tx;
      const double ge0 = G00 * nx + G10 * ny, ge1 = G01 * nx + G11 * ny;
      const int kind = sel3(l, kindv[0], kindv[1], kindv[2]);
      const int lf = sel3(l, lfv[0], lfv[1], lfv[2]);
      const int f = sel3(l, fv[0], fv[1], fv[2]);
      if (kind == DGB_EDGE_INTERIOR) {
        // the neighbour in its vertex order rotated to (opposite, b, a) (p1_tables<.., true>)
        const Geo gf = element_geo_coords(my_po, pb, pa);
        double eps_e = eps;
        if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
          const double ef = __ldg(P.prob.diffusion.per_element + f);
          eps_e = ee < f ? 0.5 * (eps + ef) : 0.5 * (ef + eps);
        }
        const double bs = 0.5 * h * eps_e;
        w0 = bs * ge0;
        w1 = bs * ge1;
        const double cY0 = -bs * (gf.G00 * nx + gf.G10 * ny);
        const double cY1 = -bs * (gf.G01 * nx + gf.G11 * ny);
        const double cZ0 = -kappa * bs * ge0;
        const double cZ1 = -kappa * bs * ge1;
        const double sh = sigma_i * rh;
        const double fl = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
        const double up = fl < 0.0 ? FMUL(h, fl) : 0.0;
        cp = sh * (h * eps_e) - up;
        const double cxv = up - sh * (h * eps_e);
        // K_ef = sum_p phi^l_p (x) b1_p + a2_p (x) phi^lf_(n-1-p)  (as p1_row)
        const double* trm = tr + lf * (NQE * 3 * NL);
        double uY0 = cY0, uY1 = cY1;
        if (lf == 1) {
          uY0 = -cY0 - cY1;
          uY1 = cY0;
        } else if (lf == 2) {
          uY0 = cY1;
          uY1 = -cY0 - cY1;
        }
        double pm[NQE][NL], b1[NQE][NL];
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double cV = cxv * P.t.x[L::EW + p];
          const double* row = trm + (NQE - 1 - p) * 3 * NL;
#pragma unroll
          for (int j = 0; j < NL; ++j) {
            const double fr = row[j];
            const double g0 = P.t.x[L::EDW + ((NQE - 1 - p) * 2) * NL + j];
            const double g1 = P.t.x[L::EDW + ((NQE - 1 - p) * 2 + 1) * NL + j];
            pm[p][j] = fr;
            b1[p][j] = fma(cV, fr, fma(uY0, g0, uY1 * g1));
          }
        }
        double* blk = myrow + sel3(l, slot_of[1], slot_of[2], slot_of[3]) * N2;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          double rr[NL];
#pragma unroll
          for (int j = 0; j < NL; ++j) rr[j] = 0.0;
#pragma unroll
          for (int p = 0; p < NQE; ++p) {
            const double a2 = fma(cZ0, tab[L::EDW + ((l * NQE + p) * 2) * NL + i],
                                  cZ1 * tab[L::EDW + ((l * NQE + p) * 2 + 1) * NL + i]);
            const double ph = tab[L::EPHI + (l * NQE + p) * NL + i];
#pragma unroll
            for (int j = 0; j < NL; ++j) rr[j] = fma(ph, b1[p][j], fma(a2, pm[p][j], rr[j]));
          }
#pragma unroll
          for (int j = 0; j < NL; ++j) if (active) blk[i * NL + j] = rr[j];
        }
      } else {
        // boundary edge: diffusion (Dirichlet), inflow upwind, and the boundary RHS terms
        double fls[NQE], gb[NQE];
        bool inflow = false;
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double tq = o == 0 ? P.t.x[L::ET + p] : 1.0 - P.t.x[L::ET + p];
          const double px = FADD(A.x, FMUL(tq, dx));
          const double py = FADD(A.y, FMUL(tq, dy));
          fls[p] = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
          if (fls[p] < -1e-12 * fmax(1.0, hypot_dd(bf.p[0], bf.p[1]))) inflow = true;
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
            cG[p] = FMUL(FMUL(P.t.x[L::EW + p], h), gb[p]);
            cH[p] = 0.0;
          }
        } else {
          const double bs = h * eps;
          w0 = bs * ge0;
          w1 = bs * ge1;
          const double sh = sigma_b * rh;
          cp = sh * (h * eps) - ((inflow && fls[0] < 0.0) ? FMUL(h, fls[0]) : 0.0);
#pragma unroll
          for (int p = 0; p < NQE; ++p) {
            const double w = FMUL(P.t.x[L::EW + p], h);
            const double win = (inflow && fls[p] < 0.0) ? -FMUL(w, fls[p]) : 0.0;
            const double wgd = w * gb[p];
            cG[p] = wgd * (sh * eps) + win * gb[p];
            cH[p] = wgd * (kappa * eps);
          }
        }
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double h0 = cH[p] * ge0, h1 = cH[p] * ge1;
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            F[i] = fma(cG[p], tab[L::EPHI + (l * NQE + p) * NL + i],
                       fma(h0, tab[L::EDPHI + ((l * NQE + p) * 2) * NL + i],
                           fma(h1, tab[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], F[i])));
          }
        }
      }
    }

    // ---- face terms of the diagonal: edges 0, 1, 2 in order, into this lane's row l -------
#pragma unroll
    for (int ed = 0; ed < 3; ++ed) {
      const double e_w0 = grp_shfl(w0, base, ed), e_w1 = grp_shfl(w1, base, ed);
      const double e_cp = grp_shfl(cp, base, ed);
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int k = l * NL + j;
        acc[j] = fma(e_w0, tab[L::W + 2 * ed * N2 + k], fma(e_w1, tab[L::W + (2 * ed + 1) * N2 + k], acc[j]));
        acc[j] = fma(e_cp, tab[L::P + ed * N2 + k], acc[j]);
      }
    }
    if (active) {
#pragma unroll
      for (int j = 0; j < NL; ++j) myrow[slot_of[0] * N2 + l * NL + j] = acc[j];
    }

    // ---- RHS: the group's partial sums; lane l stores entry l (the warp's 30 entries are
    // contiguous, so the stores coalesce) --------------------------------------------------
    {
      double tot = 0.0;
#pragma unroll
      for (int i = 0; i < NL; ++i) {
        const double s0 = grp_shfl(F[i], base, 0), s1 = grp_shfl(F[i], base, 1);
        const double s2 = grp_shfl(F[i], base, 2);
        const double t = (s0 + s1) + s2;
        if (i == l) tot = t;
      }
      if (active) store_one(o_rhs + static_cast<long long>(r) * NL + l, tot, pol_out);
    }

    // ---- the warp's row range: 16-byte coalesced stores from the staging --------------------
    __syncwarp();
    {
      const int n = (rp_last - rp_first) * N2;
      double* dst = o_val + static_cast<long long>(rp_first) * N2;
      const int head = rp_first & 1;
      const double2* s2 = reinterpret_cast<const double2*>(srow + head);
      const int npair = (n - head) >> 1;
#pragma unroll 4
      for (int k = lane; k < npair; k += 32) {
        const double2 w = s2[k];
        store_pair(dst + head + 2 * k, w.x, w.y, pol_out);
      }
      if (lane == 1 && head && n > 0) store_one(dst, srow[0], pol_out);
      if (lane == 2 && n > 0 && ((n - head) & 1)) store_one(dst + n - 1, srow[n - 1], pol_out);
    }
    __syncwarp();
  }
}

}  // namespace v2
}  // namespace dgb
