// assemble_p1.cuh -- the block-row kernel for P1 with constant velocity (configs 1 and 4),
// included by dg_assembly.cu after assemble_v2.cuh.
//
// Same decomposition and the same arithmetic, in the same order, as the general
// element-per-thread kernel (assemble_v2.cuh), restructured for occupancy: every block
// slot is known before the edge loop (the neighbour ids come first), so each edge's
// neighbour block is computed and staged the moment its coefficients exist, and its face
// terms go straight into the diagonal block held in registers.  No per-edge coefficient
// stash is needed (6 KB of shared memory per warp on the general path), which lifts the P1
// kernel from 12 to 16 resident warps per SM.  The staged rows leave as one bulk copy per
// warp (the warp's row range is contiguous in the BSR).
#pragma once

// Persistent kernel's copy-out: 1 = one bulk asynchronous copy per chunk whose read of the
// staging is awaited a volume phase later; 0 = the warp copies its range itself.
#ifndef DGB_P1_BULK_OUT
#define DGB_P1_BULK_OUT 1
#endif
// Where the persistent kernel waits for the previous chunk's bulk copy to have read the staging:
// before the edge loop, or (p1_late_stage) only before the chunk's first staging store, edge 0's
// neighbour block being computed into registers first.  Measured same-box on the specialised
// kernels: the late wait is 6% faster with the sine-product source (config-1 batch 0.138 ->
// 0.129 ms) and 4% slower with the Gaussian (config 4 0.660 -> 0.689 ms; keeping the blocks in
// registers across the branch alone costs 1.4% there), so it is chosen per source family;
// -DDGB_P1_WAIT_IN_EDGE0=0/1 forces it for A/B runs.
#ifndef DGB_P1_WAIT_IN_EDGE0
#define DGB_P1_WAIT_IN_EDGE0 -1
#endif
// The volume RHS term (the source at the volume points) may run after the copy-out has been
// issued instead of before the diagonal block (p1_row's kSrcLate).  Measured same-box on the
// specialised kernels: late is 8% faster with the sine-product source (config-1 batch 0.151 ->
// 0.140 ms) and 3% slower with the Gaussian (config 4 0.664 -> 0.686 ms), so it is chosen per
// source family; -DDGB_P1_SRC_LATE=0/1 forces it for A/B runs.
#ifndef DGB_P1_SRC_LATE
#define DGB_P1_SRC_LATE -1
#endif

namespace dgb {
namespace v2 {

constexpr bool p1_late_stage(int src) {
  return DGB_P1_WAIT_IN_EDGE0 < 0 ? src == SRC_SIN_SIN : DGB_P1_WAIT_IN_EDGE0 != 0;
}

template <int NQV, int NQE>
struct SmemP1 {
  static constexpr int NL = 3, N2 = 9;
  static constexpr int kStage = (32 * 4 * N2 + 2 + 1) & ~1;  // the warp's row range
  static constexpr int kRhs = (32 * NL + 1) & ~1;
  static constexpr int kWarp = kStage + kRhs;
  static constexpr int kTr = (3 * NQE * 3 * NL + 1) & ~1;
};

// Per-CTA trace table tr[l][p][c][j]: phi, w d0 phi, w d1 phi of local edge l's points.
// ROTATED (bound mesh): the gradient pair of edge lf is expressed in the neighbour's vertex
// order rotated to start at its vertex opposite the shared edge, (q_lf, q_lf+1, q_lf+2), so the
// block-row kernel builds the neighbour's geometry from (opposite, b, a) without selecting on
// lf.  With x = q_0 + xi e1 + eta e2, the rotated reference coordinates satisfy
// grad' phi = M_lf grad phi, M_0 = I, M_1 = [[-1, 1], [-1, 0]], M_2 = [[0, -1], [1, -1]], and
// G_f^T n . g = G'^T n . (M_lf g): the neighbour terms are unchanged.
template <int NQV, int NQE, bool ROTATED = false>
__device__ __forceinline__ void p1_tables(const Params2<3, NQV, NQE, false, true>& P, double* tr) {
  constexpr int NL = 3;
  using L = Lay<NL, NQV, NQE, false, true>;
  for (int i = threadIdx.x; i < 3 * NQE * 3 * NL; i += blockDim.x) {
    const int j = i % NL, c = (i / NL) % 3, p = (i / (3 * NL)) % NQE, l = i / (3 * NL * NQE);
    const double g0 = P.t.x[L::EDW + ((l * NQE + p) * 2) * NL + j];
    const double g1 = P.t.x[L::EDW + ((l * NQE + p) * 2 + 1) * NL + j];
    double v;
    if (c == 0) {
      v = P.t.x[L::EPHI + (l * NQE + p) * NL + j];
    } else if (!ROTATED || l == 0) {
      v = c == 1 ? g0 : g1;
    } else if (l == 1) {
      v = c == 1 ? g1 - g0 : -g0;
    } else {
      v = c == 1 ? -g1 : g0 - g1;
    }
    tr[i] = v;
  }
}

// make_side / edge_geometry of local edge l (assembly.cpp:125-126, mesh.cpp:232-257) from the
// element's vertices: direction in the sorted-pair orientation o (0: a < b), length and its
// reciprocal from one rsqrt, unit outward normal.  Shared by the block-row kernel and the
// bind-time geometry kernel (dg_assembly.cu), so a bound record holds the kernel's own values.
// The outward normal does not depend on the orientation o: reversing the edge negates (dx, dy)
// exactly, and make_side's sign flip negates the rotated tangent back.  So the direction is
// taken from vertex l+1 to vertex l+2 (o = 0); only a boundary edge's quadrature points need the
// oriented start vertex and direction (p1_edge_oriented).
struct EdgeFrame {
  double dx, dy, rh, nx, ny;
};
__device__ __forceinline__ void p1_edge_dir(const double2 (&pv)[3], int l, double& dx, double& dy) {
  dx = FSUB(pv[(l + 2) % 3].x, pv[(l + 1) % 3].x);
  dy = FSUB(pv[(l + 2) % 3].y, pv[(l + 1) % 3].y);
}
__device__ __forceinline__ void p1_edge_normal(double dx, double dy, double rh, double& nx, double& ny) {
  nx = FMUL(dy, rh);
  ny = -FMUL(dx, rh);
}
__device__ __forceinline__ EdgeFrame p1_edge_frame(const double2 (&pv)[3], int l) {
  EdgeFrame f;
  p1_edge_dir(pv, l, f.dx, f.dy);
  f.rh = rsqrt_nr(fma(f.dx, f.dx, FMUL(f.dy, f.dy)));
  p1_edge_normal(f.dx, f.dy, f.rh, f.nx, f.ny);
  return f;
}
// G_f^T n: the neighbour's inverse-transposed Jacobian, in its vertex order rotated to
// (opposite, b, a), applied to this element's outward normal.
__device__ __forceinline__ double2 p1_neighbour_normal(double2 opp, double2 pb, double2 pa, double nx, double ny) {
  const Geo gf = element_geo_coords(opp, pb, pa);
  return make_double2(fma(gf.G00, nx, FMUL(gf.G10, ny)), fma(gf.G01, nx, FMUL(gf.G11, ny)));
}

// The element's extent for source_points: the largest squared distance from a centre to a vertex.
struct VertexExtent {
  static constexpr bool kKnown = true;
  const double2 (&pv)[3];
  __device__ __forceinline__ double operator()(double cx, double cy) const {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double dx = pv[k].x - cx, dy = pv[k].y - cy;
      m = fmax(m, fma(dx, dx, dy * dy));
    }
    return m;
  }
};

// The block row of one element (one lane), after its gathers: neighbours, slots, block columns,
// geometry, volume and face terms, the neighbour blocks staged in the warp's row range, and the
// warp's RHS slice and row range sent by bulk copies.  `wait_stage` (persistent kernel): the
// staging is reused by the next chunk, so the warp copies its row range out itself.
// `mid()` runs between the volume terms and the edge loop (the persistent kernel issues the next
// chunk's node gathers there).
// SRC: the source family the kernel is specialised for (source_points' ONLY).
// GEO (persistent kernel, bound geometry record): po[l] holds the neighbour's G_f^T n (and, in a
// DGB_GEO_RECIPROCALS build, gx the reciprocals (1 / det, 1 / h_0), (1 / h_1, 1 / h_2)); slots,
// orientations and the block count come from the adjacency word.
template <int NQV, int NQE, bool BOUND, bool GEO, int SRC, class MID, class STG>
__device__ __forceinline__ void p1_row(const Params2<3, NQV, NQE, false, true>& P, const double* tr,
                                       int mset, double* stw, double* srhs, int lane, int e_first,
                                       int ee, bool active, const int (&v)[3], int4 anb, int4 aop,
                                       int rp, int rp_next, const double2 (&pv)[3],
                                       const double2 (&po)[3], const double2 (&gx)[2], bool wait_stage,
                                       MID&& mid, STG&& before_stage) {
  constexpr int NL = 3, N2 = 9;
  using L = Lay<NL, NQV, NQE, false, true>;
  using SM = SmemP1<NQV, NQE>;
  const double kappa = P.bt[mset].kappa, sigma_i = P.bt[mset].sigma_i, sigma_b = P.bt[mset].sigma_b;
  int32_t* const o_row_ptr = P.bt[mset].row_ptr;
  int32_t* const o_col = P.bt[mset].col;
  double* const o_val = P.bt[mset].val;
  double* const o_rhs = P.bt[mset].rhs;
  const dgb_vector_field& bf = P.prob.advection;
  constexpr bool bound = BOUND;
  // neighbours first: kind, neighbour, its local edge (and, unbound, its vertices)
  int kindv[3], lfv[3], fv[3], edgev[3], vfv[3][3];
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int a = v[(l + 1) % 3], b = v[(l + 2) % 3];
    edgev[l] = -1;
    lfv[l] = 0;
    fv[l] = -1;
    if constexpr (bound) {
      kindv[l] = (anb.w >> (4 * l)) & 3;
      lfv[l] = (anb.w >> (4 * l + 2)) & 3;
      fv[l] = l == 0 ? anb.x : (l == 1 ? anb.y : anb.z);
    } else {
      edgev[l] = __ldg(P.element_edges + 3 * ee + l);
      kindv[l] = __ldg(P.edge_kind + edgev[l]);
      if (kindv[l] == DGB_EDGE_INTERIOR) {
        const int2 lr = __ldg(reinterpret_cast<const int2*>(P.edge_elements) + edgev[l]);
        fv[l] = lr.x == ee ? lr.y : lr.x;
#pragma unroll
        for (int k = 0; k < 3; ++k) vfv[l][k] = __ldg(P.elements + 3 * fv[l] + k);
#pragma unroll
        for (int k = 0; k < 3; ++k) if (vfv[l][k] != a && vfv[l][k] != b) lfv[l] = k;
      }
    }
    if (kindv[l] != DGB_EDGE_INTERIOR) fv[l] = -1;
  }
  // sorted block columns -> slots (rank among the row's distinct columns)
  int slot_of[4], nb = 1;
  if constexpr (GEO) {
#pragma unroll
    for (int i = 0; i < 4; ++i) slot_of[i] = (anb.w >> (12 + 2 * i)) & 3;
    nb = (anb.w >> 23) & 7;
  } else {
    const int cx[4] = {ee, fv[0], fv[1], fv[2]};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) r += (j != i && cx[j] >= 0 && cx[j] < cx[i]) ? 1 : 0;
      slot_of[i] = r;
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) nb += fv[l] >= 0 ? 1 : 0;
  }
  if (P.row_ptr_src) {
    if (active) {
      o_row_ptr[ee - P.row_begin + 1] = rp_next;
      if (ee == P.row_begin) o_row_ptr[0] = 0;
    }
  } else {
    rp = o_row_ptr[ee - P.row_begin];
  }
  if (active) {
    o_col[rp + slot_of[0]] = ee;
#pragma unroll
    for (int l = 0; l < 3; ++l) if (fv[l] >= 0) o_col[rp + slot_of[1 + l]] = fv[l];
  }
  const int rp_first = __shfl_sync(0xffffffffu, rp, 0);
  const int rp_last = __reduce_max_sync(0xffffffffu, active ? rp + nb : 0);
  double* srow = stw + (rp_first & 1);  // same 16-byte phase as val + rp_first * N2
  double* const myrow = srow + (rp - rp_first) * N2;

  // ---- own geometry, coefficients of the volume terms ------------------------------------------
  const double B00 = FSUB(pv[1].x, pv[0].x), B01 = FSUB(pv[2].x, pv[0].x);
  const double B10 = FSUB(pv[1].y, pv[0].y), B11 = FSUB(pv[2].y, pv[0].y);
  const double det = FSUB(FMUL(B00, B11), FMUL(B01, B10));
  const double rdet = (GEO && kGeoRows == 8) ? gx[0].x : rcp_nr(det);
  const double G00 = B11 * rdet, G01 = -B10 * rdet;
  const double G10 = -B01 * rdet, G11 = B00 * rdet;
  const double eps = scalar_element(P.prob.diffusion, ee);
  if (DGB_ABLATE(32)) {  // (profiling ablation: gathers and own geometry only)
    if (active) o_rhs[ee - P.row_begin] = det + po[0].x + po[1].x + po[2].x;
    return;
  }

  // RHS volume term.  kSrcLate: evaluated after the row range's copy-out has been issued
  // (the source needs no staging, so the copy engine drains the staging meanwhile); the boundary
  // terms of the edge loop then come first in F's sums (a boundary element's F differs in the
  // last bit from the early order).
  double F[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) F[i] = 0.0;
  auto volume_rhs = [&] {
    source_points<NQV, false, SRC>(
        P.prob.source, ee, DGB_ABLATE(2),
        [&](int q, double& px, double& py) {
          // volume points only evaluate coefficients (no term selection): fused
          px = fma(B01, P.t.x[L::VY + q], fma(B00, P.t.x[L::VX + q], pv[0].x));
          py = fma(B11, P.t.x[L::VY + q], fma(B10, P.t.x[L::VX + q], pv[0].y));
        },
        [&](int q, double f, double, double) {
          const double c = (det * P.t.x[L::VW + q]) * f;
#pragma unroll
          for (int i = 0; i < NL; ++i) F[i] = fma(c, P.t.x[L::PHI + q * NL + i], F[i]);
        },
        0, 1, VertexExtent{pv});
  };
  constexpr bool kSrcLate = DGB_P1_SRC_LATE < 0 ? SRC == SRC_SIN_SIN : DGB_P1_SRC_LATE != 0;
  if constexpr (!kSrcLate) volume_rhs();

  // diagonal block: volume terms (registers)
  double acc[N2];
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
    for (int k = 0; k < N2; ++k) {
      double x = cD0 * P.t.x[L::S + k];
      x = fma(cD1, P.t.x[L::S + N2 + k], x);
      x = fma(cD2, P.t.x[L::S + 2 * N2 + k], x);
      x = fma(cR, P.t.x[L::M + k], x);
      x = fma(cC0, P.t.x[L::T + k], x);
      x = fma(cC1, P.t.x[L::T + N2 + k], x);
      acc[k] = x;
    }
  }

  mid();
  // ---- edges: face terms into the diagonal, neighbour blocks staged at once --------------------
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    // edge_geometry (mesh.cpp:232-257): length and its reciprocal from one rsqrt, outward normal
    double dx, dy, nx, ny;
    p1_edge_dir(pv, l, dx, dy);
    const double r2 = fma(dx, dx, FMUL(dy, dy));
    const double rh = (GEO && kGeoRows == 8) ? (l == 0 ? gx[0].y : (l == 1 ? gx[1].x : gx[1].y)) : rsqrt_nr(r2);
    const double h = r2 * rh;
    p1_edge_normal(dx, dy, rh, nx, ny);
    const double ge0 = G00 * nx + G10 * ny, ge1 = G01 * nx + G11 * ny;
    const int kind = kindv[l], lf = lfv[l], f = fv[l];
    double w0 = 0.0, w1 = 0.0, cp = 0.0;
    double rr[N2];  // (p1_late_stage) the neighbour block of an interior edge, staged after the branch
    bool have_block = false;
    if (kind == DGB_EDGE_INTERIOR) {
      double2 gn;  // G_f^T n of the neighbour
      if constexpr (GEO) {
        gn = po[l];
      } else if constexpr (bound) {
        // the neighbour in its vertex order rotated to (opposite, b, a): the trace table's
        // gradients are rotated to match (p1_tables<.., true>)
        gn = p1_neighbour_normal(po[l], pv[(l + 2) % 3], pv[(l + 1) % 3], nx, ny);
      } else {
        const Geo gf = element_geo_fast(P.nodes, vfv[l]);
        gn = make_double2(fma(gf.G00, nx, FMUL(gf.G10, ny)), fma(gf.G01, nx, FMUL(gf.G11, ny)));
      }
      double eps_e = eps;
      if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
        const double ef = __ldg(P.prob.diffusion.per_element + f);
        eps_e = ee < f ? 0.5 * (eps + ef) : 0.5 * (ef + eps);
      }
      const double base = 0.5 * h * eps_e;
      w0 = base * ge0;
      w1 = base * ge1;
      const double cY0 = -base * gn.x;
      const double cY1 = -base * gn.y;
      const double cZ0 = -kappa * base * ge0;
      const double cZ1 = -kappa * base * ge1;
      const double sh = sigma_i * rh;
      const double fl = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
      const double up = fl < 0.0 ? FMUL(h, fl) : 0.0;
      cp = sh * (h * eps_e) - up;
      const double cx = up - sh * (h * eps_e);
      // K_ef = sum_p phi^l_p (x) b1_p + a2_p (x) phi^lf_(n-1-p)
      if (!(DGB_ABLATE(4))) {  // (profiling ablation: skip the neighbour block)
      const double* trm = tr + lf * (NQE * 3 * NL);
      // P1: the reference gradients are constant, so the neighbour's w d phi at its points are
      // the same for every edge: read them from the constant bank (edge 0) with the
      // coefficients rotated back to the neighbour's own vertex order, uY = M_lf^T cY
      // (p1_tables), instead of loading the rotated gradients per lf
      double uY0 = cY0, uY1 = cY1;
      if constexpr (bound) {
        if (lf == 1) {
          uY0 = -cY0 - cY1;
          uY1 = cY0;
        } else if (lf == 2) {
          uY0 = cY1;
          uY1 = -cY0 - cY1;
        }
      }
      double pm[NQE][NL], b1[NQE][NL];
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double cV = cx * P.t.x[L::EW + p];
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
      have_block = true;
      double* blk = myrow + slot_of[1 + l] * N2;
#pragma unroll
      for (int i = 0; i < NL; ++i) {
        double r[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) r[j] = 0.0;
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double a2 = fma(cZ0, P.t.x[L::EDW + ((l * NQE + p) * 2) * NL + i],
                                cZ1 * P.t.x[L::EDW + ((l * NQE + p) * 2 + 1) * NL + i]);
          const double ph = P.t.x[L::EPHI + (l * NQE + p) * NL + i];
#pragma unroll
          for (int j = 0; j < NL; ++j) r[j] = fma(ph, b1[p][j], fma(a2, pm[p][j], r[j]));
        }
#pragma unroll
        for (int j = 0; j < NL; ++j) {
          if constexpr (p1_late_stage(SRC)) rr[i * NL + j] = r[j];
          else if (active) blk[i * NL + j] = r[j];
        }
      }
      }
    } else {
      // boundary edge: diffusion (Dirichlet), inflow upwind, and the boundary RHS terms
      const int o = GEO ? (anb.w >> (20 + l)) & 1 : (v[(l + 1) % 3] < v[(l + 2) % 3] ? 0 : 1);
      const double2 A = o == 0 ? pv[(l + 1) % 3] : pv[(l + 2) % 3];
      const dgb_scalar_field& bfld = kind == DGB_EDGE_NEUMANN ? P.prob.neumann : P.prob.dirichlet;
      const bool bfast = boundary_fast_ok(bfld, pv[(l + 1) % 3], pv[(l + 2) % 3]);
      double fls[NQE], gb[NQE];
      bool inflow = false;
      const double inflow_tol = -1e-12 * fmax(1.0, hypot_dd(bf.p[0], bf.p[1]));
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        // make_side orientation (assembly.cpp:125-126): the points run from the lower vertex id
        const double tq = o == 0 ? P.t.x[L::ET + p] : 1.0 - P.t.x[L::ET + p];
        const double px = FADD(A.x, FMUL(tq, o == 0 ? dx : -dx));
        const double py = FADD(A.y, FMUL(tq, o == 0 ? dy : -dy));
        fls[p] = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
        if (fls[p] < inflow_tol) inflow = true;
        gb[p] = scalar_point_fast(bfld, px, py, bfast);
      }
      double cG[NQE], cH[NQE];
      if (kind == DGB_EDGE_NEUMANN) {
        const int edge = bound ? __ldg(P.element_edges + 3 * ee + l) : edgev[l];
        if (inflow && !P.drop_neumann && active) {
          atomicMax(P.err_edge, (P.epoch << 32) | (0xFFFFFFFFull - static_cast<unsigned>(edge)));
        }
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          cG[p] = FMUL(FMUL(P.t.x[L::EW + p], h), gb[p]);
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
          cH[p] = wgd * (kappa * eps);
        }
      }
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double h0 = cH[p] * ge0, h1 = cH[p] * ge1;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          F[i] = fma(cG[p], P.t.x[L::EPHI + (l * NQE + p) * NL + i],
                     fma(h0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i],
                         fma(h1, P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], F[i])));
        }
      }
    }
    // (convergent again) the first staging store of the chunk: the persistent kernel waits here
    // for the previous chunk's bulk copy to have read the staging
    if constexpr (p1_late_stage(SRC)) {
      if (l == 0) before_stage();
      if (have_block && active) {
        double* blk = myrow + slot_of[1 + l] * N2;
#pragma unroll
        for (int k = 0; k < N2; ++k) blk[k] = rr[k];
      }
    }
    // face terms of the diagonal block (the general kernel's order: W then P, per edge)
#pragma unroll
    for (int k = 0; k < N2; ++k) {
      acc[k] = fma(w0, P.t.x[L::W + 2 * l * N2 + k], fma(w1, P.t.x[L::W + (2 * l + 1) * N2 + k], acc[k]));
      acc[k] = fma(cp, P.t.x[L::P + l * N2 + k], acc[k]);
    }
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < N2; ++k) myrow[slot_of[0] * N2 + k] = acc[k];
  }

  // ---- the warp's row range: one bulk copy, unaligned head / tail by hand ----------------------------
  if (wait_stage && DGB_P1_BULK_OUT == 0) {
    // the warp copies its range itself (16-byte coalesced stores)
    __syncwarp();
    const int n = (rp_last - rp_first) * N2;
    double* dst = o_val + static_cast<long long>(rp_first) * N2;
    const int head = rp_first & 1;
    const unsigned long long pol = output_policy(P.evict_first);
    // srow + head is 16-byte aligned (srow has val's 16-byte phase): pairs load as one LDS.128
    const double2* s2 = reinterpret_cast<const double2*>(srow + head);
    const int npair = (n - head) >> 1;
#pragma unroll 4
    for (int k = lane; k < npair; k += 32) {
      const double2 w = s2[k];
      store_pair(dst + head + 2 * k, w.x, w.y, pol);
    }
    if (lane == 1 && head && n > 0) dst[0] = srow[0];
    if (lane == 2 && n > 0 && ((n - head) & 1)) dst[n - 1] = srow[n - 1];
    __syncwarp();
  } else {
    // (persistent kernel: the staging is reused by the next chunk, which waits for this copy's
    // read of it after its own volume terms -- the `mid` hook)
    fence_smem_to_async();  // every writer: its staged blocks -> the async (TMA) proxy
    __syncwarp();
    const int n = (rp_last - rp_first) * N2;
    double* dst = o_val + static_cast<long long>(rp_first) * N2;
    const int head = rp_first & 1;
    const int body = (n - head) & ~1;
    if (lane == 0 && body > 0 && !(DGB_ABLATE(1))) bulk_store(dst + head, srow + head, body * sizeof(double), P.evict_first);
    // (a warp past the last row has no range: n <= 0, nothing to write)
    if (lane == 1 && head && n > 0) dst[0] = srow[0];
    if (lane == 2 && n > 0 && head + body < n) dst[n - 1] = srow[n - 1];
  }
  if constexpr (kSrcLate) volume_rhs();

  // ---- RHS: direct stores (srhs == nullptr), or the warp's contiguous slice in one bulk copy --------
  if (srhs == nullptr) {
    double* dst = o_rhs + static_cast<long long>(e_first + lane) * NL;
#pragma unroll
    for (int i = 0; i < NL; ++i) if (active) dst[i] = F[i];
  } else {
#pragma unroll
    for (int i = 0; i < NL; ++i) srhs[lane * NL + i] = F[i];
    fence_smem_to_async();  // every writer: its shared-memory stores -> the async (TMA) proxy
    __syncwarp();
    const int n_here = min(32, P.row_end - P.row_begin - e_first);
    double* dst = o_rhs + static_cast<long long>(e_first) * NL;
    const int bulk = (n_here * NL) & ~1;
    if (lane == 0 && bulk > 0) bulk_store(dst, srhs, bulk * sizeof(double), P.evict_first);
    for (int idx = bulk + lane; idx < n_here * NL; idx += 32) dst[idx] = srhs[idx];
  }
}

template <int NQV, int NQE, int THREADS, int MINB, bool BOUND>
__global__ void __launch_bounds__(THREADS, MINB) assemble_p1_kernel(
    const __grid_constant__ Params2<3, NQV, NQE, false, true> P) {
  constexpr int NL = 3;
  using L = Lay<NL, NQV, NQE, false, true>;
  using SM = SmemP1<NQV, NQE>;
  extern __shared__ double smem[];
  double* tr = smem;
  p1_tables<NQV, NQE, BOUND>(P, tr);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mset = blockIdx.y;
  double* const o_rhs = P.bt[mset].rhs;
  double* stw = smem + SM::kTr + warp * SM::kWarp;
  double* srhs = stw + SM::kStage;

  const int e = P.row_begin + blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = e < P.row_end;
  const int ee = active ? e : P.row_end - 1;
  constexpr bool bound = BOUND;  // bound adjacency record (dgb_plan_bind_mesh) or not

  // ---- gathers up front ------------------------------------------------------------------------
  const bool hints = BOUND && P.load_hints;
  const unsigned long long pol_g = evict_last_policy(), pol_s = evict_first_policy();
  int v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = hints ? ld_stream(P.elements + 3 * ee + k, pol_s) : __ldg(P.elements + 3 * ee + k);
  int4 anb = make_int4(0, 0, 0, 0), aop = make_int4(0, 0, 0, 0);
  int rp = 0, rp_next = 0;
  if constexpr (bound) {
    anb = hints ? ld_stream(P.adj_nb + (ee - P.row_begin), pol_s) : __ldg(P.adj_nb + (ee - P.row_begin));
    aop = hints ? ld_stream(P.adj_op + (ee - P.row_begin), pol_s) : __ldg(P.adj_op + (ee - P.row_begin));
  }
  if (P.row_ptr_src) {
    rp = __ldg(P.row_ptr_src + (ee - P.row_begin));
    rp_next = __ldg(P.row_ptr_src + (ee - P.row_begin + 1));
  }
  if (DGB_ABLATE(64)) {  // (profiling ablation: index records only)
    if (active) o_rhs[ee - P.row_begin] = double(v[0] + v[1] + v[2] + anb.x + anb.w + aop.x + aop.z + rp + rp_next);
    return;
  }
  const double2* nodes2 = reinterpret_cast<const double2*>(P.nodes);
  double2 pv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pv[k] = hints ? ld_hint(nodes2 + v[k], pol_g) : __ldg(nodes2 + v[k]);
  double2 po[3];
  if constexpr (bound) {
    po[0] = hints ? ld_hint(nodes2 + max(aop.x, 0), pol_g) : __ldg(nodes2 + max(aop.x, 0));
    po[1] = hints ? ld_hint(nodes2 + max(aop.y, 0), pol_g) : __ldg(nodes2 + max(aop.y, 0));
    po[2] = hints ? ld_hint(nodes2 + max(aop.z, 0), pol_g) : __ldg(nodes2 + max(aop.z, 0));
  }
  const double2 gx[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
  p1_row<NQV, NQE, BOUND, false, SRC_ANY>(P, tr, mset, stw, DGB_ABLATE(128) ? srhs : nullptr, lane,
                                 blockIdx.x * blockDim.x + warp * 32, ee, active, v, anb, aop, rp, rp_next, pv,
                                 po, gx, false, [] {}, [] {});
  if (lane == 0) bulk_wait_all();
}



// ---- persistent, software-pipelined P1 kernel (bound mesh) ------------------------------------
//
// The one-shot kernel above spends its warps' time in a serial chain per 32-element chunk:
// index records (one DRAM round trip), then the node coordinates they name (a second, random,
// round trip), then the arithmetic and the stores.  Measured on config 4 (profiles/NOTES.md),
// the gathers alone take 0.35-0.40 ms of the 1.17 ms kernel, and 16 warps per SM do not hide
// them.  Here every warp walks its own sequence of chunks with both loads in flight one chunk
// ahead, landing in shared memory through asynchronous copies (LDGSTS: no registers held while
// they are in flight):
//
//   chunk j:  wait (its records and nodes have landed); read them into registers
//             issue the record copies of chunk j+1
//             source and volume terms of chunk j
//             wait (records of j+1); issue the node copies of chunk j+1
//             edge terms, neighbour blocks and stores of chunk j
//
// Each lane reads only what it copied itself, so the per-thread cp.async groups are the only
// synchronisation on the input side.
template <int NQV, int NQE, int WARPS, bool GEO>
struct SmemP1Pipe {
  using SM = SmemP1<NQV, NQE>;
  static constexpr int kNb = ChunkRec::kNb, kOp = ChunkRec::kOp, kV = ChunkRec::kV,
                       kRp = ChunkRec::kRp, kRpn = ChunkRec::kRpn, kIdxInts = ChunkRec::kIdxInts;
  static constexpr int kIdx = ChunkRec::kIdx, kNode = GEO ? ChunkRec::kNode2 : ChunkRec::kNode;
  static constexpr int kWarp = kIdx + kNode + SM::kStage;  // RHS stored directly
  static constexpr size_t kBytes = sizeof(double) * (size_t(SM::kTr) + size_t(WARPS) * kWarp);
};

// GEO: the chunk's geometry record bound by dgb_plan_bind_mesh (geometry_kernel) replaces the
// node gathers.  Chunks are dealt round-robin: measured (tools/p1_diag.py) the SMs finish within
// 0.5% of one another, and handing chunks out through an atomic ticket counter cost 6% (the
// ticket's round trip under the write stream), so the static order stays.
template <int NQV, int NQE, int WARPS, bool GEO, int SRC>
__global__ void __launch_bounds__(WARPS * 32, 1) assemble_p1_pipe_kernel(
    const __grid_constant__ Params2<3, NQV, NQE, false, true> P) {
  constexpr int NL = 3;
  using L = Lay<NL, NQV, NQE, false, true>;
  using SM = SmemP1<NQV, NQE>;
  using PS = SmemP1Pipe<NQV, NQE, WARPS, GEO>;
  extern __shared__ double smem[];
  double* tr = smem;
  p1_tables<NQV, NQE, true>(P, tr);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int mset = blockIdx.y;
  double* wbase = smem + SM::kTr + warp * PS::kWarp;
  int* idx = reinterpret_cast<int*>(wbase);                     // one chunk's records
  double2* nod = reinterpret_cast<double2*>(wbase + PS::kIdx);  // one chunk's nodes / geometry
  double* stw = wbase + PS::kIdx + PS::kNode;
  double* srhs = nullptr;  // RHS stored directly (shared memory for 16 warps)
#ifdef DGB_TUNING
  unsigned long long t_begin = 0, c_begin = 0;
  int n_done = 0;
  if (P.diag) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_begin));
    c_begin = clock64();
  }
#endif

  const int n_rows = P.row_end - P.row_begin;
  const int n_chunks = (n_rows + 31) >> 5;
  // chunks go warp-major across the CTAs (warp w of CTA b starts at chunk b + w gridDim.x): a
  // small mesh then spreads over the SMs, one busy warp each, instead of filling a few CTAs
  const int gw = warp * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x), n_gw = gridDim.x * WARPS;
  const double2* nodes2 = reinterpret_cast<const double2*>(P.nodes);

  auto issue_records = [&](int c) {
    const int e = P.row_begin + c * 32 + lane;
    const int r = min(e, P.row_end - 1) - P.row_begin;
    cp_async16(idx + PS::kNb + 4 * lane, P.adj_nb + r);
    if constexpr (GEO) {
      // the chunk's geometry record: kGeoRows coalesced 16-byte copies per lane, in flight
      // together with the index records (no dependent gather)
      const double2* g = P.geo + static_cast<size_t>(c) * (kGeoRows * 32) + lane;
#pragma unroll
      for (int k = 0; k < kGeoRows; ++k) cp_async16(nod + k * 32 + lane, g + k * 32);
    } else {
      cp_async16(idx + PS::kOp + 4 * lane, P.adj_op + r);
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async4(idx + PS::kV + 3 * lane + k, P.elements + 3 * (P.row_begin + r) + k);
    }
    cp_async4(idx + PS::kRp + lane, P.row_ptr_src + r);
    cp_async4(idx + PS::kRpn + lane, P.row_ptr_src + r + 1);
    cp_async_commit();
  };
  const bool hints = P.load_hints;
  const unsigned long long pol_g = evict_last_policy();
  auto issue_nodes = [&]() {  // from the landed records
    if (hints) {  // L2 policy bit 2: node gathers evict-last (they are gathered again)
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async16_hint(nod + k * 32 + lane, nodes2 + idx[PS::kV + 3 * lane + k], pol_g);
#pragma unroll
      for (int k = 0; k < 3; ++k)
        cp_async16_hint(nod + (3 + k) * 32 + lane, nodes2 + max(idx[PS::kOp + 4 * lane + k], 0), pol_g);
    } else {
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async16(nod + k * 32 + lane, nodes2 + idx[PS::kV + 3 * lane + k]);
#pragma unroll
      for (int k = 0; k < 3; ++k) cp_async16(nod + (3 + k) * 32 + lane, nodes2 + max(idx[PS::kOp + 4 * lane + k], 0));
    }
    cp_async_commit();
  };
  int c_cur = gw, c_next = gw + n_gw;
  if (c_cur < n_chunks) {
    issue_records(c_cur);
    if constexpr (!GEO) {
      cp_async_wait_all();
      issue_nodes();
    }
  }
#pragma unroll 1
  while (c_cur < n_chunks) {
    cp_async_wait_all();  // this chunk's records and nodes have landed
    // everything of the chunk into registers; the buffers take the next chunk from here on
    int v[3] = {0, 0, 0};
    if constexpr (!GEO) {
#pragma unroll
      for (int k = 0; k < 3; ++k) v[k] = idx[PS::kV + 3 * lane + k];
    }
    const int4 anb = *reinterpret_cast<const int4*>(idx + PS::kNb + 4 * lane);
    const int4 aop = GEO ? make_int4(0, 0, 0, 0) : *reinterpret_cast<const int4*>(idx + PS::kOp + 4 * lane);
    const int rp = idx[PS::kRp + lane], rp_next = idx[PS::kRpn + lane];
    const double2 pv[3] = {nod[lane], nod[32 + lane], nod[64 + lane]};
    const double2 po[3] = {nod[96 + lane], nod[128 + lane], nod[160 + lane]};
    double2 gx[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
    if constexpr (GEO) {
      if constexpr (kGeoRows == 8) {
        gx[0] = nod[192 + lane];
        gx[1] = nod[224 + lane];
      }
    }
    const bool more = c_next < n_chunks;
    if (more) issue_records(c_next);
    const int e_first = c_cur * 32;
    const int e = P.row_begin + e_first + lane;
    const bool active = e < P.row_end;
    const int ee = active ? e : P.row_end - 1;
    p1_row<NQV, NQE, true, GEO, SRC>(P, tr, mset, stw, srhs, lane, e_first, ee, active, v, anb, aop, rp,
                                rp_next, pv, po, gx, true, [&] {
                                  if constexpr (DGB_P1_BULK_OUT != 0 && !p1_late_stage(SRC)) {
                                    // the previous chunk's row range has left the staging (its bulk
                                    // copy was issued a whole volume phase ago)
                                    if (lane == 0) bulk_wait_read();
                                    __syncwarp();
                                  }
                                  if constexpr (!GEO) {
                                    if (more) {
                                      cp_async_wait_all();  // the next chunk's records
                                      issue_nodes();
                                    }
                                  }
                                }, [&] {
                                  if constexpr (DGB_P1_BULK_OUT != 0 && p1_late_stage(SRC)) {
                                    if (lane == 0) bulk_wait_read();
                                    __syncwarp();
                                  }
                                });
    c_cur = c_next;
    c_next += n_gw;
#ifdef DGB_TUNING
    ++n_done;
#endif
  }
  if (lane == 0) bulk_wait_all();
#ifdef DGB_TUNING
  if (P.diag && lane == 0) {
    unsigned long long t_end;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long* d = P.diag + 4 * (static_cast<size_t>(mset) * n_gw + gw);
    d[0] = t_begin;
    d[1] = t_end;
    d[2] = clock64() - c_begin;
    d[3] = (static_cast<unsigned long long>(n_done) << 32) | smid;
  }
#endif
}

}  // namespace v2
}  // namespace dgb
