// assemble_p1_ws.cuh -- warp-specialised P1 block-row kernel (constant velocity, bound mesh:
// configs 1 and 4).  Included by dg_assembly.cu after assemble_ws.cuh.
//
// The persistent one-lane-per-element kernel (assemble_p1.cuh) holds every element's whole
// block row in one thread: 168 registers, 12 warps per SM, and ncu shows it bound by the
// dependency latency of its FP64 chains (issue slots ~50% busy, `wait` the top stall).  Here
// the row is split between two warp roles that each need about half the live state, so more
// warps fit and the two halves overlap:
//
//   producer (one lane per element of a 32-element chunk): the gathers, the element's
//     geometry, the source at the volume points and the boundary RHS terms, each local edge's
//     coefficients -- the diagonal face weights (w0, w1, cp) and the neighbour-block weights
//     (cx, the rotated uY0 / uY1, cZ0, cZ1) -- written to a shared-memory slot [field][lane];
//     it also stores the chunk's row_ptr, block columns and RHS;
//   consumer (same lane <-> element): the diagonal block (volume terms, then the face terms of
//     edges 0, 1, 2 in order) and the neighbour blocks from those coefficients, staged as the
//     chunk's contiguous BSR row range and copied out with 16-byte stores.
//
// Every term is the same expression, in the same order, as in p1_row: the outputs are bitwise
// those of the one-lane kernel.  Slots form a ring handed over with mbarriers (as the P2
// warp-specialised kernel, assemble_ws.cuh).
#pragma once

namespace dgb {
namespace v2 {

template <int NQV, int NQE, int NPROD, int NCONS, int NSLOT>
struct SmemP1Ws {
  static constexpr int NP = NPROD, NC = NCONS, NS = NSLOT;
  static constexpr int kThreads = 32 * (NP + NC);
  // slot rows [row][lane] (doubles): volume coefficients, then per edge l: w0 w1 cp cx uY0 uY1
  // cZ0 cZ1; then the ints: per edge kind | lf << 2 | slot << 4, the row's first block, the
  // diagonal slot, the active flag
  static constexpr int kVol = 6, kPerEdge = 8, kRows = kVol + 3 * kPerEdge;
  static constexpr int kInts = 6 * 32;
  static constexpr int kSlot = kRows * 32 + kInts / 2;
  static constexpr int kStage = (32 * 4 * 9 + 2 + 1) & ~1;  // consumer's staged row range
  static constexpr int kTr = (3 * NQE * 3 * 3 + 1) & ~1;
  static constexpr int kBars = 2 * NS;
  // producer gather pipeline (as the persistent one-lane kernel): one chunk's records and
  // nodes land in shared memory by cp.async while the previous chunk computes
  static constexpr int kPre = ChunkRec::kIdx + ChunkRec::kNode;
  static constexpr size_t kBytes = sizeof(double) * (size_t(kBars) + kTr + size_t(NS) * kSlot +
                                                     size_t(NC) * kStage + size_t(NP) * kPre);
};

template <int NQV, int NQE, int NP, int NC, int NS>
__global__ void __launch_bounds__(SmemP1Ws<NQV, NQE, NP, NC, NS>::kThreads, 1)
    assemble_p1_ws_kernel(const __grid_constant__ Params2<3, NQV, NQE, false, true> P) {
  constexpr int NL = 3, N2 = 9;
  using L = Lay<NL, NQV, NQE, false, true>;
  using W = SmemP1Ws<NQV, NQE, NP, NC, NS>;
  extern __shared__ double smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);  // [NS][full, empty]
  double* tr = smem + W::kBars;
  double* slots = tr + W::kTr;
  double* stage_base = slots + NS * W::kSlot;
  double* pre_base = stage_base + NC * W::kStage;
  p1_tables<NQV, NQE, true>(P, tr);
  if (threadIdx.x < W::kBars) mbar_init(bars + threadIdx.x, 32);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mset = blockIdx.y;
  const double kappa = P.bt[mset].kappa, sigma_i = P.bt[mset].sigma_i, sigma_b = P.bt[mset].sigma_b;
  const dgb_vector_field& bf = P.prob.advection;
  const int n_rows = P.row_end - P.row_begin;
  const int n_chunks = (n_rows + 31) >> 5;
  const int n_local = n_chunks > static_cast<int>(blockIdx.x)
                          ? (n_chunks - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                          : 0;
  const unsigned long long pol_out = output_policy(P.evict_first);

  if (warp < NP) {
    // ================================ producer =================================================
    int32_t* const o_row_ptr = P.bt[mset].row_ptr;
    int32_t* const o_col = P.bt[mset].col;
    double* const o_rhs = P.bt[mset].rhs;
    const double2* nodes2 = reinterpret_cast<const double2*>(P.nodes);
    const unsigned long long pol_g = evict_last_policy();
    const bool hints = P.load_hints;
    int* idx = reinterpret_cast<int*>(pre_base + warp * W::kPre);             // records
    double2* nod = reinterpret_cast<double2*>(pre_base + warp * W::kPre + ChunkRec::kIdx);
    auto chunk_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
    auto issue_records = [&](int k) {
      const int e = P.row_begin + chunk_of(k) * 32 + lane;
      const int r = min(e, P.row_end - 1) - P.row_begin;
      cp_async16(idx + ChunkRec::kNb + 4 * lane, P.adj_nb + r);
      cp_async16(idx + ChunkRec::kOp + 4 * lane, P.adj_op + r);
#pragma unroll
      for (int q = 0; q < 3; ++q) cp_async4(idx + ChunkRec::kV + 3 * lane + q, P.elements + 3 * (P.row_begin + r) + q);
      cp_async4(idx + ChunkRec::kRp + lane, P.row_ptr_src + r);
      cp_async4(idx + ChunkRec::kRpn + lane, P.row_ptr_src + r + 1);
      cp_async_commit();
    };
    auto issue_nodes = [&]() {  // from the landed records
      if (hints) {
#pragma unroll
        for (int q = 0; q < 3; ++q) cp_async16_hint(nod + q * 32 + lane, nodes2 + idx[ChunkRec::kV + 3 * lane + q], pol_g);
#pragma unroll
        for (int q = 0; q < 3; ++q)
          cp_async16_hint(nod + (3 + q) * 32 + lane, nodes2 + max(idx[ChunkRec::kOp + 4 * lane + q], 0), pol_g);
      } else {
#pragma unroll
        for (int q = 0; q < 3; ++q) cp_async16(nod + q * 32 + lane, nodes2 + idx[ChunkRec::kV + 3 * lane + q]);
#pragma unroll
        for (int q = 0; q < 3; ++q) cp_async16(nod + (3 + q) * 32 + lane, nodes2 + max(idx[ChunkRec::kOp + 4 * lane + q], 0));
      }
      cp_async_commit();
    };
    if (warp < n_local) {
      issue_records(warp);
      cp_async_wait_all();
      issue_nodes();
    }
#pragma unroll 1
    for (int k = warp; k < n_local; k += NP) {
      const int s = k % NS, rnd = k / NS;
      double* sl = slots + s * W::kSlot;
      int* si = reinterpret_cast<int*>(sl + W::kRows * 32);
      const int e_first = chunk_of(k) * 32;
      const int e = P.row_begin + e_first + lane;
      const bool active = e < P.row_end;
      const int ee = active ? e : P.row_end - 1;
      const int r = ee - P.row_begin;
      // ---- this chunk's records and nodes (landed), then the next chunk's record copies
      cp_async_wait_all();
      const int v[3] = {idx[ChunkRec::kV + 3 * lane], idx[ChunkRec::kV + 3 * lane + 1],
                        idx[ChunkRec::kV + 3 * lane + 2]};
      const int4 anb = *reinterpret_cast<const int4*>(idx + ChunkRec::kNb + 4 * lane);
      const int rp = idx[ChunkRec::kRp + lane], rp_next = idx[ChunkRec::kRpn + lane];
      const double2 pv[3] = {nod[lane], nod[32 + lane], nod[64 + lane]};
      const double2 po[3] = {nod[96 + lane], nod[128 + lane], nod[160 + lane]};
      const bool more = k + NP < n_local;
      if (more) issue_records(k + NP);  // each lane overwrites only what it read itself
      // ---- neighbours, sorted block columns -> slots (p1_row, bound)
      int kindv[3], lfv[3], fv[3];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        kindv[l] = (anb.w >> (4 * l)) & 3;
        lfv[l] = (anb.w >> (4 * l + 2)) & 3;
        fv[l] = l == 0 ? anb.x : (l == 1 ? anb.y : anb.z);
        if (kindv[l] != DGB_EDGE_INTERIOR) fv[l] = -1;
      }
      int slot_of[4];
      {
        const int cx[4] = {ee, fv[0], fv[1], fv[2]};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          int rk = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) rk += (j != i && cx[j] >= 0 && cx[j] < cx[i]) ? 1 : 0;
          slot_of[i] = rk;
        }
      }
      if (rnd > 0) mbar_wait(bars + 2 * s + 1, (rnd - 1) & 1);  // empty: round rnd - 1 consumed
      if (active) {
        o_row_ptr[r + 1] = rp_next;
        if (r == 0) o_row_ptr[0] = 0;
        o_col[rp + slot_of[0]] = ee;
#pragma unroll
        for (int l = 0; l < 3; ++l) if (fv[l] >= 0) o_col[rp + slot_of[1 + l]] = fv[l];
      }
#pragma unroll
      for (int l = 0; l < 3; ++l) si[l * 32 + lane] = kindv[l] | (lfv[l] << 2) | (slot_of[1 + l] << 4);
      si[3 * 32 + lane] = rp;
      si[4 * 32 + lane] = slot_of[0];
      si[5 * 32 + lane] = active ? 1 : 0;

      // ---- own geometry, volume coefficients
      const double B00 = FSUB(pv[1].x, pv[0].x), B01 = FSUB(pv[2].x, pv[0].x);
      const double B10 = FSUB(pv[1].y, pv[0].y), B11 = FSUB(pv[2].y, pv[0].y);
      const double det = FSUB(FMUL(B00, B11), FMUL(B01, B10));
      const double rdet = rcp_nr(det);
      const double G00 = B11 * rdet, G01 = -B10 * rdet;
      const double G10 = -B01 * rdet, G11 = B00 * rdet;
      const double eps = scalar_element(P.prob.diffusion, ee);
      {
        const double alpha = scalar_element(P.prob.linear_reaction, ee);
        const double de = det * eps;
        sl[0 * 32 + lane] = de * (G00 * G00 + G10 * G10);
        sl[1 * 32 + lane] = de * (G00 * G01 + G10 * G11);
        sl[2 * 32 + lane] = de * (G01 * G01 + G11 * G11);
        sl[3 * 32 + lane] = det * alpha;
        sl[4 * 32 + lane] = det * (G00 * bf.p[0] + G10 * bf.p[1]);
        sl[5 * 32 + lane] = det * (G01 * bf.p[0] + G11 * bf.p[1]);
      }
      // ---- RHS volume term
      double F[NL];
#pragma unroll
      for (int i = 0; i < NL; ++i) F[i] = 0.0;
      source_points<NQV, false>(
          P.prob.source, ee, false,
          [&](int q, double& px, double& py) {
            px = fma(B01, P.t.x[L::VY + q], fma(B00, P.t.x[L::VX + q], pv[0].x));
            py = fma(B11, P.t.x[L::VY + q], fma(B10, P.t.x[L::VX + q], pv[0].y));
          },
          [&](int q, double f, double, double) {
            const double c = (det * P.t.x[L::VW + q]) * f;
#pragma unroll
            for (int i = 0; i < NL; ++i) F[i] = fma(c, P.t.x[L::PHI + q * NL + i], F[i]);
          });
      if (more) {  // the next chunk's records have landed: issue its node gathers
        cp_async_wait_all();
        issue_nodes();
      }
      // ---- edges: coefficients (the expressions of p1_row)
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double* er = sl + (W::kVol + l * W::kPerEdge) * 32 + lane;
        const int a = v[(l + 1) % 3], b = v[(l + 2) % 3];
        const int o = a < b ? 0 : 1;
        const double2 A = o == 0 ? pv[(l + 1) % 3] : pv[(l + 2) % 3];
        const double2 Bn = o == 0 ? pv[(l + 2) % 3] : pv[(l + 1) % 3];
        const double dx = FSUB(Bn.x, A.x), dy = FSUB(Bn.y, A.y);
        const double rh = rsqrt_nr(fma(dx, dx, dy * dy));
        const double h = fma(dx, dx, dy * dy) * rh;
        const double tx = dx * rh, ty = dy * rh;
        const double nx = o == 0 ? ty : -ty, ny = o == 0 ? -tx : tx;
        const double ge0 = G00 * nx + G10 * ny, ge1 = G01 * nx + G11 * ny;
        const int kind = kindv[l], lf = lfv[l], f = fv[l];
        double w0 = 0.0, w1 = 0.0, cp = 0.0;
        if (kind == DGB_EDGE_INTERIOR) {
          const Geo gf = element_geo_coords(po[l], pv[(l + 2) % 3], pv[(l + 1) % 3]);
          double eps_e = eps;
          if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
            const double ef = __ldg(P.prob.diffusion.per_element + f);
            eps_e = ee < f ? 0.5 * (eps + ef) : 0.5 * (ef + eps);
          }
          const double base = 0.5 * h * eps_e;
          w0 = base * ge0;
          w1 = base * ge1;
          const double cY0 = -base * (gf.G00 * nx + gf.G10 * ny);
          const double cY1 = -base * (gf.G01 * nx + gf.G11 * ny);
          const double cZ0 = -kappa * base * ge0;
          const double cZ1 = -kappa * base * ge1;
          const double sh = sigma_i * rh;
          const double fl = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
          const double up = fl < 0.0 ? FMUL(h, fl) : 0.0;
          cp = sh * (h * eps_e) - up;
          const double cxv = up - sh * (h * eps_e);
          double uY0 = cY0, uY1 = cY1;
          if (lf == 1) {
            uY0 = -cY0 - cY1;
            uY1 = cY0;
          } else if (lf == 2) {
            uY0 = cY1;
            uY1 = -cY0 - cY1;
          }
          er[3 * 32] = cxv;
          er[4 * 32] = uY0;
          er[5 * 32] = uY1;
          er[6 * 32] = cZ0;
          er[7 * 32] = cZ1;
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
        er[0] = w0;
        er[32] = w1;
        er[2 * 32] = cp;
      }
      if (active) {
        double* dst = o_rhs + static_cast<long long>(r) * NL;
#pragma unroll
        for (int i = 0; i < NL; ++i) store_one(dst + i, F[i], pol_out);
      }
      mbar_arrive(bars + 2 * s);  // full (release: this lane's slot writes)
    }
  } else {
    // ================================ consumer =================================================
    double* const o_val = P.bt[mset].val;
    const int cw = warp - NP;
    double* stw = stage_base + cw * W::kStage;
#pragma unroll 1
    for (int k = cw; k < n_local; k += NC) {
      const int s = k % NS, rnd = k / NS;
      const double* sl = slots + s * W::kSlot;
      const int* si = reinterpret_cast<const int*>(sl + W::kRows * 32);
      mbar_wait(bars + 2 * s, rnd & 1);  // full: round rnd produced
      const int rp = si[3 * 32 + lane];
      const int diag_slot = si[4 * 32 + lane];
      const bool active = si[5 * 32 + lane] != 0;
      int nb = 1;
#pragma unroll
      for (int l = 0; l < 3; ++l) nb += (si[l * 32 + lane] & 3) == DGB_EDGE_INTERIOR ? 1 : 0;
      const int rp_first = __shfl_sync(0xffffffffu, rp, 0);
      const int rp_last = __reduce_max_sync(0xffffffffu, active ? rp + nb : 0);
      double* srow = stw + (rp_first & 1);
      double* const myrow = srow + (rp - rp_first) * N2;
      // diagonal: volume terms (p1_row's chain)
      double acc[N2];
      {
        const double cD0 = sl[0 * 32 + lane], cD1 = sl[1 * 32 + lane], cD2 = sl[2 * 32 + lane];
        const double cR = sl[3 * 32 + lane], cC0 = sl[4 * 32 + lane], cC1 = sl[5 * 32 + lane];
#pragma unroll
        for (int q = 0; q < N2; ++q) {
          double x = cD0 * P.t.x[L::S + q];
          x = fma(cD1, P.t.x[L::S + N2 + q], x);
          x = fma(cD2, P.t.x[L::S + 2 * N2 + q], x);
          x = fma(cR, P.t.x[L::M + q], x);
          x = fma(cC0, P.t.x[L::T + q], x);
          x = fma(cC1, P.t.x[L::T + N2 + q], x);
          acc[q] = x;
        }
      }
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const double* er = sl + (W::kVol + l * W::kPerEdge) * 32 + lane;
        const int meta = si[l * 32 + lane];
        if ((meta & 3) == DGB_EDGE_INTERIOR) {
          const int lf = (meta >> 2) & 3, bslot = meta >> 4;
          const double cxv = er[3 * 32], uY0 = er[4 * 32], uY1 = er[5 * 32];
          const double cZ0 = er[6 * 32], cZ1 = er[7 * 32];
          const double* trm = tr + lf * (NQE * 3 * NL);
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
          double* blk = myrow + bslot * N2;
#pragma unroll
          for (int i = 0; i < NL; ++i) {
            double rr[NL];
#pragma unroll
            for (int j = 0; j < NL; ++j) rr[j] = 0.0;
#pragma unroll
            for (int p = 0; p < NQE; ++p) {
              const double a2 = fma(cZ0, P.t.x[L::EDW + ((l * NQE + p) * 2) * NL + i],
                                    cZ1 * P.t.x[L::EDW + ((l * NQE + p) * 2 + 1) * NL + i]);
              const double ph = P.t.x[L::EPHI + (l * NQE + p) * NL + i];
#pragma unroll
              for (int j = 0; j < NL; ++j) rr[j] = fma(ph, b1[p][j], fma(a2, pm[p][j], rr[j]));
            }
#pragma unroll
            for (int j = 0; j < NL; ++j) if (active) blk[i * NL + j] = rr[j];
          }
        }
        const double w0 = er[0], w1 = er[32], cp = er[2 * 32];
#pragma unroll
        for (int q = 0; q < N2; ++q) {
          acc[q] = fma(w0, P.t.x[L::W + 2 * l * N2 + q], fma(w1, P.t.x[L::W + (2 * l + 1) * N2 + q], acc[q]));
          acc[q] = fma(cp, P.t.x[L::P + l * N2 + q], acc[q]);
        }
      }
      mbar_arrive(bars + 2 * s + 1);  // empty: the slot's values are in registers / staging
      if (active) {
#pragma unroll
        for (int q = 0; q < N2; ++q) myrow[diag_slot * N2 + q] = acc[q];
      }
      __syncwarp();
      {
        const int n = (rp_last - rp_first) * N2;
        double* dst = o_val + static_cast<long long>(rp_first) * N2;
        const int head = rp_first & 1;
        const double2* s2 = reinterpret_cast<const double2*>(srow + head);
        const int npair = (n - head) >> 1;
#pragma unroll 4
        for (int q = lane; q < npair; q += 32) {
          const double2 w = s2[q];
          store_pair(dst + head + 2 * q, w.x, w.y, pol_out);
        }
        if (lane == 1 && head && n > 0) store_one(dst, srow[0], pol_out);
        if (lane == 2 && n > 0 && ((n - head) & 1)) store_one(dst + n - 1, srow[n - 1], pol_out);
      }
      __syncwarp();
    }
  }
}

}  // namespace v2
}  // namespace dgb
