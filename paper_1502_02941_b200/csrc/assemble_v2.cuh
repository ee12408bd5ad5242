// assemble_v2.cuh -- the element-per-thread block-row kernel (included by dg_assembly.cu).
//
// One thread assembles one element's whole BSR block row (diagonal block + one block per
// interior neighbour) and RHS slice, entirely in registers:
//
//  * element-independent reference tensors (volume Gram / mass / transport tensors, the
//    kappa-folded face consistency tensors W = kappa Q^T - Q, face mass tensors, basis and
//    trace tables) travel as a __grid_constant__ kernel parameter, so with every loop index
//    known at compile time each DFMA reads its tensor operand straight from the constant bank
//    (no load instruction);
//  * per-point face terms and the neighbour blocks use the factored form
//        K_ef = sum_p phi^l_p (x) b1_p + a2_p (x) phi^lf_(n-1-p)
//    (SURVEY.md Appendix A regrouped): only the neighbour's trace rows depend on the
//    neighbour's local edge lf, and those are read per lane from a shared-memory copy --
//    no divergent tensor selection;
//  * a warp stages each block kind (diagonal, then the neighbour across local edge 0, 1, 2)
//    in shared memory and writes it back with coalesced stores at the block's sorted slot.
#pragma once

namespace dgb {
namespace v2 {

// Flat layout of the tensor parameter block (offsets in doubles, all compile-time).
template <int NL, int NQV, int NQE, bool TRIG>
struct Lay {
  static constexpr int N2 = NL * NL;
  static constexpr bool kHasP = !TRIG && NL <= 10;   // face mass tensors (constant b)
  static constexpr bool kHasTA = !TRIG && NL <= 10;  // affine transport tensors
  static constexpr int S = 0;                               // 3: S00, S01 + S10, S11
  static constexpr int M = S + 3 * N2;                      // 1: mass
  static constexpr int W = M + N2;                          // 6: kappa Q^T - Q  [l][a]
  static constexpr int T = W + 6 * N2;                      // 2: transport (constant b)
  static constexpr int TA = T + (TRIG ? 0 : 2) * N2;        // 4: affine transport [a][c]
  static constexpr int P = TA + (kHasTA ? 4 : 0) * N2;      // 3: face mass [l]
  static constexpr int PHI = P + (kHasP ? 3 : 0) * N2;      // [q][i]
  static constexpr int DPHI = PHI + NQV * NL;               // [q][a][i]      (TRIG only)
  static constexpr int EPHI = DPHI + (TRIG ? NQV * 2 * NL : 0);  // [l][p][i]
  static constexpr int EDPHI = EPHI + 3 * NQE * NL;         // [l][p][a][i]
  static constexpr int VX = EDPHI + 3 * NQE * 2 * NL;
  static constexpr int VY = VX + NQV;
  static constexpr int VW = VY + NQV;
  static constexpr int ET = VW + NQV;
  static constexpr int EW = ET + NQE;
  static constexpr int TOTAL = EW + NQE;
};

template <int NL, int NQV, int NQE, bool TRIG>
struct Tab {
  double x[Lay<NL, NQV, NQE, TRIG>::TOTAL];
};

template <int NL, int NQV, int NQE, bool TRIG>
struct Params2 {
  const double* nodes;
  const int32_t* elements;
  const uint8_t* edge_kind;
  const int32_t* edge_elements;
  const int32_t* element_edges;
  const int32_t* row_ptr;
  int32_t* col;
  double* val;
  double* rhs;
  int32_t* err_edge;
  int32_t n_elements;
  int32_t row_begin, row_end;  // block rows [row_begin, row_end) of this launch (a shard)
  int32_t drop_neumann;
  double kappa, sigma_i, sigma_b;
  dgb_problem prob;
  Tab<NL, NQV, NQE, TRIG> t;
};

// Per-edge state of one element (registers).
struct EdgeState {
  double ax, ay, dx, dy;  // sorted-pair start point and direction (edge points a + t d)
  double h, rh, nx, ny;   // length, 1 / length, outward unit normal of this element
  double ge0, ge1;        // G_e^T n
  double gf0, gf1;        // G_f^T n (interior)
  double eps;             // edge diffusivity
  int kind, lf, o, slot;  // kind, neighbour local edge, orientation, block slot
  int edge;
};

template <int NL, int NQV, int NQE, bool TRIG>
__device__ __forceinline__ void flux_point(const Params2<NL, NQV, NQE, TRIG>& P, const EdgeState& s,
                                           int q, double& px, double& py, double& fl) {
  using L = Lay<NL, NQV, NQE, TRIG>;
  px = FADD(s.ax, FMUL(P.t.x[L::ET + q], s.dx));
  py = FADD(s.ay, FMUL(P.t.x[L::ET + q], s.dy));
  double bx, by;
  velocity(P.prob.advection, px, py, bx, by);
  fl = FADD(FMUL(bx, s.nx), FMUL(by, s.ny));
}

// Staging stride (doubles) per lane: even, so 16-byte chunks stay aligned.
template <int N2>
struct Stage {
  static constexpr int kStride = (N2 % 2 == 0) ? N2 + 2 : N2 + 1;
};

// Warp-cooperative write of one staged block kind: lane L's block (if base_L >= 0) goes to
// val[base_L .. base_L + N2).  Even N2: 16-byte moves (block starts are 16-byte aligned since
// N2 * 8 is a multiple of 16); odd N2: 8-byte moves.
template <int N2>
__device__ __forceinline__ void flush_blocks(const double* st, long long base, double* val,
                                             int lane) {
  constexpr int S = Stage<N2>::kStride;
  __syncwarp();
  if constexpr (N2 % 2 == 0) {
    // 16-byte chunks c = lane + 32 it of the flattened [32 lanes][N2 / 2] staging; (L, k)
    // advance by 32 chunks per iteration without a division.
    constexpr int H = N2 / 2, DL = 32 / H, DK = 32 % H;
    int L = lane / H, k = lane - L * H;
#pragma unroll 3
    for (int it = 0; it < H; ++it) {
      const long long b = __shfl_sync(0xffffffffu, base, L & 31);
      if (L < 32) {
        const double2 x = *reinterpret_cast<const double2*>(st + L * S + 2 * k);
        if (b >= 0) *reinterpret_cast<double2*>(val + b + 2 * k) = x;
      }
      k += DK;
      L += DL;
      if (k >= H) {
        k -= H;
        ++L;
      }
    }
  } else {
    constexpr int DL = 32 / N2, DK = 32 % N2;
    int L = lane / N2, k = lane - L * N2;
#pragma unroll 3
    for (int it = 0; it < N2; ++it) {
      const long long b = __shfl_sync(0xffffffffu, base, L & 31);
      if (L < 32) {
        const double x = st[L * S + k];
        if (b >= 0) val[b + k] = x;
      }
      k += DK;
      L += DL;
      if (k >= N2) {
        k -= N2;
        ++L;
      }
    }
  }
  __syncwarp();
}

template <int NL, int NQV, int NQE, bool TRIG, int MINB>
__global__ void __launch_bounds__(128, MINB) assemble_kernel(
    const __grid_constant__ Params2<NL, NQV, NQE, TRIG> P) {
  constexpr int N2 = NL * NL;
  using L = Lay<NL, NQV, NQE, TRIG>;
  extern __shared__ double smem[];
  // [3][NQE][3][NL] trace table copy (phi, d0phi, d1phi per local edge / point) for the
  // per-lane neighbour rows, then one staging area of 32 x (N2 + 1) doubles per warp.
  double* tr = smem;
  constexpr int kTr = 3 * NQE * 3 * NL;
  for (int i = threadIdx.x; i < kTr; i += blockDim.x) {
    const int j = i % NL, c = (i / NL) % 3, p = (i / (3 * NL)) % NQE, l = i / (3 * NL * NQE);
    tr[i] = c == 0 ? P.t.x[L::EPHI + (l * NQE + p) * NL + j]
                   : P.t.x[L::EDPHI + ((l * NQE + p) * 2 + c - 1) * NL + j];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int SS = Stage<N2>::kStride;
  double* stw = smem + ((kTr + 1) & ~1) + warp * 32 * SS;
  double* st = stw + lane * SS;
  const int e = P.row_begin + blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = e < P.row_end;
  const int ee = active ? e : P.row_end - 1;  // inactive lanes mirror a valid element

  // ---- element geometry and edge states ---------------------------------------------------
  int v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * ee + k);
  double2 pv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pv[k] = __ldg(reinterpret_cast<const double2*>(P.nodes) + v[k]);
  const double B00 = FSUB(pv[1].x, pv[0].x), B01 = FSUB(pv[2].x, pv[0].x);
  const double B10 = FSUB(pv[1].y, pv[0].y), B11 = FSUB(pv[2].y, pv[0].y);
  const double det = FSUB(FMUL(B00, B11), FMUL(B01, B10));
  const double rdet = 1.0 / det;
  const double G00 = B11 * rdet, G01 = -B10 * rdet;
  const double G10 = -B01 * rdet, G11 = B00 * rdet;
  const double eps = scalar_element(P.prob.diffusion, ee);
  const double alpha = scalar_element(P.prob.linear_reaction, ee);
  const dgb_vector_field& bf = P.prob.advection;
  const bool bconst = bf.kind == DGB_VEC_CONSTANT;

  EdgeState es[3];
  int cols[4], kinds[4], nb = 1;
  cols[0] = ee;
  kinds[0] = -1;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    EdgeState& s = es[l];
    const int a = v[(l + 1) % 3], b = v[(l + 2) % 3];
    s.o = a < b ? 0 : 1;
    const double2 A = s.o == 0 ? pv[(l + 1) % 3] : pv[(l + 2) % 3];
    const double2 Bn = s.o == 0 ? pv[(l + 2) % 3] : pv[(l + 1) % 3];
    s.ax = A.x;
    s.ay = A.y;
    s.dx = FSUB(Bn.x, A.x);
    s.dy = FSUB(Bn.y, A.y);
    s.h = hypot_dd(s.dx, s.dy);
    s.rh = 1.0 / s.h;
    const double tx = s.dx * s.rh, ty = s.dy * s.rh;
    s.nx = s.o == 0 ? ty : -ty;
    s.ny = s.o == 0 ? -tx : tx;
    s.ge0 = G00 * s.nx + G10 * s.ny;
    s.ge1 = G01 * s.nx + G11 * s.ny;
    s.edge = __ldg(P.element_edges + 3 * ee + l);
    s.kind = __ldg(P.edge_kind + s.edge);
    s.eps = eps;
    s.lf = 0;
    s.gf0 = s.gf1 = 0.0;
    s.slot = -1;
    if (s.kind == DGB_EDGE_INTERIOR) {
      const int2 lr = __ldg(reinterpret_cast<const int2*>(P.edge_elements) + s.edge);
      const int f = lr.x == ee ? lr.y : lr.x;
      int vf[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) vf[k] = __ldg(P.elements + 3 * f + k);
#pragma unroll
      for (int k = 0; k < 3; ++k) if (vf[k] != a && vf[k] != b) s.lf = k;
      const Geo gf = element_geo_fast(P.nodes, vf);
      s.gf0 = gf.G00 * s.nx + gf.G10 * s.ny;
      s.gf1 = gf.G01 * s.nx + gf.G11 * s.ny;
      if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
        const double ef = __ldg(P.prob.diffusion.per_element + f);
        s.eps = ee < f ? 0.5 * (eps + ef) : 0.5 * (ef + eps);
      }
      cols[nb] = f;
      kinds[nb++] = l;
    }
  }
  // sorted block columns -> slots
#pragma unroll
  for (int a = 1; a < 4; ++a) {
#pragma unroll
    for (int b = a; b > 0; --b) {
      if (b < nb && cols[b - 1] > cols[b]) {
        int t = cols[b]; cols[b] = cols[b - 1]; cols[b - 1] = t;
        t = kinds[b]; kinds[b] = kinds[b - 1]; kinds[b - 1] = t;
      }
    }
  }
  const int rp = __ldg(P.row_ptr + (ee - P.row_begin));
  int diag_slot = 0;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (s < nb) {
      if (active) P.col[rp + s] = cols[s];
      if (kinds[s] < 0) diag_slot = s;
#pragma unroll
      for (int l = 0; l < 3; ++l) if (kinds[s] == l) es[l].slot = s;
    }
  }

  // ---- diagonal block ----------------------------------------------------------------------
  {
    const double de = det * eps;
    const double cD0 = de * (G00 * G00 + G10 * G10);
    const double cD1 = de * (G00 * G01 + G10 * G11);
    const double cD2 = de * (G01 * G01 + G11 * G11);
    const double cR = det * alpha;
    double cC0 = 0.0, cC1 = 0.0, cA[4] = {0.0, 0.0, 0.0, 0.0};
    if (!TRIG) {
      if (bconst) {
        cC0 = det * (G00 * bf.p[0] + G10 * bf.p[1]);
        cC1 = det * (G01 * bf.p[0] + G11 * bf.p[1]);
      } else if (bf.kind == DGB_VEC_AFFINE) {
        const double bo0 = bf.p[0] + bf.p[2] * pv[0].x + bf.p[3] * pv[0].y;
        const double bo1 = bf.p[1] + bf.p[4] * pv[0].x + bf.p[5] * pv[0].y;
        const double AB00 = bf.p[2] * B00 + bf.p[3] * B10, AB01 = bf.p[2] * B01 + bf.p[3] * B11;
        const double AB10 = bf.p[4] * B00 + bf.p[5] * B10, AB11 = bf.p[4] * B01 + bf.p[5] * B11;
        cC0 = det * (G00 * bo0 + G10 * bo1);
        cC1 = det * (G01 * bo0 + G11 * bo1);
        cA[0] = det * (G00 * AB00 + G10 * AB10);
        cA[1] = det * (G00 * AB01 + G10 * AB11);
        cA[2] = det * (G01 * AB00 + G11 * AB10);
        cA[3] = det * (G01 * AB01 + G11 * AB11);
      }
    }
    // face coefficients: W weights and either the per-edge P weight (constant b) or the
    // per-point weights cU (penalty + upwind at each point, canonical point order)
    double cW[3][2], cP[3], cU[3][NQE];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const EdgeState& s = es[l];
      cW[l][0] = cW[l][1] = cP[l] = 0.0;
#pragma unroll
      for (int p = 0; p < NQE; ++p) cU[l][p] = 0.0;
      if (s.kind == DGB_EDGE_NEUMANN) {
        if (!P.drop_neumann && active) {
          bool inflow = false;
          for (int q = 0; q < NQE; ++q) {
            double px, py, fl;
            flux_point(P, s, q, px, py, fl);
            double bx, by;
            velocity(bf, px, py, bx, by);
            if (fl < -1e-12 * fmax(1.0, hypot_dd(bx, by))) inflow = true;
          }
          if (inflow) atomicMin(P.err_edge, s.edge);
        }
        continue;
      }
      const bool interior = s.kind == DGB_EDGE_INTERIOR;
      const double sig = interior ? P.sigma_i : P.sigma_b;
      const double base = (interior ? 0.5 : 1.0) * s.h * s.eps;
      cW[l][0] = base * s.ge0;
      cW[l][1] = base * s.ge1;
      const double sh = sig * s.rh;
      if (bconst && L::kHasP) {
        const double fl = FADD(FMUL(bf.p[0], s.nx), FMUL(bf.p[1], s.ny));
        double up = 0.0;
        if (interior) {
          if (fl < 0.0) up = -FMUL(s.h, fl);
        } else if (fl < -1e-12 * fmax(1.0, hypot_dd(bf.p[0], bf.p[1]))) {
          up = -FMUL(s.h, fl);
        }
        cP[l] = sh * (s.h * s.eps) + up;
      } else {
        double fls[NQE];  // indexed by canonical point p (physical point q = q(p))
        bool inflow = false;
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const int q = s.o == 0 ? p : NQE - 1 - p;
          double px, py;
          flux_point(P, s, q, px, py, fls[p]);
          if (!interior) {
            double bx, by;
            velocity(bf, px, py, bx, by);
            if (fls[p] < -1e-12 * fmax(1.0, hypot_dd(bx, by))) inflow = true;
          }
        }
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const int q = s.o == 0 ? p : NQE - 1 - p;
          const double w = FMUL(P.t.x[L::EW + q], s.h);
          double c = FMUL(sh, FMUL(w, s.eps));
          if ((interior || inflow) && fls[p] < 0.0) c -= FMUL(w, fls[p]);
          cU[l][p] = c;
        }
      }
    }
    double bq[TRIG ? NQV : 1][2];
    if (TRIG) {
#pragma unroll
      for (int q = 0; q < NQV; ++q) {
        const double px = FADD(FADD(pv[0].x, FMUL(B00, P.t.x[L::VX + q])), FMUL(B01, P.t.x[L::VY + q]));
        const double py = FADD(FADD(pv[0].y, FMUL(B10, P.t.x[L::VX + q])), FMUL(B11, P.t.x[L::VY + q]));
        double bx, by;
        velocity(bf, px, py, bx, by);
        const double dw = det * P.t.x[L::VW + q];
        bq[q][0] = dw * (G00 * bx + G10 * by);
        bq[q][1] = dw * (G01 * bx + G11 * by);
      }
    }
    constexpr int RC = NL <= 6 ? NL : (NL <= 10 ? 2 : 1);  // rows per register chunk
#pragma unroll 1
    for (int i0 = 0; i0 < NL; i0 += RC) {
      double acc[RC][NL];
#pragma unroll
      for (int r = 0; r < RC; ++r) {
#pragma unroll
        for (int j = 0; j < NL; ++j) {
          const int k = (i0 + r) * NL + j;
          double x = cD0 * P.t.x[L::S + k];
          x = fma(cD1, P.t.x[L::S + N2 + k], x);
          x = fma(cD2, P.t.x[L::S + 2 * N2 + k], x);
          x = fma(cR, P.t.x[L::M + k], x);
          if (!TRIG) {
            x = fma(cC0, P.t.x[L::T + k], x);
            x = fma(cC1, P.t.x[L::T + N2 + k], x);
            if (L::kHasTA && !bconst) {
#pragma unroll
              for (int a = 0; a < 4; ++a) x = fma(cA[a], P.t.x[L::TA + a * N2 + k], x);
            }
          }
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            x = fma(cW[l][0], P.t.x[L::W + 2 * l * N2 + k], x);
            x = fma(cW[l][1], P.t.x[L::W + (2 * l + 1) * N2 + k], x);
            if (L::kHasP) x = fma(cP[l], P.t.x[L::P + l * N2 + k], x);
          }
          acc[r][j] = x;
        }
      }
      if (!(bconst && L::kHasP)) {
#pragma unroll
        for (int l = 0; l < 3; ++l) {
#pragma unroll
          for (int p = 0; p < NQE; ++p) {
#pragma unroll
            for (int r = 0; r < RC; ++r) {
              const double u = cU[l][p] * P.t.x[L::EPHI + (l * NQE + p) * NL + i0 + r];
#pragma unroll
              for (int j = 0; j < NL; ++j) acc[r][j] = fma(u, P.t.x[L::EPHI + (l * NQE + p) * NL + j], acc[r][j]);
            }
          }
        }
      }
      if (TRIG) {
#pragma unroll
        for (int q = 0; q < NQV; ++q) {
#pragma unroll
          for (int r = 0; r < RC; ++r) {
            const double f0 = bq[TRIG ? q : 0][0] * P.t.x[L::PHI + q * NL + i0 + r];
            const double f1 = bq[TRIG ? q : 0][1] * P.t.x[L::PHI + q * NL + i0 + r];
#pragma unroll
            for (int j = 0; j < NL; ++j) {
              acc[r][j] = fma(f0, P.t.x[L::DPHI + (2 * q) * NL + j],
                              fma(f1, P.t.x[L::DPHI + (2 * q + 1) * NL + j], acc[r][j]));
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < RC; ++r) {
#pragma unroll
        for (int j = 0; j < NL; ++j) st[(i0 + r) * NL + j] = acc[r][j];
      }
    }
    flush_blocks<N2>(stw, active ? static_cast<long long>(rp + diag_slot) * N2 : -1LL, P.val,
                     lane);
  }

  // ---- neighbour blocks (one pass per local edge) -------------------------------------------
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const EdgeState& s = es[l];
    const bool has = s.kind == DGB_EDGE_INTERIOR;
    if (has) {
      // coefficients (off-diagonal block)
      const double base = 0.5 * s.h * s.eps;
      const double cY0 = -base * s.gf0, cY1 = -base * s.gf1;
      const double cZ0 = -P.kappa * base * s.ge0, cZ1 = -P.kappa * base * s.ge1;
      const double sh = P.sigma_i * s.rh;
      double cV[NQE];
      double flc = 0.0;
      if (bconst) flc = FADD(FMUL(bf.p[0], s.nx), FMUL(bf.p[1], s.ny));
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const int q = s.o == 0 ? p : NQE - 1 - p;
        const double w = FMUL(P.t.x[L::EW + q], s.h);
        double fl = flc;
        if (!bconst) {
          double px, py;
          flux_point(P, s, q, px, py, fl);
        }
        double c = -FMUL(sh, FMUL(w, s.eps));
        if (fl < 0.0) c += FMUL(w, fl);
        cV[p] = c;
      }
      const double* trm = tr + s.lf * (NQE * 3 * NL);
      constexpr int CJ = NL <= 6 ? NL : 2;  // columns per register chunk
#pragma unroll 1
      for (int j0 = 0; j0 < NL; j0 += CJ) {
        double pm[NQE][CJ], b1[NQE][CJ];
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double* row = trm + (NQE - 1 - p) * 3 * NL;
#pragma unroll
          for (int c = 0; c < CJ; ++c) {
            const int j = j0 + c;
            const double f = row[j], g0 = row[NL + j], g1 = row[2 * NL + j];
            pm[p][c] = f;
            b1[p][c] = fma(cV[p], f, P.t.x[L::EW + p] * fma(cY0, g0, cY1 * g1));
          }
        }
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          double acc[CJ];
#pragma unroll
          for (int c = 0; c < CJ; ++c) acc[c] = 0.0;
#pragma unroll
          for (int p = 0; p < NQE; ++p) {
            const double a2 = P.t.x[L::EW + p] * fma(cZ0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i], cZ1 * P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i]);
#pragma unroll
            for (int c = 0; c < CJ; ++c) {
              acc[c] = fma(P.t.x[L::EPHI + (l * NQE + p) * NL + i], b1[p][c], fma(a2, pm[p][c], acc[c]));
            }
          }
#pragma unroll
          for (int c = 0; c < CJ; ++c) st[i * NL + j0 + c] = acc[c];
        }
      }
    }
    const long long bb = (active && has) ? static_cast<long long>(rp + s.slot) * N2 : -1LL;
    if (__any_sync(0xffffffffu, bb >= 0)) flush_blocks<N2>(stw, bb, P.val, lane);
  }

  // ---- RHS --------------------------------------------------------------------------------
  {
    double F[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) F[i] = 0.0;
    const dgb_scalar_field& fs = P.prob.source;
#pragma unroll
    for (int q = 0; q < NQV; ++q) {
      double f;
      if (fs.kind == DGB_FIELD_CONSTANT) {
        f = fs.value;
      } else if (fs.kind == DGB_FIELD_PER_ELEMENT) {
        f = __ldg(fs.per_element + ee);
      } else {
        const double px = FADD(FADD(pv[0].x, FMUL(B00, P.t.x[L::VX + q])), FMUL(B01, P.t.x[L::VY + q]));
        const double py = FADD(FADD(pv[0].y, FMUL(B10, P.t.x[L::VX + q])), FMUL(B11, P.t.x[L::VY + q]));
        f = scalar_point(fs, px, py);
      }
      const double c = det * P.t.x[L::VW + q] * f;
#pragma unroll
      for (int i = 0; i < NL; ++i) F[i] = fma(c, P.t.x[L::PHI + q * NL + i], F[i]);
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      const EdgeState& s = es[l];
      if (s.kind == DGB_EDGE_INTERIOR) continue;
      double cG[NQE], cH[NQE];
      if (s.kind == DGB_EDGE_NEUMANN) {
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const int q = s.o == 0 ? p : NQE - 1 - p;
          const double px = FADD(s.ax, FMUL(P.t.x[L::ET + q], s.dx));
          const double py = FADD(s.ay, FMUL(P.t.x[L::ET + q], s.dy));
          cG[p] = FMUL(FMUL(P.t.x[L::EW + q], s.h), scalar_point(P.prob.neumann, px, py));
          cH[p] = 0.0;
        }
      } else {
        double fls[NQE], gds[NQE];  // canonical point order
        bool inflow = false;
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const int q = s.o == 0 ? p : NQE - 1 - p;
          double px, py;
          flux_point(P, s, q, px, py, fls[p]);
          double bx, by;
          velocity(bf, px, py, bx, by);
          if (fls[p] < -1e-12 * fmax(1.0, hypot_dd(bx, by))) inflow = true;
          gds[p] = scalar_point(P.prob.dirichlet, px, py);
        }
        const double sh = P.sigma_b * s.rh;
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const int q = s.o == 0 ? p : NQE - 1 - p;
          const double w = FMUL(P.t.x[L::EW + q], s.h);
          const double wgd = w * gds[p];
          double g = wgd * (sh * s.eps);
          if (inflow && fls[p] < 0.0) g += -FMUL(w, fls[p]) * gds[p];
          cG[p] = g;
          cH[p] = wgd * (P.kappa * s.eps);
        }
      }
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double h0 = cH[p] * s.ge0, h1 = cH[p] * s.ge1;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          F[i] = fma(cG[p], P.t.x[L::EPHI + (l * NQE + p) * NL + i],
                     fma(h0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i], fma(h1, P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], F[i])));
        }
      }
    }
    // stage the warp's contiguous RHS range and write it coalesced
#pragma unroll
    for (int i = 0; i < NL; ++i) st[i] = F[i];
    __syncwarp();
    const int e_first = blockIdx.x * blockDim.x + warp * 32;  // relative to row_begin
    const int n_here = min(32, P.row_end - P.row_begin - e_first);
    for (int idx = lane; idx < n_here * NL; idx += 32) {
      const int L = idx / NL, i = idx - L * NL;
      P.rhs[static_cast<long long>(e_first) * NL + idx] = stw[L * SS + i];
    }
  }
}

}  // namespace v2
}  // namespace dgb
