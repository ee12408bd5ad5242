// dg_assembly.cu -- B200 (sm_100a) assembly of the interior-penalty DG system.
//
// Replaces the reference hot path dgfem::assemble_all + DgSystem::stiffness
// (/root/reference/proj/src/assembly.cpp:725-737, :508-510).  Design:
//
//  * Gather formulation: every element writes only its own BSR block
//    row -- diagonal block plus one block per interior-edge neighbour, block columns sorted --
//    and its own RHS slice.  Each interior face is evaluated from both sides; no atomics, no
//    triplet sort, bitwise reproducible.
//  * Reference-tensor contraction: on affine triangles with element-constant eps / alpha
//    every block is a short linear combination of element-independent nl x nl tensors built
//    once per plan from the reference tables (volume Gram / mass / transport tensors,
//    per-(local edge, neighbour local edge) face tensors).  Coefficients that depend on the
//    element (geometry, edge normals, penalties, per-point upwind weights, per-point source
//    and boundary data) are computed per element in phase A and combined in phase B.
//  * Decisions that select terms (upwind side per point, exact-zero flux skip, inflow
//    tolerance gate, outward normal) use unfused IEEE operations (__dmul_rn/__dadd_rn) on
//    the reference's expressions so they fall the same way as on the CPU.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <limits>
#include <map>
#include <type_traits>
#include <vector>

#include <cub/device/device_scan.cuh>

#include "common.hpp"
#include "device_math.cuh"

namespace dgb {

// ------------------------------------------------------------------------------------------
// layouts
// ------------------------------------------------------------------------------------------
constexpr int kTensorQ = 64;  // max volume points supported
constexpr int kMaxQE = 8;     // max edge points supported

// Offsets (in doubles) of the reference-contraction tensors in the plan's device buffer.
// Every tensor is nl x nl row-major [i][j]; the per-point tables are [.][i].
struct Layout {
  int S;     // 3 tensors: S00, S01 + S10, S11      S^ab_ij = sum_q w_q d_a phi_qj d_b phi_qi
  int M;     // 1: sum_q w_q phi_qi phi_qj
  int T;     // 2: T^a_ij = sum_q w_q phi_qi d_a phi_qj
  int TA;    // 4: TA^{a,c}_ij = sum_q w_q xhat_qc phi_qi d_a phi_qj   (affine velocity)
  int TQ;    // 2 nqv: TQ^{q,a}_ij = phi_qi d_a phi_qj                  (pointwise velocity)
  int Q;     // 6: Q^{l,a}_ij = sum_p w_p phi^l_pi d_a phi^l_pj        (face consistency)
  int U;     // 3 nqe: U^{l,p}_ij = phi^l_pi phi^l_pj                  (face penalty/upwind)
  int V;     // 9 nqe: V^{l,m,p}_ij = phi^l_pi phi^m_(n-1-p)j          (cross penalty/upwind)
  int Y;     // 18: Y^{l,m,a}_ij = sum_p w_p phi^l_pi d_a phi^m_(n-1-p)j
  int Z;     // 18: Z^{l,m,a}_ij = sum_p w_p d_a phi^l_pi phi^m_(n-1-p)j
  int PHI;   // nqv x nl volume basis
  int EPHI;  // 3 nqe x nl edge traces (canonical orientation)
  int EDPHI; // 3 nqe 2 x nl edge gradients
  int VX, VY, VW, ET, EW;  // quadrature points / weights
  int total;
};

// Offsets (in doubles) inside one element's coefficient record (shared memory).
struct Rec {
  int cD, cR, cC, cCA, cCQ, cF, cW, cU, cY, cZ, cV, cG, cH, gam, size;
};

constexpr int kMeta = 16;  // ints per element: see phase A0

struct KParams {
  // mesh (device)
  const double* nodes;
  const int32_t* elements;
  const uint8_t* edge_kind;
  const int32_t* edge_elements;
  const int32_t* element_edges;
  int32_t n_elements;
  int32_t row_begin, row_end;  // block rows of this launch
  // problem (by value; per-element pointers are device pointers)
  dgb_problem prob;
  double kappa, sigma_i, sigma_b;
  int32_t drop_neumann;
  // tables
  const double* tens;
  Layout L;
  Rec R;
  int nl, nqv, nqe;
  int tile;
  // outputs
  const int32_t* row_ptr;
  int32_t* col;
  double* val;
  double* rhs;
  unsigned long long* err_edge;  // epoch << 32 | ~edge (see dgb_plan_status)
  unsigned long long epoch;
};

// ------------------------------------------------------------------------------------------
// device helpers (FMUL / FADD / FSUB / FDIV and hypot_dd: device_math.cuh)
// ------------------------------------------------------------------------------------------

// The two transcendental families, out of family() so the hoisted-dispatch source loop
// (source_points) runs them with the same expressions.
// gx = p0 / p3, gy = p1 / p3 are point-independent: source_points computes them once per
// element (the same divisions, so the same bits).
__device__ __forceinline__ void family_tanh_g(const double* p, double gx, double gy, double x,
                                              double y, double& u, double& ux, double& uy,
                                              double& lap) {
  // Same expressions as the reference's BoundaryLayer (problems.cpp:81-98): far from the
  // layer F is dominated by the rounding of u = (1 - tanh s) / 2, so parity needs tanh.
  const double s = (p[0] * x + p[1] * y + p[2]) / p[3];
  const double t = tanh(s);
  const double c = cosh(s);
  const double sech2 = 1.0 / (c * c);
  u = 0.5 * (1.0 - t);
  ux = -0.5 * sech2 * gx;
  uy = -0.5 * sech2 * gy;
  lap = t * sech2 * (gx * gx + gy * gy);
}
__device__ __forceinline__ void family_tanh(const double* p, double x, double y, double& u,
                                            double& ux, double& uy, double& lap) {
  family_tanh_g(p, p[0] / p[3], p[1] / p[3], x, y, u, ux, uy, lap);
}
__device__ __forceinline__ void family_gauss(const double* p, double x, double y, double& u,
                                             double& ux, double& uy, double& lap) {
  const double dx = x - p[1], dy = y - p[2];
  const double r2 = dx * dx + dy * dy;
  const double v = exp_fast(-p[0] * r2);
  u = v;
  ux = -2.0 * p[0] * dx * v;
  uy = -2.0 * p[0] * dy * v;
  lap = (4.0 * p[0] * p[0] * r2 - 4.0 * p[0]) * v;
}

__device__ __forceinline__ void family(int fn, const double* p, double x, double y, double& u,
                                       double& ux, double& uy, double& lap) {
  constexpr double pi = 3.14159265358979323846;
  switch (fn) {
    case DGB_FN_SIN_SIN: {
      double sx, cx, sy, cy;
      sincos(pi * x, &sx, &cx);
      sincos(pi * y, &sy, &cy);
      u = p[0] * (sx * sy);
      ux = p[0] * (pi * cx * sy);
      uy = p[0] * (pi * sx * cy);
      lap = -2.0 * pi * pi * u;
      return;
    }
    case DGB_FN_TANH_LAYER:
      family_tanh(p, x, y, u, ux, uy, lap);
      return;
    case DGB_FN_GAUSSIAN:
      family_gauss(p, x, y, u, ux, uy, lap);
      return;
    case DGB_FN_AFFINE:
      u = p[0] + p[1] * x + p[2] * y;
      ux = p[1];
      uy = p[2];
      lap = 0.0;
      return;
    case DGB_FN_STEP_Y:
      u = (y < p[0]) ? p[1] : p[2];
      ux = uy = lap = 0.0;
      return;
    default:
      u = ux = uy = lap = nan("");
  }
}

// FUNCTION scalar field at a point (out of line: one copy of the transcendental families).
__device__ __noinline__ double scalar_function(int fn, int mode, double p0, double p1, double p2,
                                               double p3, double q0, double q1, double q2,
                                               double q3, double x, double y) {
  const double p[4] = {p0, p1, p2, p3};
  double u, ux, uy, lap;
  family(fn, p, x, y, u, ux, uy, lap);
  switch (mode) {
    case DGB_MODE_VALUE: return u;
    case DGB_MODE_SOURCE: return q0 * u - q1 * lap + q2 * ux + q3 * uy;
    case DGB_MODE_SOURCE_SQUARE: return (q0 * u - q1 * lap + q2 * ux + q3 * uy) + u * u;
    case DGB_MODE_FLUX_X: return q1 * ux;
    default: return nan("");
  }
}

// CONSTANT / FUNCTION scalar field at a point (device twin of oracle/dg_coeffs.h).
__device__ __forceinline__ double scalar_point(const dgb_scalar_field& f, double x, double y) {
  if (f.kind == DGB_FIELD_CONSTANT) return f.value;
  return scalar_function(f.fn, f.mode, f.p[0], f.p[1], f.p[2], f.p[3], f.q[0], f.q[1], f.q[2],
                         f.q[3], x, y);
}

// Boundary data g(x, y) on an edge with end points a, b, through the branch-free cores
// (device_math.cuh) when the field is the VALUE of a sine-product or Gaussian family and the
// edge lies inside the cores' ranges; otherwise scalar_point.  A boundary edge is evaluated by
// one or two lanes of a warp while the others wait, so its instruction count is paid by all 32.
__device__ __forceinline__ bool boundary_fast_ok(const dgb_scalar_field& f, double2 a, double2 b) {
  if (f.kind != DGB_FIELD_FUNCTION || f.mode != DGB_MODE_VALUE) return false;
  if (f.fn == DGB_FN_SIN_SIN) {
    return fmax(fmax(fabs(a.x), fabs(a.y)), fmax(fabs(b.x), fabs(b.y))) < 1e8;
  }
  if (f.fn == DGB_FN_GAUSSIAN) {
    const double ax = a.x - f.p[1], ay = a.y - f.p[2], bx = b.x - f.p[1], by = b.y - f.p[2];
    return fabs(f.p[0]) * fmax(fma(ax, ax, ay * ay), fma(bx, bx, by * by)) < 708.0;
  }
  return false;
}
__device__ __forceinline__ double scalar_point_fast(const dgb_scalar_field& f, double x, double y, bool fast) {
  if (fast) {
    if (f.fn == DGB_FN_SIN_SIN) {
      // the penalty multiplies g by sigma eps / h, so where F is small (g ~ 0 on the unit
      // square's boundary) parity at 1e-12 needs the reference's sin(pi * x) of the ROUNDED
      // product, not sin of the exact pi x
      return f.p[0] * (sin_pi_product(x) * sin_pi_product(y));
    }
    const double dx = x - f.p[1], dy = y - f.p[2];
    return exp_core(-f.p[0] * fma(dx, dx, dy * dy));
  }
  return scalar_point(f, x, y);
}

__device__ __forceinline__ double scalar_point_inline(const dgb_scalar_field& f, double x, double y) {
  if (f.kind == DGB_FIELD_CONSTANT) return f.value;
  double u, ux, uy, lap;
  family(f.fn, f.p, x, y, u, ux, uy, lap);
  switch (f.mode) {
    case DGB_MODE_VALUE: return u;
    case DGB_MODE_SOURCE: return f.q[0] * u - f.q[1] * lap + f.q[2] * ux + f.q[3] * uy;
    case DGB_MODE_SOURCE_SQUARE: return (f.q[0] * u - f.q[1] * lap + f.q[2] * ux + f.q[3] * uy) + u * u;
    case DGB_MODE_FLUX_X: return f.q[1] * ux;
    default: return nan("");
  }
}

// The source at every volume point of an element, with the coefficient dispatch hoisted out
// of the point loop: one loop per common (family, SOURCE) pair, the generic loop otherwise.
// xy(q, x, y) gives point q, use(q, f, x, y) consumes its value; same expressions as
// scalar_point_inline.  UseXY: the caller needs the points even for constant sources.  skip
// (profiling ablation): f = x.
#ifndef DGB_SRC_UNROLL
#define DGB_SRC_UNROLL 1
#endif
constexpr int kSrcUnroll = DGB_SRC_UNROLL;  // Gaussian source point loop (tuning: -DDGB_SRC_UNROLL)
#ifndef DGB_SRC_FAST_UNROLL
#define DGB_SRC_FAST_UNROLL 6
#endif
constexpr int kSrcFastUnroll = DGB_SRC_FAST_UNROLL;  // branch-free Gaussian point loop
// No bound on the element's extent: the Gaussian source keeps its per-point range check.
struct NoExtent {
  static constexpr bool kKnown = false;
  __device__ __forceinline__ double operator()(double, double) const { return -1.0; }
};
// EXTENT (optional): r2max(cx, cy) = the largest squared distance from (cx, cy) to a vertex of
// the element, called by every lane of the warp; the volume points are convex combinations of
// the vertices, so r^2 <= r2max at each of them.
// ONLY (a kernel specialised by the host for the source it will see, source_only()): the other
// families' code is left out, which matters to a kernel whose hot loop is larger than the
// instruction cache (the P1 persistent kernel gained 3% from it).
enum SourceOnly { SRC_ANY = -1, SRC_CONST = 0, SRC_SIN_SIN = 1, SRC_GAUSSIAN = 2 };
inline int source_only(const dgb_scalar_field& fs) {
  if (fs.kind == DGB_FIELD_PER_ELEMENT || fs.kind == DGB_FIELD_CONSTANT) return SRC_CONST;
  if (fs.kind == DGB_FIELD_FUNCTION && fs.mode == DGB_MODE_SOURCE) {
    if (fs.fn == DGB_FN_SIN_SIN) return SRC_SIN_SIN;
    if (fs.fn == DGB_FN_GAUSSIAN) return SRC_GAUSSIAN;
  }
  return SRC_ANY;
}
template <int NQV, bool UseXY, int ONLY = SRC_ANY, class XY, class USE, class EXTENT = NoExtent>
__device__ __forceinline__ void source_points(const dgb_scalar_field& fs, int e, bool skip, XY xy,
                                              USE use, int q_first = 0, int q_step = 1,
                                              EXTENT r2max = EXTENT{}) {
  constexpr bool kAny = ONLY == SRC_ANY;
  if constexpr (kAny || ONLY == SRC_CONST) {
  if (!kAny || fs.kind == DGB_FIELD_PER_ELEMENT || fs.kind == DGB_FIELD_CONSTANT) {
    const double f = fs.kind == DGB_FIELD_PER_ELEMENT ? __ldg(fs.per_element + e) : fs.value;
#pragma unroll 1
    for (int q = q_first; q < NQV; q += q_step) {
      double x = 0.0, y = 0.0;
      if (UseXY) xy(q, x, y);
      use(q, f, x, y);
    }
    return;
  }
  }
  if constexpr (kAny || ONLY == SRC_SIN_SIN) {
  if (!kAny || (!skip && fs.mode == DGB_MODE_SOURCE && fs.fn == DGB_FN_SIN_SIN)) {
    // u = p0 sin(pi x) sin(pi y): the source q0 u - q1 lap(u) + q2 u_x + q3 u_y regrouped as
    // p0 ((q0 + 2 pi^2 q1) sx sy + pi q2 cx sy + pi q3 sx cy), with sincospi: a cheaper
    // reduction than sincos of the rounded product pi * x (the reference's sin(pi * x) differs
    // from sin of the exact pi x by at most ~7e-16 absolute).  Config 1's batch: 0.198 -> 0.163 ms.
    constexpr double pi = 3.14159265358979323846;
    const double A = fs.p[0] * fma(2.0 * pi * pi, fs.q[1], fs.q[0]);
    const double Bx = fs.p[0] * (pi * fs.q[2]), By = fs.p[0] * (pi * fs.q[3]);
    if constexpr (EXTENT::kKnown) {
      // every point's coordinates are inside sincospi_core's range (checked once, at the
      // vertices, for the whole warp): branch-free point loop, unrolled points overlap
      if (__all_sync(0xffffffffu, r2max(0.0, 0.0) < 1e16)) {
#pragma unroll kSrcFastUnroll
        for (int q = q_first; q < NQV; q += q_step) {
          double x, y, sx, cx, sy, cy;
          xy(q, x, y);
          sincospi_core(x, sx, cx);
          sincospi_core(y, sy, cy);
          use(q, fma(A * sx, sy, fma(Bx * cx, sy, (By * sx) * cy)), x, y);
        }
        return;
      }
    }
#pragma unroll 1
    for (int q = q_first; q < NQV; q += q_step) {
      double x, y, sx, cx, sy, cy;
      xy(q, x, y);
      sincospi(x, &sx, &cx);
      sincospi(y, &sy, &cy);
      use(q, fma(A * sx, sy, fma(Bx * cx, sy, (By * sx) * cy)), x, y);
    }
    return;
  }
  }
  if constexpr (kAny || ONLY == SRC_GAUSSIAN) {
  if (!kAny || (!skip && fs.mode == DGB_MODE_SOURCE && (fs.fn == DGB_FN_GAUSSIAN || fs.fn == DGB_FN_TANH_LAYER))) {
    const double q0 = fs.q[0], q1 = fs.q[1], q2 = fs.q[2], q3 = fs.q[3];
    if (!kAny || fs.fn == DGB_FN_GAUSSIAN) {
      // u = exp(-a r^2), r = (x - cx, y - cy): the source
      //   q0 u - q1 lap(u) + q2 u_x + q3 u_y = u (K0 + K1 r^2 + K2 dx + K3 dy),
      //   K0 = q0 + 4 a q1, K1 = -4 a^2 q1, K2 = -2 a q2, K3 = -2 a q3,
      // is the same function as family_gauss's four-term form (no cancellation between the
      // regrouped terms: they are each O(a^2 r^2) or O(a)), at 8 instead of 14 operations
      // per point besides the exp
      const double a = fs.p[0], cx = fs.p[1], cy = fs.p[2];
      const double K0 = fma(4.0 * a, q1, q0), K1 = -4.0 * a * a * q1;
      const double K2 = -2.0 * a * q2, K3 = -2.0 * a * q3;
      if constexpr (EXTENT::kKnown) {
        // every point's exponent is inside exp_core's range (checked once, at the vertices, for
        // the whole warp): the point loop is branch-free, so unrolled points overlap
        if (__all_sync(0xffffffffu, fabs(a) * r2max(cx, cy) < 708.0)) {
#pragma unroll kSrcFastUnroll
          for (int q = q_first; q < NQV; q += q_step) {
            double x, y;
            xy(q, x, y);
            const double dx = x - cx, dy = y - cy;
            const double r2 = fma(dx, dx, dy * dy);
            const double v = exp_core(-a * r2);
            use(q, v * fma(K1, r2, fma(K2, dx, fma(K3, dy, K0))), x, y);
          }
          return;
        }
      }
#pragma unroll kSrcUnroll
      for (int q = q_first; q < NQV; q += q_step) {
        double x, y;
        xy(q, x, y);
        const double dx = x - cx, dy = y - cy;
        const double r2 = fma(dx, dx, dy * dy);
        const double v = exp_fast(-a * r2);
        use(q, v * fma(K1, r2, fma(K2, dx, fma(K3, dy, K0))), x, y);
      }
    } else if constexpr (kAny) {
      const double gx = fs.p[0] / fs.p[3], gy = fs.p[1] / fs.p[3];
#pragma unroll 1
      for (int q = q_first; q < NQV; q += q_step) {
        double x, y, u, ux, uy, lap;
        xy(q, x, y);
        family_tanh_g(fs.p, gx, gy, x, y, u, ux, uy, lap);
        use(q, q0 * u - q1 * lap + q2 * ux + q3 * uy, x, y);
      }
    }
    return;
  }
  }
  if constexpr (kAny) {
#pragma unroll 1
    for (int q = q_first; q < NQV; q += q_step) {
      double x, y;
      xy(q, x, y);
      use(q, skip ? x : scalar_point_inline(fs, x, y), x, y);
    }
  }
}

__device__ __forceinline__ double scalar_element(const dgb_scalar_field& f, int e) {
  return f.kind == DGB_FIELD_PER_ELEMENT ? __ldg(f.per_element + e) : f.value;
}

__device__ __noinline__ void velocity_trig(double w0, double w1, double x, double y, double& bx,
                                          double& by) {
  bx = cos(FMUL(w0, y));
  by = sin(FMUL(w1, x));
}

// Velocity at a point; the affine form keeps the reference's unfused evaluation order.
__device__ __forceinline__ void velocity(const dgb_vector_field& b, double x, double y,
                                         double& bx, double& by) {
  switch (b.kind) {
    case DGB_VEC_CONSTANT:
      bx = b.p[0];
      by = b.p[1];
      return;
    case DGB_VEC_AFFINE:
      bx = FADD(FADD(b.p[0], FMUL(b.p[2], x)), FMUL(b.p[3], y));
      by = FADD(FADD(b.p[1], FMUL(b.p[4], x)), FMUL(b.p[5], y));
      return;
    case DGB_VEC_TRIG:
      velocity_trig(b.p[0], b.p[1], x, y, bx, by);
      return;
    default:
      bx = by = nan("");
  }
}

struct Geo {
  double B00, B01, B10, B11, G00, G01, G10, G11, det, ox, oy;
};

// element_geometry (mesh.cpp:212-230), unfused.
__device__ __forceinline__ Geo element_geo(const double* __restrict__ nodes,
                                           const int32_t* v) {
  Geo g;
  const double2 p0 = __ldg(reinterpret_cast<const double2*>(nodes) + v[0]);
  const double2 p1 = __ldg(reinterpret_cast<const double2*>(nodes) + v[1]);
  const double2 p2 = __ldg(reinterpret_cast<const double2*>(nodes) + v[2]);
  g.B00 = FSUB(p1.x, p0.x);
  g.B01 = FSUB(p2.x, p0.x);
  g.B10 = FSUB(p1.y, p0.y);
  g.B11 = FSUB(p2.y, p0.y);
  g.det = FSUB(FMUL(g.B00, g.B11), FMUL(g.B01, g.B10));
  g.G00 = FDIV(g.B11, g.det);
  g.G01 = FDIV(-g.B10, g.det);
  g.G10 = FDIV(-g.B01, g.det);
  g.G11 = FDIV(g.B00, g.det);
  g.ox = p0.x;
  g.oy = p0.y;
  return g;
}

// element_geometry with one reciprocal instead of four divisions (values only; no term-selecting
// decision depends on G).
// element_geo_fast from coordinates already in registers (same arithmetic).
__device__ __forceinline__ Geo element_geo_coords(double2 p0, double2 p1, double2 p2) {
  Geo g;
  g.B00 = p1.x - p0.x;
  g.B01 = p2.x - p0.x;
  g.B10 = p1.y - p0.y;
  g.B11 = p2.y - p0.y;
  g.det = FSUB(FMUL(g.B00, g.B11), FMUL(g.B01, g.B10));
  const double rd = rcp_nr(g.det);
  g.G00 = g.B11 * rd;
  g.G01 = -g.B10 * rd;
  g.G10 = -g.B01 * rd;
  g.G11 = g.B00 * rd;
  g.ox = p0.x;
  g.oy = p0.y;
  return g;
}

__device__ __forceinline__ Geo element_geo_fast(const double* __restrict__ nodes,
                                                const int32_t* v) {
  Geo g;
  const double2 p0 = __ldg(reinterpret_cast<const double2*>(nodes) + v[0]);
  const double2 p1 = __ldg(reinterpret_cast<const double2*>(nodes) + v[1]);
  const double2 p2 = __ldg(reinterpret_cast<const double2*>(nodes) + v[2]);
  g.B00 = p1.x - p0.x;
  g.B01 = p2.x - p0.x;
  g.B10 = p1.y - p0.y;
  g.B11 = p2.y - p0.y;
  g.det = FSUB(FMUL(g.B00, g.B11), FMUL(g.B01, g.B10));
  const double rd = rcp_nr(g.det);
  g.G00 = g.B11 * rd;
  g.G01 = -g.B10 * rd;
  g.G10 = -g.B01 * rd;
  g.G11 = g.B00 * rd;
  g.ox = p0.x;
  g.oy = p0.y;
  return g;
}

// Meta ints per element (shared memory):
//  0: n_blocks   1: diagonal slot   2..4: slot of local edge l (-1: boundary)
//  5..7: neighbour local edge lf    8..10: edge kind    11..13: vertices    14: element
enum { M_NB = 0, M_DIAG = 1, M_SLOT = 2, M_LF = 5, M_KIND = 8, M_VERT = 11 };
constexpr int kGeo = 13;  // doubles per element: B(4) G(4) det ox oy eps alpha

}  // namespace dgb

#include "assemble_v2.cuh"
#include "assemble_ws.cuh"
#include "assemble_p1.cuh"
#include "nonlinear.cuh"
#include "postprocess.cuh"

namespace dgb {

// ------------------------------------------------------------------------------------------
// pattern: row_ptr = scan(1 + #interior edges); also resets the error word
// ------------------------------------------------------------------------------------------
__global__ void count_blocks_kernel(const uint8_t* __restrict__ edge_kind,
                                    const int32_t* __restrict__ element_edges, int32_t begin,
                                    int32_t n, int32_t* __restrict__ row_ptr) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r == 0) row_ptr[0] = 0;
  if (r >= n) return;
  const int e = begin + r;
  int c = 1;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    c += __ldg(edge_kind + __ldg(element_edges + 3 * e + l)) == DGB_EDGE_INTERIOR;
  }
  row_ptr[r + 1] = c;
}

// Element adjacency record of rows [begin, begin + n) (bound once per mesh): per local edge l
// the neighbour element, the neighbour's vertex opposite the shared edge, and kind | lf << 2 in
// bits 4l..4l+3 of nb.w (bits 12..25: block slots, edge orientations, block count).  Replaces the per-assembly chain element_edges -> edge_elements ->
// elements[f] of dependent gathers (the "geometry / neighbour precompute" of the north star).
__global__ void adjacency_kernel(const int32_t* __restrict__ elements,
                                 const uint8_t* __restrict__ edge_kind,
                                 const int32_t* __restrict__ edge_elements,
                                 const int32_t* __restrict__ element_edges, int32_t begin,
                                 int32_t n, int4* __restrict__ nb, int4* __restrict__ op) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int e = begin + r;
  int nbr[3] = {-1, -1, -1}, opp[3] = {-1, -1, -1}, meta = 0;
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int edge = __ldg(element_edges + 3 * e + l);
    const int kind = __ldg(edge_kind + edge);
    int lf = 0;
    if (kind == DGB_EDGE_INTERIOR) {
      const int2 lr = __ldg(reinterpret_cast<const int2*>(edge_elements) + edge);
      const int f = lr.x == e ? lr.y : lr.x;
      const int a = __ldg(elements + 3 * e + (l + 1) % 3), b = __ldg(elements + 3 * e + (l + 2) % 3);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const int v = __ldg(elements + 3 * f + k);
        if (v != a && v != b) {
          lf = k;
          opp[l] = v;
        }
      }
      nbr[l] = f;
    }
    meta |= (kind | (lf << 2)) << (4 * l);
    // make_side orientation of local edge l (assembly.cpp:125-126): 1 when a > b
    const int a = __ldg(elements + 3 * e + (l + 1) % 3), b = __ldg(elements + 3 * e + (l + 2) % 3);
    meta |= (a < b ? 0 : 1) << (20 + l);
  }
  {
    // slots of the row's blocks (rank among its sorted block columns) in bits 12..19: the
    // diagonal, then local edges 0..2; the row's block count in bits 23..25
    const int cx[4] = {e, nbr[0], nbr[1], nbr[2]};
    int n_blocks = 1;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int rank = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) rank += (j != i && cx[j] >= 0 && cx[j] < cx[i]) ? 1 : 0;
      meta |= rank << (12 + 2 * i);
      if (i > 0 && cx[i] >= 0) ++n_blocks;
    }
    meta |= n_blocks << 23;
  }
  nb[r] = make_int4(nbr[0], nbr[1], nbr[2], meta);
  op[r] = make_int4(opp[0], opp[1], opp[2], 0);
}

// Geometry record of rows [begin, begin + n) per 32-row chunk (bound once per mesh, the P1
// persistent kernel; the "geometry precompute" of the north star):
//   geo[(chunk * kGeoRows + k) * 32 + lane], k = 0..2: the element's own vertices
//                                     k = 3..5: G_f^T n of the neighbour across local edge k - 3
//                                               (the neighbour's inverse-transposed Jacobian in
//                                               its (opposite, b, a) vertex order applied to
//                                               this element's outward normal; 0 on a boundary)
//                                     k = 6, 7 (DGB_GEO_RECIPROCALS builds only):
//                                               (1 / det, 1 / h_0), (1 / h_1, 1 / h_2)
// The block-row kernel then reads its geometry with coalesced 16-byte copies: no random node
// gathers and no neighbour Jacobians.  The values come from the same device functions the
// kernels without a record use (p1_edge_frame, p1_neighbour_normal); results agree to the last
// bits (each kernel instantiation has its own FMA contraction).  Lanes past the last row repeat it.
__global__ void geometry_kernel(const double* __restrict__ nodes, const int32_t* __restrict__ elements,
                                const int4* __restrict__ nb, const int4* __restrict__ op,
                                int32_t begin, int32_t n, double2* __restrict__ geo) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ((n + 31) & ~31)) return;
  const int r = min(t, n - 1);
  const int e = begin + r;
  const double2* nodes2 = reinterpret_cast<const double2*>(nodes);
  const int4 o = __ldg(op + r);
  const int meta = __ldg(nb + r).w;
  double2* g = geo + static_cast<size_t>(t >> 5) * (v2::kGeoRows * 32) + (t & 31);
  double2 pv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pv[k] = __ldg(nodes2 + __ldg(elements + 3 * e + k));
  const int opp[3] = {o.x, o.y, o.z};
  double rh[3];
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const v2::EdgeFrame fr = v2::p1_edge_frame(pv, l);
    rh[l] = fr.rh;
    double2 gn = make_double2(0.0, 0.0);
    if (((meta >> (4 * l)) & 3) == DGB_EDGE_INTERIOR) {
      gn = v2::p1_neighbour_normal(__ldg(nodes2 + opp[l]), pv[(l + 2) % 3], pv[(l + 1) % 3], fr.nx, fr.ny);
    }
    g[(3 + l) * 32] = gn;
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) g[k * 32] = pv[k];
  const double det = FSUB(FMUL(FSUB(pv[1].x, pv[0].x), FSUB(pv[2].y, pv[0].y)),
                          FMUL(FSUB(pv[2].x, pv[0].x), FSUB(pv[1].y, pv[0].y)));
  if constexpr (v2::kGeoRows == 8) {
    g[6 * 32] = make_double2(rcp_nr(det), rh[0]);
    g[7 * 32] = make_double2(rh[1], rh[2]);
  }
}

// ------------------------------------------------------------------------------------------
// the block-row kernel
// ------------------------------------------------------------------------------------------
template <int NL>
__global__ void __launch_bounds__(256) assemble_kernel(const __grid_constant__ KParams P) {
  extern __shared__ double smem[];
  constexpr int NL2 = NL * NL;
  const int TE = P.tile;
  const int e0 = P.row_begin + blockIdx.x * TE;
  const int ne = min(TE, P.row_end - e0);
  const int nqv = P.nqv, nqe = P.nqe;
  const Rec& R = P.R;
  const Layout& L = P.L;
  const double* __restrict__ tens = P.tens;

  double* rec = smem;                         // TE * R.size
  double* geo = rec + TE * R.size;            // TE * kGeo
  int* meta = reinterpret_cast<int*>(geo + TE * kGeo);  // TE * kMeta
  int* blk = meta + TE * kMeta;               // 4 * TE: (element << 3) | (kind + 1)
  int* s_nblk = blk + 4 * TE;

  // ---- A0: per element: geometry, neighbours, sorted block columns -----------------------
  for (int el = threadIdx.x; el < ne; el += blockDim.x) {
    const int e = e0 + el;
    int* m = meta + el * kMeta;
    int v[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * e + k);
    const Geo g = element_geo(P.nodes, v);
    double* gg = geo + el * kGeo;
    gg[0] = g.B00; gg[1] = g.B01; gg[2] = g.B10; gg[3] = g.B11;
    gg[4] = g.G00; gg[5] = g.G01; gg[6] = g.G10; gg[7] = g.G11;
    gg[8] = g.det; gg[9] = g.ox; gg[10] = g.oy;
    const double eps = scalar_element(P.prob.diffusion, e);
    const double alpha = scalar_element(P.prob.linear_reaction, e);
    gg[11] = eps;
    gg[12] = alpha;
    int cols[4], kinds[4];
    int nb = 0;
    cols[nb] = e;
    kinds[nb++] = -1;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      m[M_VERT + l] = v[l];
      const int edge = __ldg(P.element_edges + 3 * e + l);
      const int kind = __ldg(P.edge_kind + edge);
      m[M_KIND + l] = kind;
      m[M_SLOT + l] = -1;
      if (kind == DGB_EDGE_INTERIOR) {
        const int2 lr = __ldg(reinterpret_cast<const int2*>(P.edge_elements) + edge);
        cols[nb] = lr.x == e ? lr.y : lr.x;
        kinds[nb++] = l;
      }
    }
    // sort block columns ascending (CSR order of the reference's stiffness())
    for (int a = 1; a < nb; ++a) {
      for (int b = a; b > 0 && cols[b - 1] > cols[b]; --b) {
        int t = cols[b]; cols[b] = cols[b - 1]; cols[b - 1] = t;
        t = kinds[b]; kinds[b] = kinds[b - 1]; kinds[b - 1] = t;
      }
    }
    m[M_NB] = nb;
    const int base = __ldg(P.row_ptr + (e - P.row_begin));
    for (int s = 0; s < nb; ++s) {
      P.col[base + s] = cols[s];
      if (kinds[s] < 0) m[M_DIAG] = s; else m[M_SLOT + kinds[s]] = s;
    }
    // volume coefficients that are constant per element
    double* r = rec + el * R.size;
    const double de = g.det * eps;
    r[R.cD + 0] = de * (g.G00 * g.G00 + g.G10 * g.G10);
    r[R.cD + 1] = de * (g.G00 * g.G01 + g.G10 * g.G11);
    r[R.cD + 2] = de * (g.G01 * g.G01 + g.G11 * g.G11);
    r[R.cR] = g.det * alpha;
    const dgb_vector_field& b = P.prob.advection;
    if (b.kind == DGB_VEC_CONSTANT) {
      r[R.cC + 0] = g.det * (g.G00 * b.p[0] + g.G10 * b.p[1]);
      r[R.cC + 1] = g.det * (g.G01 * b.p[0] + g.G11 * b.p[1]);
    } else if (b.kind == DGB_VEC_AFFINE) {
      // b(o + B xhat) = (c + A o) + (A B) xhat
      const double bo0 = b.p[0] + b.p[2] * g.ox + b.p[3] * g.oy;
      const double bo1 = b.p[1] + b.p[4] * g.ox + b.p[5] * g.oy;
      const double AB00 = b.p[2] * g.B00 + b.p[3] * g.B10, AB01 = b.p[2] * g.B01 + b.p[3] * g.B11;
      const double AB10 = b.p[4] * g.B00 + b.p[5] * g.B10, AB11 = b.p[4] * g.B01 + b.p[5] * g.B11;
      r[R.cC + 0] = g.det * (g.G00 * bo0 + g.G10 * bo1);
      r[R.cC + 1] = g.det * (g.G01 * bo0 + g.G11 * bo1);
      r[R.cCA + 0] = g.det * (g.G00 * AB00 + g.G10 * AB10);  // a = 0, c = 0
      r[R.cCA + 1] = g.det * (g.G00 * AB01 + g.G10 * AB11);  // a = 0, c = 1
      r[R.cCA + 2] = g.det * (g.G01 * AB00 + g.G11 * AB10);  // a = 1, c = 0
      r[R.cCA + 3] = g.det * (g.G01 * AB01 + g.G11 * AB11);  // a = 1, c = 1
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int el = 0; el < ne; ++el) {
      const int* m = meta + el * kMeta;
      for (int s = 0; s < m[M_NB]; ++s) {
        int kind = -1;
        if (s != m[M_DIAG]) {
          for (int l = 0; l < 3; ++l) if (m[M_SLOT + l] == s) kind = l;
        }
        blk[n++] = (el << 3) | (kind + 1);
      }
    }
    *s_nblk = n;
  }

  // ---- A1: per (element, local edge): face coefficients ----------------------------------
  for (int t = threadIdx.x; t < 3 * ne; t += blockDim.x) {
    const int el = t / 3, l = t - 3 * el;
    const int e = e0 + el;
    int* m = meta + el * kMeta;
    const double* gg = geo + el * kGeo;
    double* r = rec + el * R.size;
    const int kind = m[M_KIND + l];
    const int va = m[M_VERT + (l + 1) % 3], vb = m[M_VERT + (l + 2) % 3];
    const int o = va < vb ? 0 : 1;  // make_side orientation (assembly.cpp:125-126)
    const int na = min(va, vb), nb_ = max(va, vb);
    const double2 A = __ldg(reinterpret_cast<const double2*>(P.nodes) + na);
    const double2 B = __ldg(reinterpret_cast<const double2*>(P.nodes) + nb_);
    // edge_geometry (mesh.cpp:232-257); outward normal of e from its orientation
    const double dx = FSUB(B.x, A.x), dy = FSUB(B.y, A.y);
    const double h = hypot_dd(dx, dy);
    const double tx = FDIV(dx, h), ty = FDIV(dy, h);
    const double nx = o == 0 ? ty : -ty, ny = o == 0 ? -tx : tx;
    const double gam0 = gg[4] * nx + gg[6] * ny;  // (G^T n)_0
    const double gam1 = gg[5] * nx + gg[7] * ny;  // (G^T n)_1
    r[R.gam + 2 * l] = gam0;
    r[R.gam + 2 * l + 1] = gam1;
    double* cW = r + R.cW + 2 * l;
    double* cU = r + R.cU + l * nqe;
    double* cY = r + R.cY + 2 * l;
    double* cZ = r + R.cZ + 2 * l;
    double* cV = r + R.cV + l * nqe;
    double* cG = r + R.cG + l * nqe;
    double* cH = r + R.cH + l * nqe;
    const double* et = tens + L.ET;
    const double* ew = tens + L.EW;
    const dgb_vector_field& bf = P.prob.advection;

    if (kind == DGB_EDGE_INTERIOR) {
      const int2 lr = __ldg(reinterpret_cast<const int2*>(P.edge_elements) +
                            __ldg(P.element_edges + 3 * e + l));
      const int f = lr.x == e ? lr.y : lr.x;
      int vf[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) vf[k] = __ldg(P.elements + 3 * f + k);
      int lf = 0;
#pragma unroll
      for (int k = 0; k < 3; ++k) if (vf[k] != va && vf[k] != vb) lf = k;
      m[M_LF + l] = lf;
      const Geo gf = element_geo(P.nodes, vf);
      double eps_e = gg[11];
      if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
        const double ef = __ldg(P.prob.diffusion.per_element + f);
        eps_e = e < f ? 0.5 * (gg[11] + ef) : 0.5 * (ef + gg[11]);
      }
      const double base = 0.5 * h * eps_e;  // avg * h * eps
      cW[0] = base * gam0;
      cW[1] = base * gam1;
      cY[0] = -base * (gf.G00 * nx + gf.G10 * ny);
      cY[1] = -base * (gf.G01 * nx + gf.G11 * ny);
      cZ[0] = -P.kappa * base * gam0;
      cZ[1] = -P.kappa * base * gam1;
      const double sh = FDIV(P.sigma_i, h);
      for (int q = 0; q < nqe; ++q) {
        const int p = o == 0 ? q : nqe - 1 - q;
        const double w = FMUL(ew[q], h);
        const double pen = FMUL(sh, FMUL(w, eps_e));
        double up = 0.0;
        if (bf.kind == DGB_VEC_CONSTANT) {
          const double fl = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
          if (fl < 0.0) up = FMUL(w, fl);
        } else {
          const double px = FADD(A.x, FMUL(et[q], dx)), py = FADD(A.y, FMUL(et[q], dy));
          double bx, by;
          velocity(bf, px, py, bx, by);
          const double fl = FADD(FMUL(bx, nx), FMUL(by, ny));
          if (fl < 0.0) up = FMUL(w, fl);
        }
        cU[p] = pen - up;   // diag: penalty + (-w b.n_e) on inflow points
        cV[p] = up - pen;   // off:  -penalty + (w b.n_e) on inflow points
        cG[p] = 0.0;
        cH[p] = 0.0;
      }
    } else {
      m[M_LF + l] = 0;
      cY[0] = cY[1] = cZ[0] = cZ[1] = 0.0;
      for (int q = 0; q < nqe; ++q) cV[q] = 0.0;
      const double eps_e = gg[11];
      // boundary convection gate (assembly.cpp:383-401)
      double flq[kMaxQE], pxq[kMaxQE], pyq[kMaxQE];
      bool any_inflow = false;
      for (int q = 0; q < nqe; ++q) {
        pxq[q] = FADD(A.x, FMUL(et[q], dx));
        pyq[q] = FADD(A.y, FMUL(et[q], dy));
        double bx, by;
        velocity(bf, pxq[q], pyq[q], bx, by);
        flq[q] = FADD(FMUL(bx, nx), FMUL(by, ny));
        const double tol = 1e-12 * fmax(1.0, hypot_dd(bx, by));
        if (flq[q] < -tol) any_inflow = true;
      }
      if (kind == DGB_EDGE_NEUMANN) {
        cW[0] = cW[1] = 0.0;
        if (any_inflow && !P.drop_neumann) {
          atomicMax(P.err_edge, (P.epoch << 32) |
                                    (0xFFFFFFFFull - static_cast<unsigned>(__ldg(P.element_edges + 3 * e + l))));
        }
        for (int q = 0; q < nqe; ++q) {
          const int p = o == 0 ? q : nqe - 1 - q;
          const double w = FMUL(ew[q], h);
          cU[p] = 0.0;
          cG[p] = FMUL(w, scalar_point(P.prob.neumann, pxq[q], pyq[q]));
          cH[p] = 0.0;
        }
      } else {  // Dirichlet
        const double base = h * eps_e;  // avg = 1
        cW[0] = base * gam0;
        cW[1] = base * gam1;
        const double sh = FDIV(P.sigma_b, h);
        for (int q = 0; q < nqe; ++q) {
          const int p = o == 0 ? q : nqe - 1 - q;
          const double w = FMUL(ew[q], h);
          const double pen = FMUL(sh, FMUL(w, eps_e));
          const double gd = scalar_point(P.prob.dirichlet, pxq[q], pyq[q]);
          const double wgd = w * gd;
          double win = 0.0;
          if (any_inflow && flq[q] < 0.0) win = -FMUL(w, flq[q]);
          cU[p] = pen + win;
          cG[p] = wgd * (sh * eps_e) + win * gd;
          cH[p] = wgd * (P.kappa * eps_e);
        }
      }
    }
  }

  // ---- A2: per (element, volume point): source and pointwise transport coefficients -----
  const bool pointwise_b = P.prob.advection.kind == DGB_VEC_TRIG;
  for (int t = threadIdx.x; t < nqv * ne; t += blockDim.x) {
    const int el = t / nqv, q = t - el * nqv;
    const int e = e0 + el;
    const double* gg = geo + el * kGeo;
    double* r = rec + el * R.size;
    const double xh = tens[L.VX + q], yh = tens[L.VY + q], wq = tens[L.VW + q];
    const double px = FADD(FADD(gg[9], FMUL(gg[0], xh)), FMUL(gg[1], yh));
    const double py = FADD(FADD(gg[10], FMUL(gg[2], xh)), FMUL(gg[3], yh));
    const dgb_scalar_field& fs = P.prob.source;
    const double f = fs.kind == DGB_FIELD_PER_ELEMENT ? __ldg(fs.per_element + e)
                                                      : scalar_point(fs, px, py);
    r[R.cF + q] = gg[8] * wq * f;
    if (pointwise_b) {
      double bx, by;
      velocity(P.prob.advection, px, py, bx, by);
      const double dw = gg[8] * wq;
      r[R.cCQ + 2 * q] = dw * (gg[4] * bx + gg[6] * by);
      r[R.cCQ + 2 * q + 1] = dw * (gg[5] * bx + gg[7] * by);
    }
  }
  __syncthreads();

  // ---- B: block-row values, streamed in output order ---------------------------------------
  const int nblk = *s_nblk;
  const long long vbase = static_cast<long long>(__ldg(P.row_ptr + (e0 - P.row_begin))) * NL2;
  const int bkind = P.prob.advection.kind;
  const double kappa = P.kappa;
  for (int g = threadIdx.x; g < nblk * NL2; g += blockDim.x) {
    const int bi = g / NL2, k = g - bi * NL2;
    const int i = k / NL, j = k - i * NL;
    const int code = blk[bi];
    const int el = code >> 3, kind = (code & 7) - 1;
    const double* r = rec + el * R.size;
    double v;
    if (kind < 0) {
      v = r[R.cD] * __ldg(tens + L.S + k);
      v = fma(r[R.cD + 1], __ldg(tens + L.S + NL2 + k), v);
      v = fma(r[R.cD + 2], __ldg(tens + L.S + 2 * NL2 + k), v);
      v = fma(r[R.cR], __ldg(tens + L.M + k), v);
      if (bkind == DGB_VEC_TRIG) {
        for (int q = 0; q < 2 * nqv; ++q) v = fma(r[R.cCQ + q], __ldg(tens + L.TQ + q * NL2 + k), v);
      } else {
        v = fma(r[R.cC], __ldg(tens + L.T + k), v);
        v = fma(r[R.cC + 1], __ldg(tens + L.T + NL2 + k), v);
        if (bkind == DGB_VEC_AFFINE) {
#pragma unroll
          for (int a = 0; a < 4; ++a) v = fma(r[R.cCA + a], __ldg(tens + L.TA + a * NL2 + k), v);
        }
      }
      const int kt = j * NL + i;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
#pragma unroll
        for (int a = 0; a < 2; ++a) {
          const double* Qla = tens + L.Q + (2 * l + a) * NL2;
          v = fma(r[R.cW + 2 * l + a], fma(kappa, __ldg(Qla + kt), -__ldg(Qla + k)), v);
        }
        for (int p = 0; p < nqe; ++p) {
          v = fma(r[R.cU + l * nqe + p], __ldg(tens + L.U + (l * nqe + p) * NL2 + k), v);
        }
      }
    } else {
      const int l = kind;
      const int lf = meta[el * kMeta + M_LF + l];
      const int lm = l * 3 + lf;
      v = 0.0;
      for (int p = 0; p < nqe; ++p) {
        v = fma(r[R.cV + l * nqe + p], __ldg(tens + L.V + (lm * nqe + p) * NL2 + k), v);
      }
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        v = fma(r[R.cY + 2 * l + a], __ldg(tens + L.Y + (lm * 2 + a) * NL2 + k), v);
        v = fma(r[R.cZ + 2 * l + a], __ldg(tens + L.Z + (lm * 2 + a) * NL2 + k), v);
      }
    }
    P.val[vbase + g] = v;
  }

  // ---- B': RHS slice --------------------------------------------------------------------
  for (int g = threadIdx.x; g < ne * NL; g += blockDim.x) {
    const int el = g / NL, i = g - el * NL;
    const double* r = rec + el * R.size;
    const int* m = meta + el * kMeta;
    double v = 0.0;
    for (int q = 0; q < nqv; ++q) v = fma(r[R.cF + q], __ldg(tens + L.PHI + q * NL + i), v);
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (m[M_KIND + l] == DGB_EDGE_INTERIOR) continue;
      const double g0 = r[R.gam + 2 * l], g1 = r[R.gam + 2 * l + 1];
      for (int p = 0; p < nqe; ++p) {
        const int row = l * nqe + p;
        const double dn = fma(g0, __ldg(tens + L.EDPHI + (2 * row) * NL + i),
                              g1 * __ldg(tens + L.EDPHI + (2 * row + 1) * NL + i));
        v = fma(r[R.cG + row], __ldg(tens + L.EPHI + row * NL + i), v);
        v = fma(r[R.cH + row], dn, v);
      }
    }
    P.rhs[static_cast<long long>(e0 - P.row_begin + el) * NL + i] = v;
  }
}

// ------------------------------------------------------------------------------------------
// host: tensors from reference tables
// ------------------------------------------------------------------------------------------
Layout make_layout(int nl, int nqv, int nqe) {
  const int n2 = nl * nl;
  Layout L;
  int o = 0;
  L.S = o; o += 3 * n2;
  L.M = o; o += n2;
  L.T = o; o += 2 * n2;
  L.TA = o; o += 4 * n2;
  L.TQ = o; o += 2 * nqv * n2;
  L.Q = o; o += 6 * n2;
  L.U = o; o += 3 * nqe * n2;
  L.V = o; o += 9 * nqe * n2;
  L.Y = o; o += 18 * n2;
  L.Z = o; o += 18 * n2;
  L.PHI = o; o += nqv * nl;
  L.EPHI = o; o += 3 * nqe * nl;
  L.EDPHI = o; o += 3 * nqe * 2 * nl;
  L.VX = o; o += nqv;
  L.VY = o; o += nqv;
  L.VW = o; o += nqv;
  L.ET = o; o += nqe;
  L.EW = o; o += nqe;
  L.total = o;
  return L;
}

Rec make_rec(int nqv, int nqe) {
  Rec R;
  int o = 0;
  R.cD = o; o += 3;
  R.cR = o; o += 1;
  R.cC = o; o += 2;
  R.cCA = o; o += 4;
  R.cCQ = o; o += 2 * nqv;
  R.cF = o; o += nqv;
  R.cW = o; o += 6;
  R.cU = o; o += 3 * nqe;
  R.cY = o; o += 6;
  R.cZ = o; o += 6;
  R.cV = o; o += 3 * nqe;
  R.cG = o; o += 3 * nqe;
  R.cH = o; o += 3 * nqe;
  R.gam = o; o += 6;
  R.size = o | 1;  // odd stride: spreads per-element records over banks
  return R;
}

std::vector<double> build_tensors(const dgb_reference_tables& t, const Layout& L) {
  const int nl = t.n_local, nq = t.nq_vol, ne = t.nq_edge, n2 = nl * nl;
  std::vector<double> out(L.total, 0.0);
  auto phi = [&](int q, int i) { return t.phi[q * nl + i]; };
  auto dphi = [&](int q, int i, int a) { return t.dphi[(q * nl + i) * 2 + a]; };
  auto ephi = [&](int l, int p, int i) { return t.edge_phi[((l * 2) * ne + p) * nl + i]; };
  auto edphi = [&](int l, int p, int i, int a) {
    return t.edge_dphi[(((l * 2) * ne + p) * nl + i) * 2 + a];
  };
  for (int i = 0; i < nl; ++i) {
    for (int j = 0; j < nl; ++j) {
      const int k = i * nl + j;
      long double s00 = 0, s01 = 0, s11 = 0, m = 0, t0 = 0, t1 = 0, ta[4] = {0, 0, 0, 0};
      for (int q = 0; q < nq; ++q) {
        const long double w = t.vol_w[q];
        s00 += w * dphi(q, j, 0) * dphi(q, i, 0);
        s01 += w * (static_cast<long double>(dphi(q, j, 0)) * dphi(q, i, 1) +
                    static_cast<long double>(dphi(q, j, 1)) * dphi(q, i, 0));
        s11 += w * dphi(q, j, 1) * dphi(q, i, 1);
        m += w * phi(q, j) * phi(q, i);
        t0 += w * phi(q, i) * dphi(q, j, 0);
        t1 += w * phi(q, i) * dphi(q, j, 1);
        const long double xq[2] = {t.vol_x[q], t.vol_y[q]};
        for (int a = 0; a < 2; ++a) {
          for (int c = 0; c < 2; ++c) ta[a * 2 + c] += w * xq[c] * phi(q, i) * dphi(q, j, a);
        }
        for (int a = 0; a < 2; ++a) {
          out[L.TQ + (2 * q + a) * n2 + k] = phi(q, i) * dphi(q, j, a);
        }
      }
      out[L.S + k] = static_cast<double>(s00);
      out[L.S + n2 + k] = static_cast<double>(s01);
      out[L.S + 2 * n2 + k] = static_cast<double>(s11);
      out[L.M + k] = static_cast<double>(m);
      out[L.T + k] = static_cast<double>(t0);
      out[L.T + n2 + k] = static_cast<double>(t1);
      for (int a = 0; a < 4; ++a) out[L.TA + a * n2 + k] = static_cast<double>(ta[a]);
      for (int l = 0; l < 3; ++l) {
        for (int a = 0; a < 2; ++a) {
          long double qs = 0;
          for (int p = 0; p < ne; ++p) qs += static_cast<long double>(t.edge_w[p]) * ephi(l, p, i) * edphi(l, p, j, a);
          out[L.Q + (2 * l + a) * n2 + k] = static_cast<double>(qs);
        }
        for (int p = 0; p < ne; ++p) out[L.U + (l * ne + p) * n2 + k] = ephi(l, p, i) * ephi(l, p, j);
        for (int mm = 0; mm < 3; ++mm) {
          const int lm = l * 3 + mm;
          for (int p = 0; p < ne; ++p) {
            out[L.V + (lm * ne + p) * n2 + k] = ephi(l, p, i) * ephi(mm, ne - 1 - p, j);
          }
          for (int a = 0; a < 2; ++a) {
            long double ys = 0, zs = 0;
            for (int p = 0; p < ne; ++p) {
              const long double w = t.edge_w[p];
              ys += w * ephi(l, p, i) * edphi(mm, ne - 1 - p, j, a);
              zs += w * edphi(l, p, i, a) * ephi(mm, ne - 1 - p, j);
            }
            out[L.Y + (lm * 2 + a) * n2 + k] = static_cast<double>(ys);
            out[L.Z + (lm * 2 + a) * n2 + k] = static_cast<double>(zs);
          }
        }
      }
    }
  }
  for (int q = 0; q < nq; ++q) {
    for (int i = 0; i < nl; ++i) out[L.PHI + q * nl + i] = phi(q, i);
    out[L.VX + q] = t.vol_x[q];
    out[L.VY + q] = t.vol_y[q];
    out[L.VW + q] = t.vol_w[q];
  }
  for (int l = 0; l < 3; ++l) {
    for (int p = 0; p < ne; ++p) {
      for (int i = 0; i < nl; ++i) {
        out[L.EPHI + (l * ne + p) * nl + i] = ephi(l, p, i);
        for (int a = 0; a < 2; ++a) out[L.EDPHI + ((l * ne + p) * 2 + a) * nl + i] = edphi(l, p, i, a);
      }
    }
  }
  for (int p = 0; p < ne; ++p) {
    out[L.ET + p] = t.edge_t[p];
    out[L.EW + p] = t.edge_w[p];
  }
  return out;
}

void cuda_check(cudaError_t err, const char* what) {
  if (err != cudaSuccess) {
    throw Error(DGB_STATUS_CUDA, std::string(what) + ": " + cudaGetErrorString(err));
  }
}

int tile_for(int nl) { return nl <= 6 ? 64 : 32; }

// The dynamic shared-memory limit is an attribute of a kernel in one device context: raise it
// once per (kernel, device) pair, under a lock (a process-wide flag would skip a second device,
// and concurrent first calls would race on it).
void ensure_dynamic_smem(const void* fn, size_t bytes, const char* what) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{fn, dev}];
  if (bytes > have) {
    cuda_check(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(bytes)), what);
    have = bytes;
  }
}

}  // namespace dgb

// ------------------------------------------------------------------------------------------
// plan + C-ABI
// ------------------------------------------------------------------------------------------
// The persisting-L2 carve-out (cudaLimitPersistingL2CacheSize) is one limit per device,
// shared by everything in the process.  Plans that want one hold a reference on their device:
// the first reference saves the caller's limit, the limit is only ever raised while references
// are held, and the last release restores the saved value.
namespace {
struct CarveOut {
  int refs = 0;
  size_t saved = 0;
};
std::mutex g_carve_mu;
std::map<int, CarveOut> g_carve;

// Takes (or keeps) a reference on `device`'s carve-out and raises it to at least `want`;
// returns the limit now in force.
size_t carve_acquire(int device, size_t want, bool held) {
  std::lock_guard<std::mutex> lock(g_carve_mu);
  CarveOut& c = g_carve[device];
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (!held) {
    if (c.refs == 0) c.saved = cur;
    ++c.refs;
  }
  if (cur < want) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  }
  cudaGetLastError();
  return cur;
}

void carve_release(int device) {
  std::lock_guard<std::mutex> lock(g_carve_mu);
  CarveOut& c = g_carve[device];
  if (c.refs > 0 && --c.refs == 0) {
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, c.saved);
    cudaGetLastError();
  }
}
}  // namespace

struct dgb_plan {
  int device = 0;
  int degree = 0, nl = 0, nqv = 0, nqe = 0;
  dgb::Layout L;
  dgb::Rec R;
  double* d_tens = nullptr;
  // InflowOnNeumann word: max over (epoch << 32 | ~edge), so the newest assembly's lowest
  // offending edge wins and no per-assembly reset is needed
  unsigned long long* d_err = nullptr;
  unsigned long long epoch = 0;
  // dgb_plan_status reports an InflowOnNeumann raised by any launch of the latest call, i.e.
  // an error word with epoch in [status_from, epoch] (a per-set batch spans several epochs)
  unsigned long long status_from = 0;
  bool in_batch = false;
  void* d_scan = nullptr;
  size_t scan_bytes = 0;
  int32_t scan_n = 0;
  int last_status = DGB_OK;
  cudaEvent_t ev_start = nullptr, ev_stop = nullptr;  // measurement hook (not owned)
  std::vector<double> h_tens;   // V1 layout (host copy)
  std::vector<double> h_P;      // [3][nl*nl] face mass tensors P^l
  std::vector<double> h_dphi;   // [nqv][2][nl] volume gradients
  int force_generic = 0;        // testing: always use the generic kernel
  int minblocks = 0;            // tuning: min resident CTAs/SM for the P2 kernel (0 = default)
  // pattern bound by dgb_plan_bind_mesh: row_ptr of rows [bound_begin, bound_end) of the mesh
  // whose element_edges / edge_kind arrays are bound_ee / bound_kind
  int32_t* d_pattern = nullptr;
  size_t pattern_cap = 0;
  const void* bound_ee = nullptr;
  const void* bound_kind = nullptr;
  int32_t bound_n = -1, bound_begin = -1, bound_end = -1;
  int4* d_adj = nullptr;  // neighbour records [adj_rows] then opposite vertices [adj_rows]
  size_t adj_cap = 0, adj_rows = 0;
  const void* bound_elements = nullptr;
  const void* bound_edge_elements = nullptr;
  // P1 persistent kernel: the bound rows' vertex coordinates per chunk (geometry_kernel), valid
  // for the node array bound_nodes
  double2* d_geo = nullptr;
  size_t geo_cap = 0;
  const void* bound_nodes = nullptr;
  int geo_cache = 1;            // bind the vertex coordinates too (P1 persistent kernel)
  int32_t last_launches = 0;
  size_t l2_persist_bytes = 0;  // persisting-L2 carve-out available to the node window
  bool carve_held = false;      // this plan holds a reference on its device's carve-out
  size_t l2_window_max = 0;     // cudaDevAttrMaxAccessPolicyWindowSize
  size_t l2_persist_max = 0;    // cudaDevAttrMaxPersistingL2CacheSize
  int l2_policy = -1;           // bit 0: persist nodes in L2, bit 1: evict-first output; -1 auto
  bool batch_fuse = true;       // dgb_assemble_batch: one CTA writes every kappa set
  int warp_specialized = 1;     // P-form tensor-core kernel: 0 off, 1 default split, n producers
  int sm_count = 0;
  int l2_carve_mb = 0;          // persisting-L2 carve-out cap (MiB, 0: the node array) -- tuning
  int p1_pipe = 1;              // P1 bound mesh: persistent pipelined kernel (0 off, 1 on)
  // DMMA B fragments of the diagonal terms, one table per kappa (W depends on kappa)
  std::vector<std::pair<double, double*>> bfrag_cache;
  int ablate = 0;  // profiling diagnostics (dgb_plan_set_option 1000)
  unsigned long long* d_diag = nullptr;  // tuning builds: per-warp timing records (not owned)
  // nonlinear reaction Jacobian: Phi_q,(i,j) = phi_qj phi_qi as DMMA B fragments [ks][nt][lane]
  double* d_nlfrag = nullptr;
  int nl_ks = 0;
  // neighbour trace table of the block-row kernels (phi, w d0 phi, w d1 phi of each local
  // edge's points, gradients rotated to the neighbour's (opposite, b, a) order), built once
  // per plan instead of by every CTA
  double* d_trace = nullptr;
};

namespace {

using dgb::cuda_check;

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <int NL>
void launch_assemble(const dgb::KParams& P, int n_tiles, size_t smem, cudaStream_t s) {
  dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(dgb::assemble_kernel<NL>), 200 * 1024,
                           "cudaFuncSetAttribute");
  dgb::assemble_kernel<NL><<<n_tiles, 256, smem, s>>>(P);
}

void validate_tables(const dgb_reference_tables* t) {
  if (!t || t->degree < 1 || t->degree > 4) {
    throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "polynomial degree must be between 1 and 4",
                     t ? t->degree : -1);
  }
  if (t->n_local != (t->degree + 1) * (t->degree + 2) / 2) {
    throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "n_local does not match the degree");
  }
  if (t->nq_vol < 1 || t->nq_vol > dgb::kTensorQ || t->nq_edge < 1 || t->nq_edge > dgb::kMaxQE) {
    throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "unsupported quadrature size");
  }
}

void validate_field(const dgb_scalar_field& f, bool element_constant, const char* name) {
  if (f.kind == DGB_FIELD_PER_ELEMENT && !f.per_element) {
    throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, std::string(name) + ": per_element is null");
  }
  if (element_constant && f.kind == DGB_FIELD_FUNCTION) {
    throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT,
                     std::string(name) + " must be CONSTANT or PER_ELEMENT on the GPU path");
  }
  if (f.kind > DGB_FIELD_FUNCTION || f.kind < 0) {
    throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, std::string(name) + ": unknown field kind");
  }
}

// Fills the V2 tensor parameter block from the plan's host tensors (W = kappa Q^T - Q is
// folded per launch) and launches the element-per-thread kernel.
template <int NL, int NQV, int NQE, int BK, int THREADS, int MINB>
void launch_v2(const dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
               const dgb_params* params, dgb_bsr* out, double* const* rhs, int nb, cudaStream_t s,
               int out_row_begin, int out_row_end, const int32_t* row_ptr_src) {
  constexpr bool TRIG = BK == 2;
  constexpr bool FULL = dgb::v2::full_tensors(NL, BK);
  using L = dgb::v2::Lay<NL, NQV, NQE, TRIG>;  // full host-side layout
  using LK = dgb::v2::Lay<NL, NQV, NQE, TRIG, FULL>;  // the kernel's parameter block
  using PT = dgb::v2::Params2<NL, NQV, NQE, TRIG, FULL>;
  using SM = dgb::v2::Smem<NL, NQV, NQE, BK>;
  static_assert(sizeof(PT) <= 32000, "tensor parameter block exceeds the kernel parameter limit");
  constexpr int N2 = NL * NL;
  static thread_local PT P;  // up to ~30 KB: keep it off the stack
  std::memset(&P, 0, sizeof P);
  P.nodes = mesh->nodes;
  P.elements = mesh->elements;
  P.edge_kind = mesh->edge_kind;
  P.edge_elements = mesh->edge_elements;
  P.element_edges = mesh->element_edges;
  if (nb < 1 || nb > dgb::v2::kMaxBatch || (nb > 1 && FULL)) {
    throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "unsupported batch size for this kernel", nb);
  }
  P.n_batch = nb;
  for (int i = 0; i < nb; ++i) {
    P.bt[i].row_ptr = out[i].row_ptr;
    P.bt[i].col = out[i].col;
    P.bt[i].val = out[i].val;
    P.bt[i].rhs = rhs[i];
    P.bt[i].kappa = params[i].kappa;
    P.bt[i].sigma_i = params[i].sigma_interior;
    P.bt[i].sigma_b = params[i].sigma_boundary;
  }
  P.row_ptr_src = row_ptr_src;
  if (row_ptr_src) {
    P.adj_nb = plan->d_adj;
    P.adj_op = plan->d_adj + plan->adj_rows;
    if (plan->d_geo && plan->geo_cache > 0 && plan->bound_nodes == mesh->nodes) P.geo = plan->d_geo;
  }
  P.err_edge = plan->d_err;
  P.diag = plan->d_diag;
  P.epoch = plan->epoch & 0xFFFFFFFFull;
  P.n_elements = mesh->n_elements;
  P.row_begin = out_row_begin;
  P.row_end = out_row_end;
  // P4 only: measured -1.5% on config 5, but +25% on config 3 (whose CTAs start faster from the
  // constant bank than from an L2 round trip)
  P.tr_src = NL == 15 ? plan->d_trace : nullptr;
  P.drop_neumann = params->neumann_inflow == DGB_INFLOW_DROP;
  // auto (-1): evict-first output for odd N2 only (measured, profiles/NOTES.md: P4's 8-byte
  // fragment stores gain 33%; P2's 16-byte fragment stores lose 5%: the L2 must hold a block
  // line until its n-tiles have all landed)
  P.evict_first = plan->l2_policy < 0 ? (N2 % 2 == 1) : (plan->l2_policy & 2) != 0;
  P.ablate = plan->ablate;
  P.load_hints = plan->l2_policy > 0 && (plan->l2_policy & 4) != 0;
  if (NL == 3 && plan->l2_policy < 0 && plan->p1_pipe > 0 && plan->l2_persist_bytes > 0 && row_ptr_src) {
    P.load_hints = 1;  // the P1 persistent kernel's auto policy (bind time): hints, normal output
    P.evict_first = 0;
  }
  if (P.geo) P.load_hints = 0;  // no node gathers left to hint
  P.prob = *problem;
  const double* h = plan->h_tens.data();
  const dgb::Layout& V = plan->L;
  static thread_local std::vector<double> xfull;
  xfull.assign(L::TOTAL, 0.0);
  double* x = xfull.data();
  auto copy = [&](int dst, int src, int n) { std::memcpy(x + dst, h + src, sizeof(double) * n); };
  copy(L::S, V.S, 3 * N2);
  copy(L::M, V.M, N2);
  for (int la = 0; la < 6; ++la) {
    for (int i = 0; i < NL; ++i) {
      for (int j = 0; j < NL; ++j) {
        x[L::W + la * N2 + i * NL + j] =
            params[0].kappa * h[V.Q + la * N2 + j * NL + i] - h[V.Q + la * N2 + i * NL + j];
      }
    }
  }
  if (!TRIG) copy(L::T, V.T, 2 * N2);
  if (L::kHasTA) copy(L::TA, V.TA, 4 * N2);
  if (L::kHasP) std::memcpy(x + L::P, plan->h_P.data(), sizeof(double) * 3 * N2);
  copy(L::PHI, V.PHI, NQV * NL);
  if (TRIG) std::memcpy(x + L::DPHI, plan->h_dphi.data(), sizeof(double) * NQV * 2 * NL);
  copy(L::EPHI, V.EPHI, 3 * NQE * NL);
  copy(L::EDPHI, V.EDPHI, 3 * NQE * 2 * NL);
  for (int lp = 0; lp < 3 * NQE; ++lp) {
    const double w = h[V.EW + lp % NQE];
    for (int a = 0; a < 2 * NL; ++a) x[L::EDW + lp * 2 * NL + a] = w * h[V.EDPHI + lp * 2 * NL + a];
  }
  copy(L::VX, V.VX, NQV);
  copy(L::VY, V.VY, NQV);
  copy(L::VW, V.VW, NQV);
  copy(L::ET, V.ET, NQE);
  copy(L::EW, V.EW, NQE);
  // the compact block is the full one from PHI on (same sections, same order)
  static_assert(LK::TOTAL - LK::PHI == L::TOTAL - L::PHI, "compact layout mismatch");
  std::memcpy(P.t.x, x + (L::PHI - LK::PHI), sizeof(double) * LK::TOTAL);
  const size_t smem = sizeof(double) * (SM::kTr + (THREADS / 32) * SM::kWarp);
  // tensor-core kernel, sets differing only in kappa: one CTA writes every set (FUSE); in the
  // P-form the products are shared too (split tables, kappa applied at the store)
  bool fuse = false, split = false;
  if constexpr (SM::kMma) {
    fuse = nb > 1 && plan->batch_fuse;
    for (int i = 1; i < nb; ++i) {
      fuse = fuse && params[i].sigma_interior == params[0].sigma_interior &&
             params[i].sigma_boundary == params[0].sigma_boundary;
    }
    split = fuse && !SM::kUForm;
  }
  if constexpr (SM::kMma) {
    // B operands in mma.m8n8k4 fragment order: lane (g, t) of tile (ks, nt) holds term 4 ks + t
    // at entry 8 nt + g.  First the diagonal terms (K = 16), then per (l, lf) the five
    // neighbour terms of local edge l against the neighbour's local edge lf (K = 8),
    //   X  = sum_p w_p phi^l_p (x) phi^lf_(n-1-p)      Y_a = sum_p phi^l_p (x) w dphi_a^lf_(n-1-p)
    //   Z_a = kappa sum_p w dphi_a^l_p (x) phi^lf_(n-1-p)
    // (the factored neighbour block of the CUDA-core path, expanded; kappa sits here, not in
    // the per-element A rows, so sets differing only in kappa share one A operand -- FUSE).
    // Built once per (plan, kappa) on the host.
    dgb_plan* mp = const_cast<dgb_plan*>(plan);
    auto ephi = [&](int l, int p, int i) { return x[L::EPHI + (l * NQE + p) * NL + i]; };
    auto edw = [&](int l, int p, int a, int i) { return x[L::EDW + ((l * NQE + p) * 2 + a) * NL + i]; };
    // the neighbour's gradients in its vertex order rotated to (opposite, b, a), the order
    // the kernels build its geometry in (assemble_p1.cuh p1_tables: grad' = M_lf grad)
    auto edw_rot = [&](int lf, int p, int a, int i) {
      const double g0 = edw(lf, p, 0, i), g1 = edw(lf, p, 1, i);
      if (lf == 0) return a == 0 ? g0 : g1;
      if (lf == 1) return a == 0 ? g1 - g0 : -g0;
      return a == 0 ? -g1 : g0 - g1;
    };
    // neighbour term of (l, lf) at entry (bi, bj): 0 X, 1 Y0, 2 Y1, 3 Z0, 4 Z1 (Z unscaled)
    auto neigh = [&](int term, int l, int lf, int bi, int bj) {
      double acc = 0.0;
      for (int p = 0; p < NQE; ++p) {
        const int q = NQE - 1 - p;
        switch (term) {
          case 0: acc += x[L::EW + p] * ephi(l, p, bi) * ephi(lf, q, bj); break;
          case 1: acc += ephi(l, p, bi) * edw_rot(lf, q, 0, bj); break;
          case 2: acc += ephi(l, p, bi) * edw_rot(lf, q, 1, bj); break;
          case 3: acc += edw(l, p, 0, bi) * ephi(lf, q, bj); break;
          default: acc += edw(l, p, 1, bi) * ephi(lf, q, bj); break;
        }
      }
      return acc;
    };
    // diagonal term k at entry n for this kappa
    auto diag = [&](int k, int n, double kap) -> double {
      const int bi = n / NL, bj = n % NL;
      const int kw = SM::kWRow;
      if (k < 3) return x[L::S + k * N2 + n];
      if (k == 3) return x[L::M + n];
      if (SM::kTForm && k < kw) {  // TQ[q][a] = phi_q (x) d_a phi_q
        const int q = (k - 4) / 2, a = (k - 4) % 2;
        return plan->h_tens[plan->L.PHI + q * NL + bi] * plan->h_dphi[(q * 2 + a) * NL + bj];
      }
      if (k < 6) return x[L::T + (k - 4) * N2 + n];
      if (k < kw) return x[L::TA + (k - 6) * N2 + n];
      if (k < kw + 6) {  // W = kappa Q^T - Q for this set's kappa
        const int la = k - kw;
        return kap * h[V.Q + la * N2 + bj * NL + bi] - h[V.Q + la * N2 + bi * NL + bj];
      }
      if constexpr (SM::kUForm) {
        const int l = (k - kw - 6) / NQE, p = (k - kw - 6) % NQE;
        return ephi(l, p, bi) * ephi(l, p, bj);  // U[l][p] = phi^l_p (x) phi^l_p
      }
      return x[L::P + (k - kw - 6) * N2 + n];
    };
    // fragment-order position i of a [ks][nt][lane] table -> (k, n)
    auto kn = [&](int r, int& k, int& n) {
      const int ln = r & 31, tile = r >> 5;
      const int ks = tile / SM::kNT, nt = tile - ks * SM::kNT;
      k = 4 * ks + (ln & 3);
      n = 8 * nt + (ln >> 2);
    };
    auto upload = [&](const std::vector<double>& hb, double key) {
      double* frag = nullptr;
      cuda_check(cudaMalloc(&frag, hb.size() * sizeof(double)), "cudaMalloc(bfrag)");
      cuda_check(cudaMemcpyAsync(frag, hb.data(), hb.size() * sizeof(double),
                                 cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(bfrag)");
      cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(bfrag)");
      mp->bfrag_cache.emplace_back(key, frag);
      return frag;
    };
    auto cached = [&](double key) -> double* {
      for (auto& c : mp->bfrag_cache) {
        if (c.first == key) return c.second;
      }
      return nullptr;
    };
    if (split) {
      // fused P-form batch: [diag, kappa = 0][diag kappa coefficient: Q^T at rows 4..11]
      // [per (l, lf): k-step 0 = X Y0 Y1 0, k-step 1 = Z0 Z1 0 0]
      const double key = std::numeric_limits<double>::infinity();
      double* frag = cached(key);
      if (!frag) {
        const int nq = 2 * SM::kNT * 32, nn = 2 * SM::kNT * 32;
        std::vector<double> hb(SM::kFragTile + nq + 9 * nn, 0.0);
        for (int i = 0; i < SM::kFragTile; ++i) {
          int k, n;
          kn(i, k, n);
          if (k < SM::kTerms && n < N2) hb[i] = diag(k, n, 0.0);
        }
        for (int i = 0; i < nq; ++i) {
          int k, n;
          kn(i, k, n);
          k += 4;  // k-steps 1 and 2 of the diagonal operand
          const int la = k - SM::kWRow;
          if (n < N2 && la >= 0 && la < 6) hb[SM::kFragTile + i] = h[V.Q + la * N2 + (n % NL) * NL + n / NL];
        }
        for (int w = 0; w < 9; ++w) {
          for (int i = 0; i < nn; ++i) {
            int k, n;
            kn(i, k, n);
            const int term = k < 4 ? (k < 3 ? k : -1) : (k - 4 < 2 ? 3 + (k - 4) : -1);
            if (n < N2 && term >= 0) {
              hb[SM::kFragTile + nq + w * nn + i] = neigh(term, w / 3, w % 3, n / NL, n % NL);
            }
          }
        }
        frag = upload(hb, key);
      }
      for (int bi_ = 0; bi_ < nb; ++bi_) P.bt[bi_].bfrag = frag;
    } else {
    for (int bi_ = 0; bi_ < nb; ++bi_) {
    const double kap = params[bi_].kappa;
    double* frag = cached(kap);
    if (!frag) {  // first assembly with this kappa: build and upload (stream-ordered) once
      std::vector<double> hb(SM::kBt, 0.0);
      for (int i = 0; i < SM::kBt; ++i) {
        const bool dg = i < SM::kFragTile;
        const int which = dg ? 0 : 1 + (i - SM::kFragTile) / SM::kOffTile;  // 1 + l * 3 + lf
        int k, n;
        kn(dg ? i : (i - SM::kFragTile) % SM::kOffTile, k, n);
        if (k >= (dg ? SM::kTerms : SM::kOffT) || n >= N2) continue;
        const int bi = n / NL, bj = n % NL;
        if (which == 0) {
          // diagonal terms: S0 S1 S2 M T0 T1 [TA0..3] W[6] then P[3] (P-form) / U[3][NQE] (U-form)
          hb[i] = diag(k, n, kap);
        } else {
          // neighbour terms of (l, lf): P-form X Y0 Y1 Z0 Z1; U-form X[p] (per point) Y0 Y1 Z0 Z1
          const int l = (which - 1) / 3, lf = (which - 1) % 3;
          int term = k;
          if constexpr (SM::kUForm) {
            if (k < NQE) {
              hb[i] = ephi(l, k, bi) * ephi(lf, NQE - 1 - k, bj);  // X[p], point weight in cV
              continue;
            }
            term = k - NQE + 1;  // Y0 Y1 Z0 Z1 as terms 1..4
          }
          const double acc = neigh(term, l, lf, bi, bj);
          hb[i] = term >= 3 ? kap * acc : acc;
        }
      }
      frag = upload(hb, kap);
    }
    P.bt[bi_].bfrag = frag;
    }
    }
  }
  auto kernel = dgb::v2::assemble_kernel<NL, NQV, NQE, BK, THREADS, MINB>;
  if (fuse) kernel = dgb::v2::assemble_kernel<NL, NQV, NQE, BK, THREADS, MINB, true>;
  size_t smem_bytes = smem;
  if constexpr (NL == 3 && BK == 0) {
    // P1, constant velocity: the stash-free kernel (assemble_p1.cuh); option MIN_BLOCKS = 11
    // selects the general kernel for comparison
    if (plan->minblocks != 11) {
      using SP = dgb::v2::SmemP1<NQV, NQE>;
      kernel = row_ptr_src ? dgb::v2::assemble_p1_kernel<NQV, NQE, THREADS, MINB, true>
                           : dgb::v2::assemble_p1_kernel<NQV, NQE, THREADS, MINB, false>;
      smem_bytes = sizeof(double) * (SP::kTr + (THREADS / 32) * SP::kWarp);
    }
  }
  {  // every kernel this instantiation may launch
    const size_t bytes = std::max(smem_bytes, smem);
    dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(dgb::v2::assemble_kernel<NL, NQV, NQE, BK, THREADS, MINB>),
                             bytes, "cudaFuncSetAttribute(v2)");
    if constexpr (SM::kMma) {
      dgb::ensure_dynamic_smem(
          reinterpret_cast<const void*>(dgb::v2::assemble_kernel<NL, NQV, NQE, BK, THREADS, MINB, true>), bytes,
          "cudaFuncSetAttribute(v2 fused)");
    }
    if constexpr (NL == 3 && BK == 0) {
      dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(dgb::v2::assemble_p1_kernel<NQV, NQE, THREADS, MINB, true>),
                               bytes, "cudaFuncSetAttribute(p1)");
      dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(dgb::v2::assemble_p1_kernel<NQV, NQE, THREADS, MINB, false>),
                               bytes, "cudaFuncSetAttribute(p1)");
    }
  }
  const int grid = (out_row_end - out_row_begin + THREADS - 1) / THREADS;
  // Keep the node coordinates (gathered by every element and its neighbours, in random order
  // for permuted meshes) persisting in L2 while the output streams through with evict-first.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, fuse ? 1 : nb);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem_bytes;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  int nattr = 0;
  const size_t node_bytes = sizeof(double) * 2 * static_cast<size_t>(mesh->n_nodes);
  if (plan->l2_policy > 0 && (plan->l2_policy & 1) && plan->l2_persist_bytes > 0 && node_bytes > 0) {
    attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[0].val.accessPolicyWindow.base_ptr = const_cast<double*>(mesh->nodes);
    attr[0].val.accessPolicyWindow.num_bytes = std::min(node_bytes, plan->l2_window_max);
    attr[0].val.accessPolicyWindow.hitRatio =
        static_cast<float>(std::min(1.0, double(plan->l2_persist_bytes) /
                                             double(attr[0].val.accessPolicyWindow.num_bytes)));
    attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    nattr = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = nattr;
  if constexpr (SM::kMma && !SM::kUForm) {
    // P-form tensor-core kernel on a bound mesh: the warp-specialised persistent kernel
    // (assemble_ws.cuh), one CTA per SM
    // measured (profiles/NOTES.md): the split pays off for fused batches only so far
    if (plan->warp_specialized > 0 && row_ptr_src && (fuse || plan->warp_specialized > 1)) {
      if (plan->sm_count <= 0) {
        int dev = 0, n = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
        const_cast<dgb_plan*>(plan)->sm_count = n;
      }
      const int n_chunks = (out_row_end - out_row_begin + 31) / 32;
      cfg.gridDim = dim3(std::max(1, std::min(plan->sm_count, n_chunks)), 1);
      // producer : consumer warps (16 per CTA): option value 1 = the default per batch kind
      // measured on config 2 (profiles/NOTES.md): 8 producers + 4 consumers (12 warps at 146
      // registers) beats every 16-warp split at 128 registers (best 10 / 6)
      const int np = plan->warp_specialized == 1 ? 804 : plan->warp_specialized;
      auto launch = [&](auto tag, auto ctag) {
        constexpr int NPW = decltype(tag)::value, NCW = decltype(ctag)::value;
        using WS = dgb::v2::SmemWs<NL, NQV, NQE, NPW, NCW>;
        auto wk = fuse ? dgb::v2::assemble_ws_kernel<NL, NQV, NQE, true, NPW, NCW>
                       : dgb::v2::assemble_ws_kernel<NL, NQV, NQE, false, NPW, NCW>;
        dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(wk), WS::kBytes, "cudaFuncSetAttribute(ws)");
        cfg.blockDim = dim3(WS::kThreads);
        cfg.dynamicSmemBytes = WS::kBytes;
        cuda_check(cudaLaunchKernelEx(&cfg, wk, P), "cudaLaunchKernelEx(ws)");
      };
#ifdef DGB_TUNING
      if constexpr (NL == 6 && NQV == 7) {  // config 2's kernel: producer share tunable
        // n (4..12): n producers of 16 warps; 100 p + c: p producers, c consumers
        switch (np) {
          case 4: launch(std::integral_constant<int, 4>{}, std::integral_constant<int, 12>{}); break;
          case 6: launch(std::integral_constant<int, 6>{}, std::integral_constant<int, 10>{}); break;
          case 8: launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{}); break;
          case 12: launch(std::integral_constant<int, 12>{}, std::integral_constant<int, 4>{}); break;
          case 1105: launch(std::integral_constant<int, 11>{}, std::integral_constant<int, 5>{}); break;
          case 1206: launch(std::integral_constant<int, 12>{}, std::integral_constant<int, 6>{}); break;
          case 1406: launch(std::integral_constant<int, 14>{}, std::integral_constant<int, 6>{}); break;
          case 804: launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{}); break;
          case 903: launch(std::integral_constant<int, 9>{}, std::integral_constant<int, 3>{}); break;
          case 705: launch(std::integral_constant<int, 7>{}, std::integral_constant<int, 5>{}); break;
          default: launch(std::integral_constant<int, 10>{}, std::integral_constant<int, 6>{}); break;
        }
      } else {
        launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{});
      }
#else
      // the shipped split (profiles/NOTES.md): 8 producer + 4 consumer warps for config 2's
      // kernel, 8 + 8 for the other P-form shapes
      (void)np;
      if constexpr (NL == 6 && NQV == 7) {
        launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 4>{});
      } else {
        launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 8>{});
      }
#endif
      return;
    }
  }
  if constexpr (NL == 3 && BK == 0) {
    // P1 on a bound mesh: the persistent software-pipelined kernel (assemble_p1.cuh)
    if (plan->p1_pipe > 0 && row_ptr_src && plan->minblocks != 11) {
      if (plan->sm_count <= 0) {
        int dev = 0, n = 0;
        cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
        cuda_check(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev), "sm count");
        const_cast<dgb_plan*>(plan)->sm_count = n;
      }
      auto launch = [&](auto tag, auto geo_tag, auto src_tag) {
        constexpr int W = decltype(tag)::value;
        constexpr bool GEO = decltype(geo_tag)::value;
        constexpr int SRC = decltype(src_tag)::value;
        using PS = dgb::v2::SmemP1Pipe<NQV, NQE, W, GEO>;
        auto pk = dgb::v2::assemble_p1_pipe_kernel<NQV, NQE, W, GEO, SRC>;
        dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(pk), PS::kBytes, "cudaFuncSetAttribute(p1 pipe)");
        const int n_chunks = (out_row_end - out_row_begin + 31) / 32;
        cfg.gridDim = dim3(std::max(1, std::min(plan->sm_count, n_chunks)), nb);
        cfg.blockDim = dim3(32 * W);
        cfg.dynamicSmemBytes = PS::kBytes;
        cuda_check(cudaLaunchKernelEx(&cfg, pk, P), "cudaLaunchKernelEx(p1 pipe)");
      };
      // 12 warps per CTA (one CTA per SM) at 166 registers.  Registers are allocated per SM
      // sub-partition, so 13-15 warps get 128 like 16; 16 warps spilled and measured slower
      // (1.103 vs 1.073 ms) and was removed.
      // (the kernel with the geometry record is specialised by source family: only that family's
      // point loop is compiled in)
      using W12 = std::integral_constant<int, 12>;
      if (P.geo) {
        switch (dgb::source_only(problem->source)) {
          case dgb::SRC_CONST: launch(W12{}, std::true_type{}, std::integral_constant<int, dgb::SRC_CONST>{}); break;
          case dgb::SRC_SIN_SIN: launch(W12{}, std::true_type{}, std::integral_constant<int, dgb::SRC_SIN_SIN>{}); break;
          case dgb::SRC_GAUSSIAN: launch(W12{}, std::true_type{}, std::integral_constant<int, dgb::SRC_GAUSSIAN>{}); break;
          default: launch(W12{}, std::true_type{}, std::integral_constant<int, dgb::SRC_ANY>{}); break;
        }
      } else {
        launch(W12{}, std::false_type{}, std::integral_constant<int, dgb::SRC_ANY>{});
      }
      return;
    }
  }
  cuda_check(cudaLaunchKernelEx(&cfg, kernel, P), "cudaLaunchKernelEx(v2)");
}

// Specialised element-per-thread kernels by (n_local, nq_vol, nq_edge, velocity kind), with
// CTA sizes / register budgets chosen by measurement (profiles/NOTES.md); returns false when
// no specialisation exists (the generic kernel runs instead).
bool try_launch_v2(const dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                   const dgb_params* params, dgb_bsr* out, double* const* rhs, int nb, cudaStream_t s,
                   int rb, int re, const int32_t* src) {
  if (plan->force_generic) return false;
  const int bk = problem->advection.kind;
  const int key = plan->nl * 10000 + plan->nqv * 100 + plan->nqe;
  const int mb = plan->minblocks;
#define DGB_V2(NL_, NQV_, NQE_, BK_, T_, MB_)                                               \
  if (key == NL_ * 10000 + NQV_ * 100 + NQE_ && bk == BK_) {                              \
    launch_v2<NL_, NQV_, NQE_, BK_, T_, MB_>(plan, mesh, problem, params, out, rhs, nb, s, rb, re, src); \
    return true;                                                                           \
  }
#ifdef DGB_TUNING
  if (mb == 3) {  // tuning variants of the headline kernels: smaller CTAs (shorter tail)
    DGB_V2(6, 7, 3, 0, 64, 6)
    DGB_V2(3, 6, 2, 0, 64, 8)
  }
  if (mb == 5) {  // register-capped variants (more resident warps)
    DGB_V2(6, 7, 3, 0, 128, 5)
    DGB_V2(3, 6, 2, 0, 128, 5)
  }
  if (mb == 6) {
    DGB_V2(6, 7, 3, 0, 128, 6)
    DGB_V2(3, 6, 2, 0, 128, 6)
  }
#endif
  DGB_V2(3, 6, 2, 0, 128, 4)
  DGB_V2(3, 6, 2, 1, 128, 4)
  DGB_V2(3, 6, 2, 2, 128, 4)
  DGB_V2(6, 7, 3, 0, 128, 4)
  DGB_V2(6, 12, 3, 0, 128, 4)
  DGB_V2(15, 19, 5, 2, 64, 3)   // P4, trigonometric velocity (config 5)
  DGB_V2(10, 16, 4, 0, 128, 3)  // measured: 168 registers, 12 warps/SM (C3 81% of roofline)
  DGB_V2(10, 16, 4, 1, 128, 3)
#undef DGB_V2
  return false;
}

// Device allocations freed on scope exit (dgb_assemble_all_host).
struct Buffers {
  std::vector<void*> ptrs;
  ~Buffers() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <typename T>
  T* alloc(size_t n) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)), "cudaMalloc");
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

// Per-device state of the host-buffer entry point (dgb_assemble_all_host): its stream, the
// plan of the last reference tables seen, and device buffers grown on demand, so a repeated
// call costs the copies and the assembly only.  Lives until process exit (never freed: the
// CUDA context may already be gone at static destruction).
struct HostContext {
  std::mutex mu;
  cudaStream_t s = nullptr;
  dgb_plan* plan = nullptr;
  std::vector<double> key;  // reference-table contents the plan was built from
  std::vector<void*> ptr;
  std::vector<size_t> cap;

  cudaStream_t stream() {
    if (!s) cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    return s;
  }
  void* buffer(int i, size_t bytes) {
    if (static_cast<int>(ptr.size()) <= i) {
      ptr.resize(i + 1, nullptr);
      cap.resize(i + 1, 0);
    }
    bytes = std::max<size_t>(bytes, 16);
    if (cap[i] < bytes) {
      if (ptr[i]) cuda_check(cudaFree(ptr[i]), "cudaFree");
      ptr[i] = nullptr;
      cap[i] = 0;
      cuda_check(cudaMalloc(&ptr[i], bytes), "cudaMalloc");
      cap[i] = bytes;
    }
    return ptr[i];
  }
  dgb_plan* plan_for(const dgb_reference_tables* t, int device) {
    std::vector<double> k = {double(t->degree), double(t->n_local), double(t->nq_vol),
                             double(t->nq_edge)};
    auto add = [&](const double* p, size_t n) {
      if (p) k.insert(k.end(), p, p + n);
    };
    const size_t nl = t->n_local, nq = t->nq_vol, ne = t->nq_edge;
    add(t->vol_x, nq);
    add(t->vol_y, nq);
    add(t->vol_w, nq);
    add(t->edge_t, ne);
    add(t->edge_w, ne);
    add(t->phi, nq * nl);
    add(t->dphi, nq * nl * 2);
    add(t->edge_phi, 6 * ne * nl);
    add(t->edge_dphi, 6 * ne * nl * 2);
    if (plan && k == key) return plan;
    if (plan) dgb_plan_destroy(plan);
    plan = nullptr;
    const int pc = dgb_plan_create(t, device, &plan);
    if (pc != DGB_OK) throw dgb::Error(pc, dgb_last_error_message(), dgb_last_error_detail());
    key = std::move(k);
    return plan;
  }
};

HostContext& host_context(int device) {
  static std::mutex mu;
  static std::vector<HostContext*> ctx;
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "negative device");
  if (static_cast<int>(ctx.size()) <= device) ctx.resize(device + 1, nullptr);
  if (!ctx[device]) ctx[device] = new HostContext();
  return *ctx[device];
}

// row_ptr of block rows [row_begin, row_end): counts (1 + #interior local edges) then an
// inclusive scan (3 launches).
void compute_pattern(dgb_plan* plan, const dgb_mesh_arrays* mesh, int row_begin, int row_end,
                     int32_t* row_ptr, cudaStream_t s) {
  const int E = row_end - row_begin;
  dgb::count_blocks_kernel<<<(E + 255) / 256, 256, 0, s>>>(mesh->edge_kind, mesh->element_edges,
                                                           row_begin, E, row_ptr);
  cuda_check(cudaGetLastError(), "count_blocks_kernel");
  if (plan->scan_n != E) {
    size_t bytes = 0;
    cub::DeviceScan::InclusiveSum(nullptr, bytes, row_ptr + 1, row_ptr + 1, E, s);
    if (bytes > plan->scan_bytes) {
      cudaFree(plan->d_scan);
      plan->d_scan = nullptr;
      cuda_check(cudaMalloc(&plan->d_scan, bytes), "cudaMalloc(scan)");
      plan->scan_bytes = bytes;
    }
    plan->scan_n = E;
  }
  size_t bytes = plan->scan_bytes;
  cuda_check(cub::DeviceScan::InclusiveSum(plan->d_scan, bytes, row_ptr + 1, row_ptr + 1, E, s),
             "DeviceScan");
}

// Nonlinear reaction (H, HJ): B fragments of Phi_q,(i,j) = phi_qj * phi_qi, built on first use.
void nonlinear_frag(dgb_plan* plan, cudaStream_t s) {
  if (plan->d_nlfrag) return;
  const int nl = plan->nl, nq = plan->nqv, n2 = nl * nl;
  const int ks = (nq + 3) / 4, nt = (n2 + 7) / 8;
  std::vector<double> hb(static_cast<size_t>(ks) * nt * 32, 0.0);
  const double* phi = plan->h_tens.data() + plan->L.PHI;
  for (size_t idx = 0; idx < hb.size(); ++idx) {
    const int ln = static_cast<int>(idx & 31), tile = static_cast<int>(idx >> 5);
    const int k = 4 * (tile / nt) + (ln & 3), n = 8 * (tile % nt) + (ln >> 2);
    if (k < nq && n < n2) {
      const int i = n / nl, j = n % nl;
      hb[idx] = phi[k * nl + j] * phi[k * nl + i];  // the reference's rounded product (nonlinear.cpp:61)
    }
  }
  cuda_check(cudaMalloc(&plan->d_nlfrag, hb.size() * sizeof(double)), "cudaMalloc(nlfrag)");
  cuda_check(cudaMemcpyAsync(plan->d_nlfrag, hb.data(), hb.size() * sizeof(double),
                             cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(nlfrag)");
  cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(nlfrag)");
  plan->nl_ks = ks;
}

template <int NL>
void launch_nonlinear(const dgb::nlr::NlParams& P, cudaStream_t s) {
  constexpr int kThreads = 128;
  const size_t smem = sizeof(double) * (((P.nq * NL + 1) & ~1) + ((P.nq + 1) & ~1) +
                                        (kThreads / 32) * (4 * P.ks * dgb::nlr::kCT + 32 * NL));
  auto kernel = dgb::nlr::nonlinear_kernel<NL>;
  dgb::ensure_dynamic_smem(reinterpret_cast<const void*>(kernel), std::max<size_t>(smem, 48 * 1024),
                           "cudaFuncSetAttribute(nonlinear)");
  const int grid = (P.n_elements + kThreads - 1) / kThreads;
  kernel<<<grid, kThreads, smem, s>>>(P);
  cuda_check(cudaGetLastError(), "nonlinear_kernel");
}

}  // namespace

extern "C" {

int dgb_plan_bind_mesh(dgb_plan* plan, const dgb_mesh_arrays* mesh, int32_t row_begin,
                       int32_t row_end, void* stream) {
  return dgb::guarded([&] {
    if (!plan || !mesh) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    if (row_begin < 0 || row_end > mesh->n_elements || row_begin > row_end) {
      throw dgb::Error(DGB_STATUS_INVALID_INDEX, "block row range outside the mesh", row_begin);
    }
    DeviceGuard guard(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t need = static_cast<size_t>(row_end - row_begin) + 1;
    if (need > plan->pattern_cap) {
      cudaFree(plan->d_pattern);
      plan->d_pattern = nullptr;
      cuda_check(cudaMalloc(&plan->d_pattern, need * sizeof(int32_t)), "cudaMalloc(pattern)");
      plan->pattern_cap = need;
    }
    const size_t rows = static_cast<size_t>(row_end - row_begin);
    if (rows > plan->adj_cap) {
      cudaFree(plan->d_adj);
      plan->d_adj = nullptr;
      cuda_check(cudaMalloc(&plan->d_adj, 2 * rows * sizeof(int4)), "cudaMalloc(adjacency)");
      plan->adj_cap = rows;
    }
    plan->adj_rows = rows;
    if (row_end > row_begin) {
      compute_pattern(plan, mesh, row_begin, row_end, plan->d_pattern, s);
      dgb::adjacency_kernel<<<(row_end - row_begin + 255) / 256, 256, 0, s>>>(
          mesh->elements, mesh->edge_kind, mesh->edge_elements, mesh->element_edges, row_begin,
          row_end - row_begin, plan->d_adj, plan->d_adj + rows);
      cuda_check(cudaGetLastError(), "adjacency_kernel");
    } else {
      cuda_check(cudaMemsetAsync(plan->d_pattern, 0, sizeof(int32_t), s), "cudaMemsetAsync");
    }
    // P1 persistent kernel: the rows' geometry record in chunk order (128 B per element)
    plan->bound_nodes = nullptr;
    const bool want_geo = plan->nl == 3 && plan->p1_pipe > 0 && plan->geo_cache > 0 && rows > 0;
    if (want_geo) {
      const size_t padded = (rows + 31) & ~size_t(31);
      if (padded > plan->geo_cap) {
        cudaFree(plan->d_geo);
        plan->d_geo = nullptr;
        plan->geo_cap = 0;
        cuda_check(cudaMalloc(&plan->d_geo, padded * dgb::v2::kGeoRows * sizeof(double2)), "cudaMalloc(geometry)");
        plan->geo_cap = padded;
      }
      dgb::geometry_kernel<<<static_cast<unsigned>((padded + 255) / 256), 256, 0, s>>>(
          mesh->nodes, mesh->elements, plan->d_adj, plan->d_adj + rows, row_begin, row_end - row_begin,
          plan->d_geo);
      cuda_check(cudaGetLastError(), "geometry_kernel");
      plan->bound_nodes = mesh->nodes;
    } else if (plan->d_geo) {
      cudaFree(plan->d_geo);
      plan->d_geo = nullptr;
      plan->geo_cap = 0;
    }
    {
      // L2 policy: permuted (gather-heavy) meshes keep their nodes persisting in L2; the
      // carve-out is sized to the node array, never more (it is taken from the write stream).
      // auto (-1) for the P1 persistent kernel: node gathers evict-last in a carve-out of at
      // most 56 MiB (a carve-out of the whole 67 MB node array at config 4 costs 50%; 48-56
      // MiB halves the DRAM reads and gains 3%, profiles/NOTES.md)
      const size_t node_bytes = sizeof(double) * 2 * static_cast<size_t>(mesh->n_nodes);
      // (with the vertex coordinates bound there are no node gathers to keep resident)
      const bool p1_auto = plan->l2_policy < 0 && plan->nl == 3 && plan->p1_pipe > 0 && !want_geo;
      size_t want = (plan->l2_policy > 0 && (plan->l2_policy & 5)) || p1_auto
                        ? std::min(node_bytes, plan->l2_persist_max) : 0;
      if (p1_auto) want = std::min(want, size_t(56) << 20);
      if (want > 0 && plan->l2_carve_mb > 0) want = std::min(want, size_t(plan->l2_carve_mb) << 20);
      plan->l2_persist_bytes = 0;
      if (want == 0 && plan->carve_held) {
        carve_release(plan->device);
        plan->carve_held = false;
      }
      if (want > 0) {
        const size_t cur = carve_acquire(plan->device, want, plan->carve_held);
        plan->carve_held = true;
        plan->l2_persist_bytes = std::min(cur, want);
      }
    }
    plan->bound_ee = mesh->element_edges;
    plan->bound_kind = mesh->edge_kind;
    plan->bound_elements = mesh->elements;
    plan->bound_edge_elements = mesh->edge_elements;
    plan->bound_n = mesh->n_elements;
    plan->bound_begin = row_begin;
    plan->bound_end = row_end;
  });
}

int dgb_plan_unbind_mesh(dgb_plan* plan) {
  if (!plan) return DGB_STATUS_INVALID_ARGUMENT;
  plan->bound_ee = plan->bound_kind = plan->bound_nodes = nullptr;
  plan->bound_n = plan->bound_begin = plan->bound_end = -1;
  return DGB_OK;
}

int32_t dgb_plan_launch_count(const dgb_plan* plan) { return plan ? plan->last_launches : -1; }

int dgb_plan_create(const dgb_reference_tables* tables, int32_t device, dgb_plan** out) {
  *out = nullptr;
  return dgb::guarded([&] {
    validate_tables(tables);
    DeviceGuard guard(device);
    auto* p = new dgb_plan();
    try {
      p->device = device;
      p->degree = tables->degree;
      p->nl = tables->n_local;
      p->nqv = tables->nq_vol;
      p->nqe = tables->nq_edge;
      p->L = dgb::make_layout(p->nl, p->nqv, p->nqe);
      p->R = dgb::make_rec(p->nqv, p->nqe);
      const std::vector<double> h = dgb::build_tensors(*tables, p->L);
      p->h_tens = h;
      {
        const int nl = p->nl, ne = p->nqe, n2 = nl * nl;
        p->h_P.assign(3 * n2, 0.0);
        for (int l = 0; l < 3; ++l) {
          for (int i = 0; i < nl; ++i) {
            for (int j = 0; j < nl; ++j) {
              long double acc = 0;
              for (int q = 0; q < ne; ++q) {
                const double* ph = tables->edge_phi + ((l * 2) * ne + q) * nl;
                acc += static_cast<long double>(tables->edge_w[q]) * ph[i] * ph[j];
              }
              p->h_P[l * n2 + i * nl + j] = static_cast<double>(acc);
            }
          }
        }
        p->h_dphi.assign(static_cast<size_t>(p->nqv) * 2 * nl, 0.0);
        for (int q = 0; q < p->nqv; ++q) {
          for (int a = 0; a < 2; ++a) {
            for (int i = 0; i < nl; ++i) {
              p->h_dphi[(q * 2 + a) * nl + i] = tables->dphi[(q * nl + i) * 2 + a];
            }
          }
        }
      }
      cuda_check(cudaMalloc(&p->d_tens, h.size() * sizeof(double)), "cudaMalloc(tensors)");
      cuda_check(cudaMemcpy(p->d_tens, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice),
                 "cudaMemcpy(tensors)");
      {
        const int nl = p->nl, ne = p->nqe, n = 3 * ne * 3 * nl;
        const dgb::Layout& V = p->L;
        std::vector<double> trh(n);
        for (int i = 0; i < n; ++i) {
          const int j = i % nl, c = (i / nl) % 3, q = (i / (3 * nl)) % ne, l = i / (3 * nl * ne);
          const int lp = l * ne + q;
          const double w = h[V.EW + q];
          const double g0 = w * h[V.EDPHI + (lp * 2) * nl + j];
          const double g1 = w * h[V.EDPHI + (lp * 2 + 1) * nl + j];
          trh[i] = c == 0 ? h[V.EPHI + lp * nl + j]
                   : l == 0 ? (c == 1 ? g0 : g1)
                   : l == 1 ? (c == 1 ? g1 - g0 : -g0)
                            : (c == 1 ? -g1 : g0 - g1);
        }
        cuda_check(cudaMalloc(&p->d_trace, n * sizeof(double)), "cudaMalloc(trace)");
        cuda_check(cudaMemcpy(p->d_trace, trh.data(), n * sizeof(double), cudaMemcpyHostToDevice),
                   "cudaMemcpy(trace)");
      }
      cuda_check(cudaMalloc(&p->d_err, sizeof(unsigned long long)), "cudaMalloc(err)");
      {
        int max_persist = 0, max_window = 0;
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
        p->l2_persist_max = static_cast<size_t>(max_persist);
        p->l2_window_max = static_cast<size_t>(max_window);
        cudaGetLastError();
      }
      cuda_check(cudaMemset(p->d_err, 0, sizeof(unsigned long long)), "cudaMemset(err)");
    } catch (...) {
      dgb_plan_destroy(p);
      throw;
    }
    *out = p;
  });
}

void dgb_plan_destroy(dgb_plan* p) {
  if (!p) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(p->device);
  if (p->carve_held) carve_release(p->device);  // restores the caller's limit with the last one
  cudaFree(p->d_tens);
  cudaFree(p->d_err);
  cudaFree(p->d_scan);
  cudaFree(p->d_pattern);
  cudaFree(p->d_adj);
  cudaFree(p->d_geo);
  for (auto& c : p->bfrag_cache) cudaFree(c.second);
  cudaFree(p->d_nlfrag);
  cudaFree(p->d_trace);
  if (prev >= 0) cudaSetDevice(prev);
  delete p;
}

int dgb_assemble_batch(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                       const dgb_params* params, int32_t n, int32_t row_begin, int32_t row_end,
                       dgb_bsr* outs, double* const* rhs, void* stream) {
  if (!plan || !mesh || !problem || !params || !outs || !rhs || n < 0) {
    return dgb::record_error(DGB_STATUS_INVALID_ARGUMENT, "null argument", -1);
  }
  if (row_begin < 0 || row_end > mesh->n_elements || row_begin > row_end) {
    return dgb::record_error(DGB_STATUS_INVALID_INDEX, "block row range outside the mesh", row_begin);
  }
  const int E = row_end - row_begin;
  bool same_drop = true;
  for (int i = 1; i < n; ++i) same_drop &= params[i].neumann_inflow == params[0].neumann_inflow;
  const bool bound = plan->d_pattern && plan->bound_ee == mesh->element_edges &&
                     plan->bound_elements == mesh->elements &&
                     plan->bound_edge_elements == mesh->edge_elements &&
                     plan->bound_kind == mesh->edge_kind && plan->bound_n == mesh->n_elements &&
                     plan->bound_begin == row_begin && plan->bound_end == row_end;
  // one launch for all parameter sets: the tensor-core P2 kernel on a bound mesh
  const bool one_launch = n > 1 && n <= dgb::v2::kMaxBatch && bound && same_drop && E > 0 &&
                          ((plan->nl == 6 && problem->advection.kind == DGB_VEC_CONSTANT) ||
                           (plan->nl == 10 && plan->nqv == 16 && plan->nqe == 4 &&
                            problem->advection.kind != DGB_VEC_TRIG)) &&
                          !plan->force_generic;
  if (one_launch) {
    // validate exactly as a single assembly would (and reject mismatched outputs)
    for (int i = 0; i < n; ++i) {
      if (!outs[i].row_ptr || !outs[i].col || !outs[i].val || !rhs[i] ||
          outs[i].block_dim != plan->nl || outs[i].n_block_rows != E) {
        return dgb::record_error(DGB_STATUS_DIMENSION_MISMATCH, "BSR output does not match rows / plan", i);
      }
    }
    const int st = dgb::guarded([&] {
      validate_field(problem->diffusion, true, "diffusion");
      validate_field(problem->linear_reaction, true, "linear_reaction");
      validate_field(problem->source, false, "source");
      validate_field(problem->dirichlet, false, "dirichlet");
      validate_field(problem->neumann, false, "neumann");
      if (problem->dirichlet.kind == DGB_FIELD_PER_ELEMENT ||
          problem->neumann.kind == DGB_FIELD_PER_ELEMENT) {
        throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "boundary data cannot be PER_ELEMENT");
      }
      DeviceGuard guard(plan->device);
      cudaStream_t s = static_cast<cudaStream_t>(stream);
      plan->last_status = DGB_OK;
      plan->status_from = ++plan->epoch;
      plan->last_launches = 1;
      if (plan->ev_start) cuda_check(cudaEventRecord(plan->ev_start, s), "cudaEventRecord");
      if (!try_launch_v2(plan, mesh, problem, params, outs, rhs, n, s, row_begin, row_end,
                         plan->d_pattern)) {
        throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "no batched kernel for this plan");
      }
      if (plan->ev_stop) cuda_check(cudaEventRecord(plan->ev_stop, s), "cudaEventRecord");
    });
    if (st != DGB_STATUS_UNSUPPORTED_DEGREE) return st;  // else: the per-set path below
  }
  int launches = 0;
  const unsigned long long from = plan->epoch + 1;
  plan->in_batch = true;
  for (int i = 0; i < n; ++i) {
    const int st = dgb_assemble_rows(plan, mesh, problem, params + i, row_begin, row_end, outs + i,
                                     rhs[i], stream);
    if (st != DGB_OK) {
      plan->in_batch = false;
      return st;
    }
    launches += plan->last_launches;
  }
  plan->in_batch = false;
  plan->status_from = std::min(from, plan->epoch);
  plan->last_launches = launches;
  return DGB_OK;
}

int dgb_assemble_rows(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                      const dgb_params* params, int32_t row_begin, int32_t row_end, dgb_bsr* out,
                      double* rhs, void* stream) {
  return dgb::guarded([&] {
    if (!plan || !mesh || !problem || !params || !out || !rhs) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    }
    validate_field(problem->diffusion, true, "diffusion");
    validate_field(problem->linear_reaction, true, "linear_reaction");
    validate_field(problem->source, false, "source");
    validate_field(problem->dirichlet, false, "dirichlet");
    validate_field(problem->neumann, false, "neumann");
    if (problem->dirichlet.kind == DGB_FIELD_PER_ELEMENT ||
        problem->neumann.kind == DGB_FIELD_PER_ELEMENT) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "boundary data cannot be PER_ELEMENT");
    }
    if (problem->advection.kind < DGB_VEC_CONSTANT || problem->advection.kind > DGB_VEC_TRIG) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "unknown velocity kind");
    }
    if (row_begin < 0 || row_end > mesh->n_elements || row_begin > row_end) {
      throw dgb::Error(DGB_STATUS_INVALID_INDEX, "block row range outside the mesh", row_begin);
    }
    if (out->block_dim != plan->nl || out->n_block_rows != row_end - row_begin) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "BSR output does not match rows / plan");
    }
    DeviceGuard guard(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int E = row_end - row_begin;
    plan->last_status = DGB_OK;
    if (E == 0) {
      cuda_check(cudaMemsetAsync(out->row_ptr, 0, sizeof(int32_t), s), "cudaMemsetAsync");
      return;
    }
    ++plan->epoch;
    if (!plan->in_batch) plan->status_from = plan->epoch;
    const bool bound = plan->d_pattern && plan->bound_ee == mesh->element_edges &&
                       plan->bound_elements == mesh->elements &&
                       plan->bound_edge_elements == mesh->edge_elements &&
                       plan->bound_kind == mesh->edge_kind && plan->bound_n == mesh->n_elements &&
                       plan->bound_begin == row_begin && plan->bound_end == row_end;
    const int32_t* src = nullptr;
    plan->last_launches = 1;
    if (bound) {
      src = plan->d_pattern;
    } else {
      compute_pattern(plan, mesh, row_begin, row_end, out->row_ptr, s);
      plan->last_launches += 3;
    }
    if (plan->ev_start) cuda_check(cudaEventRecord(plan->ev_start, s), "cudaEventRecord");
    double* rhs1[1] = {rhs};
    if (!try_launch_v2(plan, mesh, problem, params, out, rhs1, 1, s, row_begin, row_end, src)) {
      if (src) {
        cuda_check(cudaMemcpyAsync(out->row_ptr, src, sizeof(int32_t) * (E + 1),
                                   cudaMemcpyDeviceToDevice, s), "cudaMemcpyAsync(pattern)");
      }
      dgb::KParams P;
      std::memset(&P, 0, sizeof P);
      P.nodes = mesh->nodes;
      P.elements = mesh->elements;
      P.edge_kind = mesh->edge_kind;
      P.edge_elements = mesh->edge_elements;
      P.element_edges = mesh->element_edges;
      P.n_elements = mesh->n_elements;
      P.row_begin = row_begin;
      P.row_end = row_end;
      P.prob = *problem;
      P.kappa = params->kappa;
      P.sigma_i = params->sigma_interior;
      P.sigma_b = params->sigma_boundary;
      P.drop_neumann = params->neumann_inflow == DGB_INFLOW_DROP;
      P.tens = plan->d_tens;
      P.L = plan->L;
      P.R = plan->R;
      P.nl = plan->nl;
      P.nqv = plan->nqv;
      P.nqe = plan->nqe;
      P.tile = dgb::tile_for(plan->nl);
      P.row_ptr = out->row_ptr;
      P.col = out->col;
      P.val = out->val;
      P.rhs = rhs;
      P.err_edge = plan->d_err;
      P.epoch = plan->epoch & 0xFFFFFFFFull;
      const int n_tiles = (E + P.tile - 1) / P.tile;
      const size_t smem =
          static_cast<size_t>(P.tile) * (plan->R.size + dgb::kGeo) * sizeof(double) +
          static_cast<size_t>(P.tile) * (dgb::kMeta + 4) * sizeof(int) + 16;
      switch (plan->nl) {
        case 3: launch_assemble<3>(P, n_tiles, smem, s); break;
        case 6: launch_assemble<6>(P, n_tiles, smem, s); break;
        case 10: launch_assemble<10>(P, n_tiles, smem, s); break;
        case 15: launch_assemble<15>(P, n_tiles, smem, s); break;
        default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported n_local", plan->nl);
      }
    }
    cuda_check(cudaGetLastError(), "assemble_kernel");
    if (plan->ev_stop) cuda_check(cudaEventRecord(plan->ev_stop, s), "cudaEventRecord");
  });
}

int dgb_assemble(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                 const dgb_params* params, dgb_bsr* out, double* rhs, void* stream) {
  if (mesh && out && out->nnzb != dgb_bsr_nnzb(mesh->n_elements, mesh->n_interior_edges)) {
    return dgb::record_error(DGB_STATUS_DIMENSION_MISMATCH,
                             "DimensionMismatch: BSR output does not match mesh", -1);
  }
  return dgb_assemble_rows(plan, mesh, problem, params, 0, mesh ? mesh->n_elements : 0, out, rhs,
                           stream);
}

int dgb_assemble_terms(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                       const dgb_params* params, int32_t terms, dgb_bsr* out, double* rhs,
                       void* stream) {
  if (!problem) return dgb::record_error(DGB_STATUS_INVALID_ARGUMENT, "null argument", -1);
  if (terms < 0 || terms > DGB_TERM_ALL) {
    return dgb::record_error(DGB_STATUS_INVALID_ARGUMENT, "InvalidArgument: unknown term mask", terms);
  }
  dgb_problem p = *problem;
  auto zero_scalar = [](dgb_scalar_field& f) {
    std::memset(&f, 0, sizeof f);
    f.kind = DGB_FIELD_CONSTANT;
    f.value = 0.0;
  };
  if (!(terms & DGB_TERM_DIFFUSION)) zero_scalar(p.diffusion);
  if (!(terms & DGB_TERM_REACTION)) zero_scalar(p.linear_reaction);
  if (!(terms & DGB_TERM_CONVECTION)) {
    std::memset(&p.advection, 0, sizeof p.advection);
    p.advection.kind = DGB_VEC_CONSTANT;
  }
  return dgb_assemble(plan, mesh, &p, params, out, rhs, stream);
}

int64_t dgb_count_blocks_host(const dgb_mesh_arrays* mesh, int32_t row_begin, int32_t row_end) {
  if (!mesh || row_begin < 0 || row_end > mesh->n_elements || row_begin > row_end) return -1;
  int64_t n = 0;
  for (int32_t e = row_begin; e < row_end; ++e) {
    n += 1;
    for (int l = 0; l < 3; ++l) {
      n += mesh->edge_kind[mesh->element_edges[3 * static_cast<int64_t>(e) + l]] == DGB_EDGE_INTERIOR;
    }
  }
  return n;
}

int dgb_plan_set_kernel_events(dgb_plan* plan, void* start, void* stop) {
  if (!plan) return DGB_STATUS_INVALID_ARGUMENT;
  plan->ev_start = static_cast<cudaEvent_t>(start);
  plan->ev_stop = static_cast<cudaEvent_t>(stop);
  return DGB_OK;
}

#ifdef DGB_TUNING
// Tuning builds only: per-warp timing records of the persistent P1 kernel (4 words per warp:
// globaltimer at entry and exit, SM cycles in between, chunks << 32 | smid); not in the header.
extern "C" int dgb_tuning_set_diag(dgb_plan* plan, void* device_words) {
  if (!plan) return DGB_STATUS_INVALID_ARGUMENT;
  plan->d_diag = static_cast<unsigned long long*>(device_words);
  return DGB_OK;
}
#endif

int dgb_plan_set_option(dgb_plan* plan, int32_t option, int32_t value) {
  if (!plan) return DGB_STATUS_INVALID_ARGUMENT;
  switch (option) {
    case DGB_OPTION_FORCE_GENERIC_KERNEL: plan->force_generic = value; return DGB_OK;
    case DGB_OPTION_MIN_BLOCKS: plan->minblocks = value; return DGB_OK;
    case DGB_OPTION_L2_POLICY: plan->l2_policy = value; return DGB_OK;
    case DGB_OPTION_BATCH_FUSE: plan->batch_fuse = value != 0; return DGB_OK;
    case DGB_OPTION_WARP_SPECIALIZED: plan->warp_specialized = value; return DGB_OK;
    case DGB_OPTION_P1_PIPELINE: plan->p1_pipe = value; return DGB_OK;
    case DGB_OPTION_L2_CARVEOUT_MB: plan->l2_carve_mb = value; return DGB_OK;
    case DGB_OPTION_GEOMETRY_CACHE: plan->geo_cache = value; return DGB_OK;
    // profiling diagnostics (results are WRONG while set): see the header
    case DGB_OPTION_PROFILE_ABLATE:
#ifdef DGB_TUNING
      plan->ablate = value;
      return DGB_OK;
#else
      return dgb::record_error(DGB_STATUS_INVALID_ARGUMENT,
                               "profiling ablations need a tuning build (-DDGB_TUNING)", option);
#endif
    default: return DGB_STATUS_INVALID_ARGUMENT;
  }
}


int dgb_plan_status(dgb_plan* plan, void* stream) {
  return dgb::guarded([&] {
    if (!plan) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null plan");
    DeviceGuard guard(plan->device);
    cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cudaStreamSynchronize");
    unsigned long long w = 0;
    cuda_check(cudaMemcpy(&w, plan->d_err, sizeof w, cudaMemcpyDeviceToHost), "cudaMemcpy(err)");
    const unsigned long long we = w >> 32;
    if (plan->epoch != 0 && we >= (plan->status_from & 0xFFFFFFFFull) &&
        we <= (plan->epoch & 0xFFFFFFFFull)) {
      throw dgb::Error(DGB_STATUS_INFLOW_ON_NEUMANN,
                       "inflow across a Neumann edge: no boundary data to upwind from",
                       static_cast<long long>(0xFFFFFFFFull - (w & 0xFFFFFFFFull)));
    }
  });
}

int dgb_spmv(const dgb_bsr* a, const double* x, double* y, void* stream) {
  return dgb::guarded([&] {
    if (!a || !x || !y) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    if (a->n_block_rows < 0 || a->nnzb < 0) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "negative size");
    dgb::launch_bsr_spmv(a, x, y, static_cast<cudaStream_t>(stream));  // spmv.cu
  });
}

int dgb_assemble_all_host(const dgb_mesh_arrays* mesh, const dgb_reference_tables* tables,
                          const dgb_problem* problem, const dgb_params* params, int32_t device,
                          dgb_bsr* out, double* rhs) {
  return dgb::guarded([&] {
    if (!mesh || !tables || !problem || !params || !out || !rhs) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    }
    DeviceGuard guard(device);
    HostContext& cx = host_context(device);
    std::lock_guard<std::mutex> lock(cx.mu);
    const int E = mesh->n_elements, ne = mesh->n_edges, nn = mesh->n_nodes;
    const int nl = tables->n_local;
    const int64_t nnzb = dgb_bsr_nnzb(E, mesh->n_interior_edges);
    if (out->nnzb != nnzb || out->block_dim != nl || out->n_block_rows != E) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "BSR output does not match mesh / tables");
    }
    cudaStream_t s = cx.stream();
    dgb_plan* plan = cx.plan_for(tables, device);
    // every call uploads its inputs (the caller's arrays may have changed); buffers are reused
    int slot = 0;
    auto up = [&](const void* src, size_t bytes) {
      void* d = cx.buffer(slot++, bytes);
      cuda_check(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D)");
      return d;
    };
    dgb_mesh_arrays dm = *mesh;
    dm.nodes = static_cast<const double*>(up(mesh->nodes, sizeof(double) * 2 * nn));
    dm.elements = static_cast<const int32_t*>(up(mesh->elements, sizeof(int32_t) * 3 * E));
    dm.edges = nullptr;  // (the sorted vertex pairs: no device code reads them, so they stay on the host)
    dm.edge_kind = static_cast<const uint8_t*>(up(mesh->edge_kind, ne));
    dm.edge_elements = static_cast<const int32_t*>(up(mesh->edge_elements, sizeof(int32_t) * 2 * ne));
    dm.element_edges = static_cast<const int32_t*>(up(mesh->element_edges, sizeof(int32_t) * 3 * E));
    dgb_problem dp = *problem;
    dgb_scalar_field* fields[] = {&dp.diffusion, &dp.linear_reaction, &dp.source, &dp.dirichlet,
                                  &dp.neumann};
    for (dgb_scalar_field* f : fields) {
      if (f->kind == DGB_FIELD_PER_ELEMENT && f->per_element) {
        f->per_element = static_cast<const double*>(up(f->per_element, sizeof(double) * E));
      }
    }
    dgb_bsr d;
    d.n_block_rows = E;
    d.block_dim = nl;
    d.nnzb = nnzb;
    d.row_ptr = static_cast<int32_t*>(cx.buffer(slot++, sizeof(int32_t) * (E + 1)));
    d.col = static_cast<int32_t*>(cx.buffer(slot++, sizeof(int32_t) * nnzb));
    d.val = static_cast<double*>(cx.buffer(slot++, sizeof(double) * nnzb * nl * nl));
    double* d_rhs = static_cast<double*>(cx.buffer(slot++, sizeof(double) * E * nl));
    int rc = dgb_plan_bind_mesh(plan, &dm, 0, E, s);  // pattern + adjacency of this mesh
    if (rc != DGB_OK) throw dgb::Error(rc, dgb_last_error_message(), dgb_last_error_detail());
    rc = dgb_assemble(plan, &dm, &dp, params, &d, d_rhs, s);
    if (rc != DGB_OK) throw dgb::Error(rc, dgb_last_error_message(), dgb_last_error_detail());
    rc = dgb_plan_status(plan, s);
    if (rc != DGB_OK) throw dgb::Error(rc, dgb_last_error_message(), dgb_last_error_detail());
    cuda_check(cudaMemcpyAsync(out->row_ptr, d.row_ptr, sizeof(int32_t) * (E + 1), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(out->col, d.col, sizeof(int32_t) * nnzb, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(out->val, d.val, sizeof(double) * nnzb * nl * nl, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(rhs, d_rhs, sizeof(double) * E * nl, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    // the cached plan outlives the call: give the persisting-L2 carve-out back at once, so a
    // host-buffer call never leaves L2 set aside in the caller's process
    if (plan->carve_held) {
      carve_release(plan->device);
      plan->carve_held = false;
      plan->l2_persist_bytes = 0;
    }
  });
}


int dgb_assemble_nonlinear(dgb_plan* plan, const dgb_mesh_arrays* mesh, const double* coef,
                           int64_t n_coef, const dgb_reaction* reaction, double* h,
                           dgb_bsr* hj, void* stream) {
  return dgb::guarded([&] {
    if (!plan || !mesh || !reaction || !h || !hj) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    }
    const int E = mesh->n_elements, nl = plan->nl;
    // the reference's own check (nonlinear.cpp:17-19)
    if (n_coef != static_cast<int64_t>(E) * nl) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "coefficient vector size mismatch");
    }
    if (hj->n_block_rows != E || hj->nnzb != E || hj->block_dim != nl) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "HJ output is not the block diagonal of the mesh");
    }
    if (reaction->kind < DGB_REACTION_ZERO || reaction->kind > DGB_REACTION_CUBIC) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "unknown reaction kind", reaction->kind);
    }
    if (plan->nqv > dgb::nlr::kMaxQ) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "too many volume points", plan->nqv);
    }
    DeviceGuard guard(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (E == 0) {
      if (hj->row_ptr) cuda_check(cudaMemsetAsync(hj->row_ptr, 0, sizeof(int32_t), s), "cudaMemsetAsync");
      return;
    }
    if (!coef || !mesh->nodes || !mesh->elements || !hj->row_ptr || !hj->col || !hj->val) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null array");
    }
    nonlinear_frag(plan, s);
    dgb::nlr::NlParams P;
    P.nodes = mesh->nodes;
    P.elements = mesh->elements;
    // a plan bound to all rows of this mesh (P1: dgb_plan_bind_mesh builds the geometry record)
    P.geo = (plan->d_geo && plan->geo_cache > 0 && plan->bound_nodes == mesh->nodes &&
             plan->bound_elements == mesh->elements && plan->bound_begin == 0 && plan->bound_end == E)
                ? plan->d_geo : nullptr;
    P.coef = coef;
    P.phi = plan->d_tens + plan->L.PHI;
    P.w = plan->d_tens + plan->L.VW;
    P.bfrag = plan->d_nlfrag;
    P.h = h;
    P.val = hj->val;
    P.row_ptr = hj->row_ptr;
    P.col = hj->col;
    P.n_elements = E;
    P.nq = plan->nqv;
    P.ks = plan->nl_ks;
    P.kind = reaction->kind;
    switch (nl) {
      case 1: launch_nonlinear<1>(P, s); break;
      case 3: launch_nonlinear<3>(P, s); break;
      case 6: launch_nonlinear<6>(P, s); break;
      case 10: launch_nonlinear<10>(P, s); break;
      case 15: launch_nonlinear<15>(P, s); break;
      default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported n_local", nl);
    }
    plan->last_launches = 1;
  });
}

int dgb_assemble_nonlinear_host(const dgb_mesh_arrays* mesh, const dgb_reference_tables* tables,
                                const double* coef, int64_t n_coef,
                                const dgb_reaction* reaction, int32_t device, double* h,
                                dgb_bsr* hj) {
  return dgb::guarded([&] {
    if (!mesh || !tables || !reaction || !h || !hj) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    }
    const int E = mesh->n_elements, nl = tables->n_local, nn = mesh->n_nodes;
    if (n_coef != static_cast<int64_t>(E) * nl) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "coefficient vector size mismatch");
    }
    if (hj->n_block_rows != E || hj->nnzb != E || hj->block_dim != nl) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "HJ output is not the block diagonal of the mesh");
    }
    DeviceGuard guard(device);
    HostContext& cx = host_context(device);
    std::lock_guard<std::mutex> lock(cx.mu);
    cudaStream_t s = cx.stream();
    dgb_plan* plan = cx.plan_for(tables, device);
    int slot = 16;  // buffers of its own (the assembly entry point uses the low slots)
    auto up = [&](const void* src, size_t bytes) {
      void* d = cx.buffer(slot++, bytes);
      cuda_check(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, s), "cudaMemcpyAsync(H2D)");
      return d;
    };
    dgb_mesh_arrays dm = *mesh;
    dm.nodes = static_cast<const double*>(up(mesh->nodes, sizeof(double) * 2 * nn));
    dm.elements = static_cast<const int32_t*>(up(mesh->elements, sizeof(int32_t) * 3 * E));
    const double* dcoef = static_cast<const double*>(up(coef, sizeof(double) * n_coef));
    dgb_bsr d = *hj;
    d.row_ptr = static_cast<int32_t*>(cx.buffer(slot++, sizeof(int32_t) * (E + 1)));
    d.col = static_cast<int32_t*>(cx.buffer(slot++, sizeof(int32_t) * E));
    d.val = static_cast<double*>(cx.buffer(slot++, sizeof(double) * E * nl * nl));
    double* dh = static_cast<double*>(cx.buffer(slot++, sizeof(double) * E * nl));
    const int rc = dgb_assemble_nonlinear(plan, &dm, dcoef, n_coef, reaction, dh, &d, s);
    if (rc != DGB_OK) throw dgb::Error(rc, dgb_last_error_message(), dgb_last_error_detail());
    cuda_check(cudaMemcpyAsync(h, dh, sizeof(double) * E * nl, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(hj->row_ptr, d.row_ptr, sizeof(int32_t) * (E + 1), cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(hj->col, d.col, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaMemcpyAsync(hj->val, d.val, sizeof(double) * E * nl * nl, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize");
  });
}


int32_t dgb_l2_quad_order(int32_t degree, int32_t quad_order) {
  auto rule_degree = [](int q) {  // triangle_rule's delivered degree (quadrature.cpp:46-154)
    if (q <= 1) return 1;
    if (q == 3) return 4;
    if (q == 7) return 8;
    return q;
  };
  const int vol = quad_order > 0 ? quad_order : 2 * degree + 2;
  return std::max(2 * degree + 3, rule_degree(vol) + 1);
}

int dgb_l2_error(dgb_plan* plan, const dgb_mesh_arrays* mesh, const double* coef, int64_t n_coef,
                 const dgb_scalar_field* exact, double* out, void* stream) {
  return dgb::guarded([&] {
    if (!plan || !mesh || !exact || !out) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    const int E = mesh->n_elements, nl = plan->nl;
    if (n_coef != static_cast<int64_t>(E) * nl) {
      throw dgb::Error(DGB_STATUS_DIMENSION_MISMATCH, "coefficient vector size mismatch");
    }
    validate_field(*exact, false, "exact");
    if (exact->kind == DGB_FIELD_PER_ELEMENT) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "exact: a point field is required");
    }
    DeviceGuard guard(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    out[0] = out[1] = 0.0;
    if (E == 0) return;
    dgb::post::PostParams P{};
    P.nodes = mesh->nodes;
    P.elements = mesh->elements;
    P.coef = coef;
    P.phi = plan->d_tens + plan->L.PHI;
    P.vx = plan->d_tens + plan->L.VX;
    P.vy = plan->d_tens + plan->L.VY;
    P.vw = plan->d_tens + plan->L.VW;
    P.field = *exact;
    P.n_elements = E;
    P.nq = plan->nqv;
    const int nb = (E + dgb::post::kThreads - 1) / dgb::post::kThreads;
    Buffers buf;
    double* partial = buf.alloc<double>(2 * static_cast<size_t>(nb) + 2);
    P.out = partial;
    switch (nl) {
      case 3: dgb::post::l2_error_kernel<3><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      case 6: dgb::post::l2_error_kernel<6><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      case 10: dgb::post::l2_error_kernel<10><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      case 15: dgb::post::l2_error_kernel<15><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported n_local", nl);
    }
    dgb::post::l2_finish_kernel<<<1, dgb::post::kThreads, 0, s>>>(partial, nb, partial + 2 * nb);
    cuda_check(cudaGetLastError(), "l2_error_kernel");
    double h[2];
    cuda_check(cudaMemcpyAsync(h, partial + 2 * nb, sizeof h, cudaMemcpyDeviceToHost, s), "D2H(l2)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(l2)");
    out[0] = std::sqrt(h[0]);
    out[1] = h[1];
  });
}

int dgb_project(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_scalar_field* f,
                double* coef, void* stream) {
  return dgb::guarded([&] {
    if (!plan || !mesh || !f || !coef) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    validate_field(*f, false, "field");
    if (f->kind == DGB_FIELD_PER_ELEMENT) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "field: a point field is required");
    }
    DeviceGuard guard(plan->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int E = mesh->n_elements;
    if (E == 0) return;
    dgb::post::PostParams P{};
    P.nodes = mesh->nodes;
    P.elements = mesh->elements;
    P.phi = plan->d_tens + plan->L.PHI;
    P.vx = plan->d_tens + plan->L.VX;
    P.vy = plan->d_tens + plan->L.VY;
    P.vw = plan->d_tens + plan->L.VW;
    P.field = *f;
    P.out = coef;
    P.n_elements = E;
    P.nq = plan->nqv;
    const int nb = (E + dgb::post::kThreads - 1) / dgb::post::kThreads;
    switch (plan->nl) {
      case 3: dgb::post::project_kernel<3><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      case 6: dgb::post::project_kernel<6><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      case 10: dgb::post::project_kernel<10><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      case 15: dgb::post::project_kernel<15><<<nb, dgb::post::kThreads, 0, s>>>(P); break;
      default: throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "unsupported n_local", plan->nl);
    }
    cuda_check(cudaGetLastError(), "project_kernel");
  });
}

int dgb_eval_solution(const double* coef, int32_t degree, int32_t n_elements, int64_t n,
                      const int32_t* elements, const double* xhat, const double* yhat,
                      double* values, void* stream) {
  return dgb::guarded([&] {
    if (degree < 1 || degree > 4) {
      throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE, "polynomial degree must be between 1 and 4", degree);
    }
    if (n < 0) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "negative point count");
    if (n == 0) return;
    if (!coef || !elements || !xhat || !yhat || !values) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    Buffers buf;
    unsigned long long* bad = buf.alloc<unsigned long long>(1);
    cuda_check(cudaMemsetAsync(bad, 0xFF, sizeof(unsigned long long), s), "memset");
    const unsigned nb = static_cast<unsigned>((n + dgb::post::kThreads - 1) / dgb::post::kThreads);
    switch (degree) {
      case 1: dgb::post::eval_kernel<1><<<nb, dgb::post::kThreads, 0, s>>>(coef, n_elements, n, elements, xhat, yhat, values, bad); break;
      case 2: dgb::post::eval_kernel<2><<<nb, dgb::post::kThreads, 0, s>>>(coef, n_elements, n, elements, xhat, yhat, values, bad); break;
      case 3: dgb::post::eval_kernel<3><<<nb, dgb::post::kThreads, 0, s>>>(coef, n_elements, n, elements, xhat, yhat, values, bad); break;
      default: dgb::post::eval_kernel<4><<<nb, dgb::post::kThreads, 0, s>>>(coef, n_elements, n, elements, xhat, yhat, values, bad); break;
    }
    cuda_check(cudaGetLastError(), "eval_kernel");
    unsigned long long hb = 0;
    cuda_check(cudaMemcpyAsync(&hb, bad, sizeof hb, cudaMemcpyDeviceToHost, s), "D2H(eval)");
    cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(eval)");
    if (hb != ~0ull) throw dgb::Error(DGB_STATUS_INVALID_INDEX, "element index out of range", static_cast<long long>(hb));
  });
}

}  // extern "C"
