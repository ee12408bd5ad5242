/*
 * dg_coeffs.h -- TEST INFRASTRUCTURE (oracle side).  Host twins of the device coefficient
 * descriptors of include/dgfem_b200.h.  The reference library takes std::function callbacks
 * (problems.hpp:19-68); these plain-C evaluators are what the oracle restatement
 * (dg_oracle.c) calls and what ref_shim.cpp wraps into a dgfem::ProblemSpec, so the
 * reference, the oracle and the CUDA path all see the same coefficient formulas.
 *
 * Nothing in the product links this file.
 */
#ifndef DG_COEFFS_H
#define DG_COEFFS_H

#include <math.h>

#include "../include/dgfem_b200.h"

#define DGC_PI 3.14159265358979323846

/* u, du/dx, du/dy, lap(u) of an analytic family (DGB_FN_*). */
static inline void dgc_family(int fn, const double* p, double x, double y, double* u,
                              double* ux, double* uy, double* lap) {
  switch (fn) {
    case DGB_FN_SIN_SIN: {
      const double sx = sin(DGC_PI * x), sy = sin(DGC_PI * y);
      const double cx = cos(DGC_PI * x), cy = cos(DGC_PI * y);
      *u = p[0] * (sx * sy);
      *ux = p[0] * (DGC_PI * cx * sy);
      *uy = p[0] * (DGC_PI * sx * cy);
      *lap = -2.0 * DGC_PI * DGC_PI * (*u);
      return;
    }
    case DGB_FN_TANH_LAYER: {
      const double s = (p[0] * x + p[1] * y + p[2]) / p[3];
      const double t = tanh(s);
      const double c = cosh(s);
      const double sech2 = 1.0 / (c * c);
      const double gx = p[0] / p[3], gy = p[1] / p[3];
      *u = 0.5 * (1.0 - t);
      *ux = -0.5 * sech2 * gx;
      *uy = -0.5 * sech2 * gy;
      *lap = t * sech2 * (gx * gx + gy * gy);
      return;
    }
    case DGB_FN_GAUSSIAN: {
      const double dx = x - p[1], dy = y - p[2];
      const double r2 = dx * dx + dy * dy;
      const double v = exp(-p[0] * r2);
      *u = v;
      *ux = -2.0 * p[0] * dx * v;
      *uy = -2.0 * p[0] * dy * v;
      *lap = (4.0 * p[0] * p[0] * r2 - 4.0 * p[0]) * v;
      return;
    }
    case DGB_FN_AFFINE:
      *u = p[0] + p[1] * x + p[2] * y;
      *ux = p[1];
      *uy = p[2];
      *lap = 0.0;
      return;
    case DGB_FN_STEP_Y:
      *u = (y < p[0]) ? p[1] : p[2];
      *ux = 0.0;
      *uy = 0.0;
      *lap = 0.0;
      return;
    default:
      *u = *ux = *uy = *lap = NAN;
      return;
  }
}

/* Value of a CONSTANT or FUNCTION scalar field at (x, y). */
static inline double dgc_scalar_point(const dgb_scalar_field* f, double x, double y) {
  if (f->kind == DGB_FIELD_CONSTANT) {
    return f->value;
  }
  double u, ux, uy, lap;
  dgc_family(f->fn, f->p, x, y, &u, &ux, &uy, &lap);
  switch (f->mode) {
    case DGB_MODE_VALUE:
      return u;
    case DGB_MODE_SOURCE:
      return f->q[0] * u - f->q[1] * lap + f->q[2] * ux + f->q[3] * uy;
    case DGB_MODE_SOURCE_SQUARE: /* problems.cpp:113-118: f += val * val */
      return (f->q[0] * u - f->q[1] * lap + f->q[2] * ux + f->q[3] * uy) + u * u;
    case DGB_MODE_FLUX_X:
      return f->q[1] * ux;
    default:
      return NAN;
  }
}

/* Scalar field inside element `elem` (volume points). */
static inline double dgc_scalar_volume(const dgb_scalar_field* f, double x, double y, int elem) {
  if (f->kind == DGB_FIELD_PER_ELEMENT) {
    return f->per_element[elem];
  }
  return dgc_scalar_point(f, x, y);
}

/* Scalar field on an edge with adjacent elements left/right (right < 0 on the boundary);
 * a PER_ELEMENT field takes the average of the two traces on interior edges. */
static inline double dgc_scalar_edge(const dgb_scalar_field* f, double x, double y, int left,
                                     int right) {
  if (f->kind == DGB_FIELD_PER_ELEMENT) {
    return right < 0 ? f->per_element[left]
                     : 0.5 * (f->per_element[left] + f->per_element[right]);
  }
  return dgc_scalar_point(f, x, y);
}

/* Velocity field b(x, y). */
static inline void dgc_vector(const dgb_vector_field* b, double x, double y, double* bx,
                              double* by) {
  switch (b->kind) {
    case DGB_VEC_CONSTANT:
      *bx = b->p[0];
      *by = b->p[1];
      return;
    case DGB_VEC_AFFINE:
      *bx = (b->p[0] + b->p[2] * x) + b->p[3] * y;
      *by = (b->p[1] + b->p[4] * x) + b->p[5] * y;
      return;
    case DGB_VEC_TRIG:
      *bx = cos(b->p[0] * y);
      *by = sin(b->p[1] * x);
      return;
    default:
      *bx = *by = NAN;
      return;
  }
}

/* Nonlinear reaction r(u), r'(u) with the reference's expressions (dgb_reaction kinds:
 * problems.cpp:125-127, test_nonlinear.cpp square / cubic / zero / linear reactions). */
static inline void dgc_reaction(int kind, double u, double* r, double* dr) {
  switch (kind) {
    case DGB_REACTION_LINEAR: *r = u; *dr = 1.0; return;
    case DGB_REACTION_SQUARE: *r = u * u; *dr = 2.0 * u; return;
    case DGB_REACTION_CUBIC: *r = u * u * u; *dr = 3.0 * u * u; return;
    default: *r = 0.0; *dr = 0.0; return;
  }
}

#endif /* DG_COEFFS_H */
