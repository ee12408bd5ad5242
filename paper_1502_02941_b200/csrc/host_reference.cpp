// host_reference.cpp -- reference-element tables for the GPU path.
//
// dgb_reference_create builds the same tables as dgfem::ReferenceElement(degree, quad_order)
// (/root/reference/proj/src/reference.cpp:87-147): the orthonormal Dubiner basis on the unit
// triangle (0,0)-(1,0)-(0,1) (Dubiner 1991; Sherwin & Karniadakis' collapsed-coordinate form),
// the symmetric positive-weight Dunavant rules up to degree 9 (Dunavant 1985; degrees 3 and 7
// served by 4 and 8) and a Duffy-collapsed Gauss rule above, and Gauss-Legendre edge points
// on [0,1] mirrored so t[n-1-q] == 1 - t[q] exactly (quadrature.cpp:46-194).  Point order
// within each rule follows the reference so tables compare entry by entry; tests pin them
// against tables dumped from the reference (tests/golden).
//
// In a drop-in deployment the reference passes its own ReferenceElement tables to
// dgb_plan_create instead; this module makes the repo self-contained.
#include <cmath>
#include <cstdint>
#include <vector>

#include "common.hpp"

struct dgb_reference {
  int degree = 0, nl = 0;
  std::vector<double> vx, vy, vw, et, ew;
  std::vector<double> phi, dphi, edge_phi, edge_dphi;
};

namespace {

struct Rule {
  std::vector<double> x, y, w;
};

void centroid(Rule& r, double w) {
  r.x.push_back(1.0 / 3.0);
  r.y.push_back(1.0 / 3.0);
  r.w.push_back(w);
}

// Barycentric orbit (a, a, 1-2a).
void orbit3(Rule& r, double a, double w) {
  const double c = 1.0 - 2.0 * a;
  const double px[3] = {a, a, c}, py[3] = {c, a, a};
  for (int i = 0; i < 3; ++i) {
    r.x.push_back(px[i]);
    r.y.push_back(py[i]);
    r.w.push_back(w);
  }
}

// Barycentric orbit (a, b, 1-a-b), all six permutations.
void orbit6(Rule& r, double a, double b, double w) {
  const double c = 1.0 - a - b;
  const double px[6] = {b, c, a, c, a, b}, py[6] = {c, b, c, a, b, a};
  for (int i = 0; i < 6; ++i) {
    r.x.push_back(px[i]);
    r.y.push_back(py[i]);
    r.w.push_back(w);
  }
}

// Gauss-Legendre on [0,1] by Newton iteration on P_n from the classical cosine guess.
void gauss01(int n, std::vector<double>& t, std::vector<double>& w) {
  t.assign(n, 0.0);
  w.assign(n, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double x = std::cos(pi * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    const double wi = 2.0 / ((1.0 - x * x) * dp * dp);
    t[n - 1 - i] = 0.5 * (1.0 + x);
    t[i] = 1.0 - t[n - 1 - i];
    w[i] = w[n - 1 - i] = 0.5 * wi;
  }
  if (n % 2 == 1) t[n / 2] = 0.5;
}

Rule triangle_rule(int degree) {
  Rule r;
  switch (degree) {
    case 0:
    case 1:
      centroid(r, 0.5);
      return r;
    case 2:
      orbit3(r, 1.0 / 6.0, 1.0 / 6.0);
      return r;
    case 3:
    case 4:  // Dunavant degree 4, 6 points
      orbit3(r, 0.44594849091596488631832925388305, 0.22338158967801146569500700843312 * 0.5);
      orbit3(r, 0.09157621350977074345957146340220, 0.10995174365532186763832632490021 * 0.5);
      return r;
    case 5:  // degree 5, 7 points
      centroid(r, 0.225 * 0.5);
      orbit3(r, 0.47014206410511508977044120951345, 0.13239415278850618073764938783315 * 0.5);
      orbit3(r, 0.10128650732345633880098736191512, 0.12593918054482715259568394550018 * 0.5);
      return r;
    case 6:  // degree 6, 12 points
      orbit3(r, 0.24928674517091042129163855310702, 0.11678627572637936602528961138558 * 0.5);
      orbit3(r, 0.06308901449150222834033160287082, 0.05084490637020681692093680910686 * 0.5);
      orbit6(r, 0.31035245103378440541660773395655, 0.63650249912139864723014259441205,
             0.08285107561837357519355345642044 * 0.5);
      return r;
    case 7:
    case 8:  // degree 8, 16 points
      centroid(r, 0.14431560767778716825109111048906 * 0.5);
      orbit3(r, 0.17056930775176020662229350149146, 0.10321737053471825028179155029212 * 0.5);
      orbit3(r, 0.05054722831703097545842355059660, 0.03245849762319808031092592834178 * 0.5);
      orbit3(r, 0.45929258829272315602881551449417, 0.09509163426728462479389610438858 * 0.5);
      orbit6(r, 0.26311282963463811342178578628464, 0.72849239295540428124100037917606,
             0.02723031417443499426484469007390 * 0.5);
      return r;
    case 9:  // degree 9, 19 points
      centroid(r, 0.09713579628279609890744676309485 * 0.5);
      orbit3(r, 0.48968251919873762778370692483619, 0.03133470022713983234393199080984 * 0.5);
      orbit3(r, 0.43708959149293663726993036443535, 0.07782754100477543338465495857972 * 0.5);
      orbit3(r, 0.18820353561903273024096128046733, 0.07964773892720910288013526957424 * 0.5);
      orbit3(r, 0.04472951339445297061024247196780, 0.02557767565869810438673914467637 * 0.5);
      orbit6(r, 0.22196298916076569567510252769319, 0.74119859878449802069007987352342,
             0.04328353937728937728937728937729 * 0.5);
      return r;
    default: {  // Duffy-collapsed tensor Gauss rule, exact to any degree
      const int ns = (degree + 2) / 2, nr = (degree + 3) / 2;
      std::vector<double> ts, ws, tr, wr;
      gauss01(ns, ts, ws);
      gauss01(nr, tr, wr);
      for (int j = 0; j < nr; ++j) {
        for (int i = 0; i < ns; ++i) {
          r.x.push_back(ts[i] * (1.0 - tr[j]));
          r.y.push_back(tr[j]);
          r.w.push_back(ws[i] * wr[j] * (1.0 - tr[j]));
        }
      }
      return r;
    }
  }
}

// Orthonormal Dubiner basis of degree k at (x, y): psi_{m,n} = c_mn f_m(u,t) P_n^{(2m+1,0)}(z)
// with u = 2x + y - 1, t = 1 - y, z = 2y - 1, f_m = t^m P_m(u/t) (scaled Legendre, no
// singularity at t = 0), c_mn = sqrt(2(2m+1)(m+n+1)); index (m+n)(m+n+1)/2 + n.
void dubiner(int k, double x, double y, double* val, double* grad) {
  const double u = 2.0 * x + y - 1.0, t = 1.0 - y, z = 2.0 * y - 1.0;
  double f[8], fu[8], ft[8];
  f[0] = 1.0;
  fu[0] = 0.0;
  ft[0] = 0.0;
  if (k >= 1) {
    f[1] = u;
    fu[1] = 1.0;
    ft[1] = 0.0;
  }
  for (int m = 1; m < k; ++m) {
    // (m+1) f_{m+1} = (2m+1) u f_m - m t^2 f_{m-1}
    const double a = 2.0 * m + 1.0;
    f[m + 1] = (a * u * f[m] - m * t * t * f[m - 1]) / (m + 1);
    fu[m + 1] = (a * (f[m] + u * fu[m]) - m * t * t * fu[m - 1]) / (m + 1);
    ft[m + 1] = (a * u * ft[m] - m * (2.0 * t * f[m - 1] + t * t * ft[m - 1])) / (m + 1);
  }
  for (int m = 0; m <= k; ++m) {
    const double al = 2.0 * m + 1.0;
    double gm2 = 0.0, dgm2 = 0.0, gm1 = 1.0, dgm1 = 0.0;
    for (int n = 0; m + n <= k; ++n) {
      double g, dg;
      if (n == 0) {
        g = 1.0;
        dg = 0.0;
      } else if (n == 1) {
        g = 0.5 * ((al + 2.0) * z + al);
        dg = 0.5 * (al + 2.0);
      } else {
        // 2n(n+al)(2n+al-2) P_n = (2n+al-1)((2n+al)(2n+al-2) z + al^2) P_{n-1}
        //                         - 2(n+al-1)(n-1)(2n+al) P_{n-2}
        const double c0 = 2.0 * n * (n + al) * (2.0 * n + al - 2.0);
        const double c1 = 2.0 * n + al - 1.0;
        const double c2 = (2.0 * n + al) * (2.0 * n + al - 2.0);
        const double c3 = 2.0 * (n + al - 1.0) * (n - 1.0) * (2.0 * n + al);
        g = (c1 * ((c2 * z + al * al) * gm1) - c3 * gm2) / c0;
        dg = (c1 * ((c2 * z + al * al) * dgm1 + c2 * gm1) - c3 * dgm2) / c0;
      }
      if (n >= 1) {
        gm2 = gm1;
        dgm2 = dgm1;
      }
      gm1 = g;
      dgm1 = dg;
      const double c = std::sqrt(2.0 * (2.0 * m + 1.0) * (m + n + 1.0));
      const int d = m + n, j = d * (d + 1) / 2 + n;
      if (val) val[j] = c * f[m] * g;
      if (grad) {
        grad[2 * j] = c * 2.0 * fu[m] * g;
        grad[2 * j + 1] = c * ((fu[m] - ft[m]) * g + f[m] * 2.0 * dg);
      }
    }
  }
}

}  // namespace

extern "C" {

int dgb_reference_create(int32_t degree, int32_t quad_order, dgb_reference** out) {
  *out = nullptr;
  return dgb::guarded([&] {
    if (degree < 1 || degree > 4) {
      throw dgb::Error(DGB_STATUS_UNSUPPORTED_DEGREE,
                       "polynomial degree must be between 1 and 4", degree);
    }
    if (quad_order < 0) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "quadrature order must be positive");
    }
    auto* r = new dgb_reference();
    r->degree = degree;
    r->nl = (degree + 1) * (degree + 2) / 2;
    const int exact = quad_order > 0 ? quad_order : 2 * degree + 2;
    const int ne = quad_order > 0 ? (quad_order + 1) / 2 : degree + 1;
    Rule rule = triangle_rule(exact);
    r->vx = rule.x;
    r->vy = rule.y;
    r->vw = rule.w;
    gauss01(ne, r->et, r->ew);
    const int nl = r->nl, nq = static_cast<int>(r->vw.size());
    r->phi.resize(static_cast<std::size_t>(nq) * nl);
    r->dphi.resize(static_cast<std::size_t>(nq) * nl * 2);
    for (int q = 0; q < nq; ++q) {
      dubiner(degree, r->vx[q], r->vy[q], &r->phi[q * nl], &r->dphi[q * nl * 2]);
    }
    // Edge l runs from reference vertex (l+1)%3 to (l+2)%3 (reference.hpp:11-14).
    const double V[3][2] = {{0.0, 0.0}, {1.0, 0.0}, {0.0, 1.0}};
    r->edge_phi.resize(static_cast<std::size_t>(6) * ne * nl);
    r->edge_dphi.resize(static_cast<std::size_t>(6) * ne * nl * 2);
    for (int l = 0; l < 3; ++l) {
      const double* va = V[(l + 1) % 3];
      const double* vb = V[(l + 2) % 3];
      double* p0 = &r->edge_phi[static_cast<std::size_t>(l * 2) * ne * nl];
      double* g0 = &r->edge_dphi[static_cast<std::size_t>(l * 2) * ne * nl * 2];
      for (int q = 0; q < ne; ++q) {
        const double s = r->et[q];
        dubiner(degree, va[0] + s * (vb[0] - va[0]), va[1] + s * (vb[1] - va[1]), &p0[q * nl],
                &g0[q * nl * 2]);
      }
      // orientation 1: the same points traversed backwards (bitwise permutation)
      double* p1 = p0 + static_cast<std::size_t>(ne) * nl;
      double* g1 = g0 + static_cast<std::size_t>(ne) * nl * 2;
      for (int q = 0; q < ne; ++q) {
        const int p = ne - 1 - q;
        for (int j = 0; j < nl; ++j) {
          p1[q * nl + j] = p0[p * nl + j];
          g1[(q * nl + j) * 2] = g0[(p * nl + j) * 2];
          g1[(q * nl + j) * 2 + 1] = g0[(p * nl + j) * 2 + 1];
        }
      }
    }
    *out = r;
  });
}

int dgb_reference_view(const dgb_reference* r, dgb_reference_tables* out) {
  if (!r || !out) return DGB_STATUS_INVALID_ARGUMENT;
  out->degree = r->degree;
  out->n_local = r->nl;
  out->nq_vol = static_cast<int32_t>(r->vw.size());
  out->nq_edge = static_cast<int32_t>(r->ew.size());
  out->vol_x = r->vx.data();
  out->vol_y = r->vy.data();
  out->vol_w = r->vw.data();
  out->edge_t = r->et.data();
  out->edge_w = r->ew.data();
  out->phi = r->phi.data();
  out->dphi = r->dphi.data();
  out->edge_phi = r->edge_phi.data();
  out->edge_dphi = r->edge_dphi.data();
  return DGB_OK;
}

void dgb_reference_free(dgb_reference* r) { delete r; }

}  // extern "C"
