// ref_shim.cpp -- TEST INFRASTRUCTURE.  A C-ABI over the UNMODIFIED reference library
// (/root/reference/proj/src, compiled by oracle/Makefile into oracle/_ref/libdgref.so), used
// to (1) pin the C restatement oracle/dg_oracle.c, (2) generate tests/golden fixtures and
// (3) time the reference's CPU assembly for bench.py's cpu_baseline / --impl reference arm.
//
// Only reference headers are included; no reference source is copied.  The coefficient
// descriptors of include/dgfem_b200.h become std::function callbacks through the host twins
// in dg_coeffs.h (the "device coefficient descriptor with host twins" of SURVEY.md §7).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "dgfem/assembly.hpp"
#include "dgfem/errors.hpp"
#include "dgfem/execution.hpp"
#include "dgfem/mesh.hpp"
#include "dgfem/nonlinear.hpp"
#include "dgfem/postprocess.hpp"
#include "dgfem/problems.hpp"
#include "dgfem/reference.hpp"
#include "dgfem/sparse.hpp"

extern "C" {
#include "dg_coeffs.h"
}

namespace {

thread_local std::string g_message;
thread_local long g_detail = -1;

int fail(const dgfem::Error& e) {
  g_message = e.what();
  g_detail = e.detail();
  return 1 + static_cast<int>(e.code());
}

int fail_other(const std::exception& e) {
  g_message = e.what();
  g_detail = -1;
  return DGB_STATUS_INVALID_ARGUMENT;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_message.clear();
    g_detail = -1;
    return 0;
  } catch (const dgfem::Error& e) {
    return fail(e);
  } catch (const std::exception& e) {
    return fail_other(e);
  }
}

struct MeshHandle {
  dgfem::Mesh mesh;
  std::vector<double> nodes;
  std::vector<int32_t> elements, edges, edge_elements, element_edges;
  std::vector<uint8_t> kind;
  int n_interior = 0;

  void flatten() {
    const auto& m = mesh;
    nodes.resize(2 * m.nodes.size());
    for (std::size_t i = 0; i < m.nodes.size(); ++i) {
      nodes[2 * i] = m.nodes[i].x;
      nodes[2 * i + 1] = m.nodes[i].y;
    }
    elements.resize(3 * m.elements.size());
    element_edges.resize(3 * m.elements.size());
    for (std::size_t e = 0; e < m.elements.size(); ++e) {
      for (int k = 0; k < 3; ++k) {
        elements[3 * e + k] = m.elements[e][k];
        element_edges[3 * e + k] = m.element_edges[e][k];
      }
    }
    edges.resize(2 * m.edges.size());
    edge_elements.resize(2 * m.edges.size());
    kind.resize(m.edges.size());
    n_interior = 0;
    for (std::size_t i = 0; i < m.edges.size(); ++i) {
      edges[2 * i] = m.edges[i][0];
      edges[2 * i + 1] = m.edges[i][1];
      edge_elements[2 * i] = m.edge_elements[i].left;
      edge_elements[2 * i + 1] = m.edge_elements[i].right;
      kind[i] = static_cast<uint8_t>(m.edge_kind[i]);
      n_interior += m.edge_kind[i] == dgfem::EdgeKind::Interior;
    }
  }
};

struct RefHandle {
  explicit RefHandle(int k, int qo) : ref(k, qo) {
    const int nl = ref.n_local();
    const int nq = ref.volume_rule().size();
    const int ne = ref.edge_points().size();
    phi.resize(static_cast<std::size_t>(nq) * nl);
    dphi.resize(static_cast<std::size_t>(nq) * nl * 2);
    for (int q = 0; q < nq; ++q) {
      for (int j = 0; j < nl; ++j) {
        phi[q * nl + j] = ref.phi(q, j);
        dphi[(q * nl + j) * 2] = ref.dphi(q, j, 0);
        dphi[(q * nl + j) * 2 + 1] = ref.dphi(q, j, 1);
      }
    }
    edge_phi.resize(static_cast<std::size_t>(6) * ne * nl);
    edge_dphi.resize(static_cast<std::size_t>(6) * ne * nl * 2);
    for (int l = 0; l < 3; ++l) {
      for (int o = 0; o < 2; ++o) {
        for (int q = 0; q < ne; ++q) {
          for (int j = 0; j < nl; ++j) {
            const std::size_t base = ((static_cast<std::size_t>(l) * 2 + o) * ne + q) * nl + j;
            edge_phi[base] = ref.edge_phi(l, o, q, j);
            edge_dphi[base * 2] = ref.edge_dphi(l, o, q, j, 0);
            edge_dphi[base * 2 + 1] = ref.edge_dphi(l, o, q, j, 1);
          }
        }
      }
    }
  }
  dgfem::ReferenceElement ref;
  std::vector<double> phi, dphi, edge_phi, edge_dphi;
};

struct SystemHandle {
  dgfem::DgSystem system;
  dgfem::CsrMatrix K;
};

// Point location for PER_ELEMENT coefficients (SURVEY.md §8 "Config-5 policy"): the
// reference's callbacks only see (x, y), so the element (or the two elements of an edge) is
// recovered from the point.  A bucket grid over element bounding boxes keeps it O(1).
class Locator {
 public:
  explicit Locator(const dgfem::Mesh& mesh) : mesh_(mesh) {
    xmin_ = ymin_ = 1e300;
    xmax_ = ymax_ = -1e300;
    for (const auto& n : mesh.nodes) {
      xmin_ = std::min(xmin_, n.x);
      xmax_ = std::max(xmax_, n.x);
      ymin_ = std::min(ymin_, n.y);
      ymax_ = std::max(ymax_, n.y);
    }
    g_ = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(mesh.n_elements()) / 2.0)));
    buckets_.resize(static_cast<std::size_t>(g_) * g_);
    for (int e = 0; e < mesh.n_elements(); ++e) {
      double bx0 = 1e300, by0 = 1e300, bx1 = -1e300, by1 = -1e300;
      for (int v : mesh.elements[e]) {
        bx0 = std::min(bx0, mesh.nodes[v].x);
        bx1 = std::max(bx1, mesh.nodes[v].x);
        by0 = std::min(by0, mesh.nodes[v].y);
        by1 = std::max(by1, mesh.nodes[v].y);
      }
      const int i0 = cell(bx0, xmin_, xmax_), i1 = cell(bx1, xmin_, xmax_);
      const int j0 = cell(by0, ymin_, ymax_), j1 = cell(by1, ymin_, ymax_);
      for (int j = j0; j <= j1; ++j) {
        for (int i = i0; i <= i1; ++i) {
          buckets_[static_cast<std::size_t>(j) * g_ + i].push_back(e);
        }
      }
    }
  }

  // Elements whose closure contains (x, y), ascending.
  std::vector<int> find(double x, double y) const {
    std::vector<int> out;
    const int i = cell(x, xmin_, xmax_), j = cell(y, ymin_, ymax_);
    for (int e : buckets_[static_cast<std::size_t>(j) * g_ + i]) {
      const auto& el = mesh_.elements[e];
      const auto& p0 = mesh_.nodes[el[0]];
      const auto& p1 = mesh_.nodes[el[1]];
      const auto& p2 = mesh_.nodes[el[2]];
      const double det = (p1.x - p0.x) * (p2.y - p0.y) - (p2.x - p0.x) * (p1.y - p0.y);
      const double l1 = ((x - p0.x) * (p2.y - p0.y) - (p2.x - p0.x) * (y - p0.y)) / det;
      const double l2 = ((p1.x - p0.x) * (y - p0.y) - (x - p0.x) * (p1.y - p0.y)) / det;
      const double l0 = 1.0 - l1 - l2;
      const double tol = 1e-9;
      if (l0 >= -tol && l1 >= -tol && l2 >= -tol) {
        out.push_back(e);
      }
    }
    std::sort(out.begin(), out.end());
    return out;
  }

 private:
  int cell(double v, double lo, double hi) const {
    const double span = hi - lo;
    int c = span > 0 ? static_cast<int>((v - lo) / span * g_) : 0;
    return std::clamp(c, 0, g_ - 1);
  }
  const dgfem::Mesh& mesh_;
  double xmin_, xmax_, ymin_, ymax_;
  int g_;
  std::vector<std::vector<int>> buckets_;
};

// A PER_ELEMENT field as a reference callback: volume points see their element's value, edge
// points the average of the adjacent elements (boundary: the one element).
dgfem::ScalarField per_element_field(std::shared_ptr<Locator> loc,
                                     std::shared_ptr<std::vector<double>> values) {
  return [loc, values](std::span<const double> x, std::span<const double> y,
                       std::span<double> out) {
    for (std::size_t i = 0; i < x.size(); ++i) {
      const std::vector<int> hit = loc->find(x[i], y[i]);
      if (hit.empty()) {
        throw dgfem::Error(dgfem::ErrorCode::InvalidArgument, "point outside the mesh");
      }
      out[i] = hit.size() == 1 ? (*values)[hit[0]]
                               : 0.5 * ((*values)[hit[0]] + (*values)[hit[1]]);
    }
  };
}

dgfem::ScalarField scalar_field_from(const dgb_scalar_field& f, const dgfem::Mesh& mesh,
                                     std::shared_ptr<Locator>& loc) {
  if (f.kind == DGB_FIELD_PER_ELEMENT) {
    if (!loc) {
      loc = std::make_shared<Locator>(mesh);
    }
    auto values = std::make_shared<std::vector<double>>(f.per_element,
                                                        f.per_element + mesh.n_elements());
    return per_element_field(loc, values);
  }
  const dgb_scalar_field copy = f;
  return [copy](std::span<const double> x, std::span<const double> y, std::span<double> out) {
    for (std::size_t i = 0; i < x.size(); ++i) {
      out[i] = dgc_scalar_point(&copy, x[i], y[i]);
    }
  };
}

// clip_sides: unit-square sides (1: x=0, 2: x=1, 4: y=0, 8: y=1) on which the inward normal
// component of b is zeroed at boundary points -- the reference-side realisation of the
// "Neumann boundary is outflow-only" convention (SURVEY.md §8 "Config-3 policy").
dgfem::VectorField vector_field_from(const dgb_vector_field& b, int clip_sides) {
  const dgb_vector_field copy = b;
  return [copy, clip_sides](std::span<const double> x, std::span<const double> y,
                            std::span<double> ox, std::span<double> oy) {
    for (std::size_t i = 0; i < x.size(); ++i) {
      double bx, by;
      dgc_vector(&copy, x[i], y[i], &bx, &by);
      if ((clip_sides & 1) && x[i] == 0.0 && bx > 0.0) bx = 0.0;
      if ((clip_sides & 2) && x[i] == 1.0 && bx < 0.0) bx = 0.0;
      if ((clip_sides & 4) && y[i] == 0.0 && by > 0.0) by = 0.0;
      if ((clip_sides & 8) && y[i] == 1.0 && by < 0.0) by = 0.0;
      ox[i] = bx;
      oy[i] = by;
    }
  };
}

dgfem::ProblemSpec problem_from(const dgb_problem& p, const dgfem::Mesh& mesh, int clip_sides) {
  std::shared_ptr<Locator> loc;
  dgfem::ProblemSpec spec;
  spec.name = "dgb-descriptor";
  spec.diffusion = scalar_field_from(p.diffusion, mesh, loc);
  spec.advection = vector_field_from(p.advection, clip_sides);
  spec.linear_reaction = scalar_field_from(p.linear_reaction, mesh, loc);
  spec.source = scalar_field_from(p.source, mesh, loc);
  spec.dirichlet = scalar_field_from(p.dirichlet, mesh, loc);
  spec.neumann = scalar_field_from(p.neumann, mesh, loc);
  return spec;
}

dgfem::DgParameters params_from(const dgb_params& p) {
  dgfem::DgParameters out;
  out.method = p.method == DGB_NIPG   ? dgfem::DgMethod::NIPG
               : p.method == DGB_IIPG ? dgfem::DgMethod::IIPG
                                      : dgfem::DgMethod::SIPG;
  out.degree = p.degree;
  out.kappa = p.kappa;
  out.sigma_interior = p.sigma_interior;
  out.sigma_boundary = p.sigma_boundary;
  return out;
}

const dgfem::CsrMatrix* pick(const SystemHandle* s, int which) {
  switch (which) {
    case 0: return &s->K;
    case 1: return &s->system.D;
    case 2: return &s->system.C;
    case 3: return &s->system.R;
    default: return nullptr;
  }
}

}  // namespace

extern "C" {

const char* dgref_last_error(void) { return g_message.c_str(); }
long dgref_last_detail(void) { return g_detail; }

// dgfem::build_mesh (mesh.cpp:51-151).
int dgref_build_mesh(const double* nodes, int n_nodes, const int32_t* elements, int n_elements,
                     const int32_t* dirichlet, int n_dirichlet, const int32_t* neumann,
                     int n_neumann, void** out) {
  *out = nullptr;
  return guarded([&] {
    std::vector<dgfem::Node> nv(n_nodes);
    for (int i = 0; i < n_nodes; ++i) {
      nv[i] = {nodes[2 * i], nodes[2 * i + 1]};
    }
    std::vector<std::array<int, 3>> ev(n_elements);
    for (int e = 0; e < n_elements; ++e) {
      ev[e] = {elements[3 * e], elements[3 * e + 1], elements[3 * e + 2]};
    }
    std::vector<std::array<int, 2>> dv(n_dirichlet), nmv(n_neumann);
    for (int i = 0; i < n_dirichlet; ++i) dv[i] = {dirichlet[2 * i], dirichlet[2 * i + 1]};
    for (int i = 0; i < n_neumann; ++i) nmv[i] = {neumann[2 * i], neumann[2 * i + 1]};
    auto h = std::make_unique<MeshHandle>();
    h->mesh = dgfem::build_mesh(std::move(nv), std::move(ev), dv, nmv);
    h->flatten();
    *out = h.release();
  });
}

// dgfem::unit_square_mesh (mesh.cpp:189-210) refined `levels` times with uniform_refine
// (mesh.cpp:153-187).  neumann_sides as in dgb_mesh_unit_square.
int dgref_unit_square_refined(int levels, int neumann_sides, void** out) {
  *out = nullptr;
  return guarded([&] {
    auto pred = [neumann_sides](double x, double y) {
      return ((neumann_sides & 1) && x < 1e-12) || ((neumann_sides & 2) && x > 1.0 - 1e-12) ||
             ((neumann_sides & 4) && y < 1e-12) || ((neumann_sides & 8) && y > 1.0 - 1e-12);
    };
    auto h = std::make_unique<MeshHandle>();
    h->mesh = neumann_sides ? dgfem::unit_square_mesh(pred) : dgfem::unit_square_mesh();
    for (int l = 0; l < levels; ++l) {
      h->mesh = dgfem::uniform_refine(h->mesh);
    }
    h->flatten();
    *out = h.release();
  });
}

int dgref_mesh_view(void* handle, dgb_mesh_arrays* out) {
  auto* h = static_cast<MeshHandle*>(handle);
  out->n_nodes = h->mesh.n_nodes();
  out->n_elements = h->mesh.n_elements();
  out->n_edges = h->mesh.n_edges();
  out->n_interior_edges = h->n_interior;
  out->nodes = h->nodes.data();
  out->elements = h->elements.data();
  out->edges = h->edges.data();
  out->edge_kind = h->kind.data();
  out->edge_elements = h->edge_elements.data();
  out->element_edges = h->element_edges.data();
  return 0;
}

void dgref_mesh_free(void* handle) { delete static_cast<MeshHandle*>(handle); }

// dgfem::ReferenceElement(degree, quad_order) (reference.cpp:87-147) and its accessors.
int dgref_reference(int degree, int quad_order, void** out) {
  *out = nullptr;
  return guarded([&] { *out = new RefHandle(degree, quad_order); });
}

int dgref_reference_view(void* handle, dgb_reference_tables* out) {
  auto* h = static_cast<RefHandle*>(handle);
  const auto& r = h->ref;
  out->degree = r.degree();
  out->n_local = r.n_local();
  out->nq_vol = r.volume_rule().size();
  out->nq_edge = r.edge_points().size();
  out->vol_x = r.volume_rule().x.data();
  out->vol_y = r.volume_rule().y.data();
  out->vol_w = r.volume_rule().w.data();
  out->edge_t = r.edge_points().t.data();
  out->edge_w = r.edge_points().w.data();
  out->phi = h->phi.data();
  out->dphi = h->dphi.data();
  out->edge_phi = h->edge_phi.data();
  out->edge_dphi = h->edge_dphi.data();
  return 0;
}

void dgref_reference_free(void* handle) { delete static_cast<RefHandle*>(handle); }

// dgfem::set_parameters (assembly.cpp:483-506).
int dgref_set_parameters(int method, int degree, dgb_params* out) {
  return guarded([&] {
    const dgfem::DgMethod m = method == DGB_NIPG   ? dgfem::DgMethod::NIPG
                              : method == DGB_IIPG ? dgfem::DgMethod::IIPG
                                                   : dgfem::DgMethod::SIPG;
    const dgfem::DgParameters p = dgfem::set_parameters(m, degree);
    out->method = method;
    out->degree = p.degree;
    out->kappa = p.kappa;
    out->sigma_interior = p.sigma_interior;
    out->sigma_boundary = p.sigma_boundary;
    out->neumann_inflow = DGB_INFLOW_ERROR;
    out->pad_ = 0;
  });
}

// dgfem::assemble_all (assembly.cpp:725-737) + DgSystem::stiffness (:508-510) with
// Execution::parallel(threads) (threads <= 0: OpenMP default; 1: serial).  seconds[0] =
// assemble_all wall time, seconds[1] = stiffness() wall time (steady_clock).
// clip_sides: see vector_field_from (used with params->neumann_inflow == DGB_INFLOW_DROP).
int dgref_assemble(void* mesh_handle, void* ref_handle, const dgb_problem* problem,
                   const dgb_params* params, int threads, int clip_sides, double* seconds,
                   void** out) {
  *out = nullptr;
  return guarded([&] {
    auto* mh = static_cast<MeshHandle*>(mesh_handle);
    auto* rh = static_cast<RefHandle*>(ref_handle);
    const dgfem::ProblemSpec spec = problem_from(*problem, mh->mesh, clip_sides);
    const dgfem::DgParameters p = params_from(*params);
    const dgfem::Execution exec =
        threads == 1 ? dgfem::Execution::serial() : dgfem::Execution::parallel(threads);
    auto s = std::make_unique<SystemHandle>();
    const auto t0 = std::chrono::steady_clock::now();
    s->system = dgfem::assemble_all(mh->mesh, rh->ref, spec, p, exec);
    const auto t1 = std::chrono::steady_clock::now();
    s->K = s->system.stiffness();
    const auto t2 = std::chrono::steady_clock::now();
    if (seconds) {
      seconds[0] = std::chrono::duration<double>(t1 - t0).count();
      seconds[1] = std::chrono::duration<double>(t2 - t1).count();
    }
    *out = s.release();
  });
}

// Only the convection part (assemble_convection, assembly.cpp:561-609): exercises the
// InflowOnNeumann path exactly as the reference tests do (test_assembly.cpp:371-381).
int dgref_assemble_convection(void* mesh_handle, void* ref_handle, const dgb_problem* problem,
                              int threads) {
  return guarded([&] {
    auto* mh = static_cast<MeshHandle*>(mesh_handle);
    auto* rh = static_cast<RefHandle*>(ref_handle);
    const dgfem::ProblemSpec spec = problem_from(*problem, mh->mesh, 0);
    const dgfem::Execution exec =
        threads == 1 ? dgfem::Execution::serial() : dgfem::Execution::parallel(threads);
    (void)dgfem::assemble_convection(mh->mesh, rh->ref, spec, exec);
  });
}

// which: 0 = K = stiffness(), 1 = D, 2 = C, 3 = R.
int dgref_system_nnz(void* handle, int which, long long* nnz, int* n) {
  const dgfem::CsrMatrix* m = pick(static_cast<SystemHandle*>(handle), which);
  if (!m) return DGB_STATUS_INVALID_ARGUMENT;
  *nnz = static_cast<long long>(m->nnz());
  *n = m->n;
  return 0;
}

int dgref_system_copy(void* handle, int which, int32_t* row_offsets, int32_t* cols,
                      double* vals) {
  const dgfem::CsrMatrix* m = pick(static_cast<SystemHandle*>(handle), which);
  if (!m) return DGB_STATUS_INVALID_ARGUMENT;
  if (row_offsets) std::memcpy(row_offsets, m->row_offsets.data(), (m->n + 1) * sizeof(int32_t));
  if (cols) std::memcpy(cols, m->col_indices.data(), m->nnz() * sizeof(int32_t));
  if (vals) std::memcpy(vals, m->values.data(), m->nnz() * sizeof(double));
  return 0;
}

int dgref_system_rhs(void* handle, double* F) {
  auto* s = static_cast<SystemHandle*>(handle);
  std::memcpy(F, s->system.F.data(), s->system.F.size() * sizeof(double));
  return 0;
}

// dgfem::matvec(stiffness(), x) (sparse.cpp:116-129).
int dgref_matvec(void* handle, const double* x, double* y) {
  auto* s = static_cast<SystemHandle*>(handle);
  return guarded([&] {
    std::vector<double> xv(x, x + s->K.n);
    const std::vector<double> yv = dgfem::matvec(s->K, xv);
    std::memcpy(y, yv.data(), yv.size() * sizeof(double));
  });
}

void dgref_system_free(void* handle) { delete static_cast<SystemHandle*>(handle); }

// dgfem::element_geometry (mesh.cpp:212-230): out = B00 B01 B10 B11, G00 G01 G10 G11
// (inverse transpose), det, area, diameter, origin x, origin y.
int dgref_element_geometry(void* mesh_handle, int element, double* out) {
  return guarded([&] {
    const dgfem::ElementGeometry g =
        dgfem::element_geometry(static_cast<MeshHandle*>(mesh_handle)->mesh, element);
    const double v[13] = {g.jacobian[0][0],      g.jacobian[0][1],      g.jacobian[1][0],
                          g.jacobian[1][1],      g.inv_transpose[0][0], g.inv_transpose[0][1],
                          g.inv_transpose[1][0], g.inv_transpose[1][1], g.det,
                          g.area,                g.diameter,            g.origin[0],
                          g.origin[1]};
    std::memcpy(out, v, sizeof v);
  });
}

// dgfem::edge_geometry (mesh.cpp:232-257): out = length, nx, ny, tx, ty, oriented_from.
int dgref_edge_geometry(void* mesh_handle, int edge, double* out) {
  return guarded([&] {
    const dgfem::EdgeGeometryData g =
        dgfem::edge_geometry(static_cast<MeshHandle*>(mesh_handle)->mesh, edge);
    const double v[6] = {g.length,     g.normal[0], g.normal[1], g.tangent[0],
                         g.tangent[1], static_cast<double>(g.oriented_from)};
    std::memcpy(out, v, sizeof v);
  });
}


// dgfem::assemble_nonlinear (nonlinear.cpp:11-107) with the reaction of dgb_reaction `kind`
// (host twin dgc_reaction, the reference's own expressions).  h[n]; the CSR of HJ into
// row_offsets[n+1], cols[nnz], vals[nnz] (nnz = n_elements * nl * nl).  seconds[0] = wall time.
int dgref_assemble_nonlinear(void* mesh_handle, void* ref_handle, const double* coef, long long n,
                             int kind, int threads, double* h, int32_t* row_offsets, int32_t* cols,
                             double* vals, double* seconds) {
  return guarded([&] {
    auto* mh = static_cast<MeshHandle*>(mesh_handle);
    auto* rh = static_cast<RefHandle*>(ref_handle);
    const dgfem::ReactionTerm reaction{
        dgfem::scalar_map([kind](double u) { double r, dr; dgc_reaction(kind, u, &r, &dr); return r; }),
        dgfem::scalar_map([kind](double u) { double r, dr; dgc_reaction(kind, u, &r, &dr); return dr; })};
    const std::vector<double> c(coef, coef + n);
    const dgfem::Execution exec =
        threads == 1 ? dgfem::Execution::serial() : dgfem::Execution::parallel(threads);
    const auto t0 = std::chrono::steady_clock::now();
    auto [hv, hj] = dgfem::assemble_nonlinear(c, mh->mesh, rh->ref, reaction, exec);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) seconds[0] = std::chrono::duration<double>(t1 - t0).count();
    if (h) std::memcpy(h, hv.data(), hv.size() * sizeof(double));
    if (row_offsets) std::memcpy(row_offsets, hj.row_offsets.data(), (hj.n + 1) * sizeof(int32_t));
    if (cols) std::memcpy(cols, hj.col_indices.data(), hj.nnz() * sizeof(int32_t));
    if (vals) std::memcpy(vals, hj.values.data(), hj.nnz() * sizeof(double));
  });
}


// dgfem::l2_error (postprocess.cpp:14-50): out[0] = L2 error, out[1] = max element diameter.
int dgref_l2_error(void* mesh_handle, void* ref_handle, const double* coef, long long n,
                   const dgb_scalar_field* exact, double* out) {
  return guarded([&] {
    auto* mh = static_cast<MeshHandle*>(mesh_handle);
    auto* rh = static_cast<RefHandle*>(ref_handle);
    std::shared_ptr<Locator> loc;
    dgfem::ExactSolution ex;
    ex.value = scalar_field_from(*exact, mh->mesh, loc);
    ex.du_dx = ex.value;
    ex.du_dy = ex.value;
    const std::vector<double> c(coef, coef + n);
    const auto [err, h] = dgfem::l2_error(c, mh->mesh, rh->ref, ex);
    out[0] = err;
    out[1] = h;
  });
}

// dgfem::project (postprocess.cpp:56-81) into out[n_elements * nl].
int dgref_project(void* mesh_handle, void* ref_handle, const dgb_scalar_field* f, double* out) {
  return guarded([&] {
    auto* mh = static_cast<MeshHandle*>(mesh_handle);
    auto* rh = static_cast<RefHandle*>(ref_handle);
    std::shared_ptr<Locator> loc;
    const std::vector<double> c = dgfem::project(mh->mesh, rh->ref, scalar_field_from(*f, mh->mesh, loc));
    std::memcpy(out, c.data(), c.size() * sizeof(double));
  });
}

// dgfem::eval_solution (postprocess.cpp:83-93) at n points.
int dgref_eval_solution(const double* coef, long long n_coef, void* ref_handle, long long n,
                        const int32_t* elements, const double* xh, const double* yh, double* out) {
  return guarded([&] {
    auto* rh = static_cast<RefHandle*>(ref_handle);
    const std::vector<double> c(coef, coef + n_coef);
    for (long long i = 0; i < n; ++i) out[i] = dgfem::eval_solution(c, rh->ref, elements[i], xh[i], yh[i]);
  });
}

}  // extern "C"
