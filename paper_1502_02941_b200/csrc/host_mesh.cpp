// host_mesh.cpp -- host-side mesh input for the GPU path.
//
// dgb_mesh_build produces exactly the arrays of dgfem::build_mesh
// (/root/reference/proj/src/mesh.cpp:51-151) -- same edge numbering (lexicographic sorted
// node pairs), same left/right convention, same local-edge layout, same error codes and
// details -- but derives the edge table with a counting sort over the smaller node of each
// half-edge instead of a std::map, so config-4 sized meshes (8.4 M triangles) build in about
// a second instead of ~40 s.  dgb_mesh_unit_square generates the BASELINE.json meshes.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#include "common.hpp"

struct dgb_mesh {
  // input (before reorientation)
  std::vector<double> raw_nodes;
  std::vector<int32_t> raw_elements, raw_dirichlet, raw_neumann;
  // built mesh
  std::vector<double> nodes;
  std::vector<int32_t> elements, edges, edge_elements, element_edges;
  std::vector<uint8_t> edge_kind;
  int32_t n_interior = 0;
};

namespace {

inline double element_det(const double* nd, const int32_t* el) {
  const double p0x = nd[2 * el[0]], p0y = nd[2 * el[0] + 1];
  const double p1x = nd[2 * el[1]], p1y = nd[2 * el[1] + 1];
  const double p2x = nd[2 * el[2]], p2y = nd[2 * el[2] + 1];
  return (p1x - p0x) * (p2y - p0y) - (p2x - p0x) * (p1y - p0y);
}

inline double longest_edge(const double* nd, const int32_t* el) {
  double d = 0.0;
  for (int l = 0; l < 3; ++l) {
    const int a = el[(l + 1) % 3], b = el[(l + 2) % 3];
    d = std::max(d, std::hypot(nd[2 * b] - nd[2 * a], nd[2 * b + 1] - nd[2 * a + 1]));
  }
  return d;
}

void build(dgb_mesh& m) {
  const int64_t n_nodes = static_cast<int64_t>(m.raw_nodes.size() / 2);
  const int64_t n_el = static_cast<int64_t>(m.raw_elements.size() / 3);
  if (n_el > INT32_MAX / 3 || n_nodes > INT32_MAX) {
    throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "mesh too large for 32-bit indices");
  }
  m.nodes = m.raw_nodes;
  m.elements = m.raw_elements;
  const double* nd = m.nodes.data();
  // Element checks and CW -> CCW (mesh.cpp:56-73), in element order.
  for (int64_t e = 0; e < n_el; ++e) {
    int32_t* el = &m.elements[3 * e];
    for (int k = 0; k < 3; ++k) {
      if (el[k] < 0 || el[k] >= n_nodes) {
        throw dgb::Error(DGB_STATUS_INVALID_TOPOLOGY,
                         "element references a node index outside the node table", e);
      }
    }
    const double det = element_det(nd, el);
    const double diam = longest_edge(nd, el);
    if (std::abs(det) <= 1e-14 * diam * diam) {
      throw dgb::Error(DGB_STATUS_DEGENERATE_ELEMENT, "element has (numerically) zero area", e);
    }
    if (det < 0.0) std::swap(el[1], el[2]);
  }

  // Half-edges h = 3e + l with key (a, b), a < b.  A stable counting sort by a, then a stable
  // sort of each bucket by b, gives the std::map order of mesh.cpp:77-83 with each key's
  // elements in insertion (ascending) order.
  const int64_t nh = 3 * n_el;
  std::vector<int32_t> ha(nh), hb(nh);
  for (int64_t e = 0; e < n_el; ++e) {
    const int32_t* el = &m.elements[3 * e];
    for (int l = 0; l < 3; ++l) {
      const int32_t u = el[(l + 1) % 3], v = el[(l + 2) % 3];
      ha[3 * e + l] = std::min(u, v);
      hb[3 * e + l] = std::max(u, v);
    }
  }
  std::vector<int64_t> start(n_nodes + 1, 0);
  for (int64_t h = 0; h < nh; ++h) ++start[ha[h] + 1];
  std::partial_sum(start.begin(), start.end(), start.begin());
  std::vector<int32_t> order(nh);
  {
    std::vector<int64_t> cursor(start.begin(), start.end() - 1);
    for (int64_t h = 0; h < nh; ++h) order[cursor[ha[h]]++] = static_cast<int32_t>(h);
  }
  for (int64_t a = 0; a < n_nodes; ++a) {
    auto first = order.begin() + start[a], last = order.begin() + start[a + 1];
    if (last - first > 1) {
      std::stable_sort(first, last, [&](int32_t x, int32_t y) { return hb[x] < hb[y]; });
    }
  }

  m.edges.clear();
  m.edge_elements.clear();
  m.edges.reserve(nh / 2 + n_nodes);
  m.edge_elements.reserve(nh / 2 + n_nodes);
  m.element_edges.assign(3 * n_el, -1);
  for (int64_t k = 0; k < nh;) {
    int64_t k1 = k + 1;
    while (k1 < nh && ha[order[k1]] == ha[order[k]] && hb[order[k1]] == hb[order[k]]) ++k1;
    const int32_t edge = static_cast<int32_t>(m.edges.size() / 2);
    if (k1 - k > 2) {
      throw dgb::Error(DGB_STATUS_NON_MANIFOLD, "edge is shared by more than two elements",
                       edge);
    }
    m.edges.push_back(ha[order[k]]);
    m.edges.push_back(hb[order[k]]);
    int32_t left = order[k] / 3, right = (k1 - k == 2) ? order[k + 1] / 3 : -1;
    if (right >= 0 && right < left) std::swap(left, right);
    m.edge_elements.push_back(left);
    m.edge_elements.push_back(right);
    for (int64_t i = k; i < k1; ++i) m.element_edges[order[i]] = edge;
    k = k1;
  }
  const int64_t n_edges = static_cast<int64_t>(m.edges.size() / 2);

  // Edge lookup by sorted pair: edges are sorted by (a, b); bucket by a.
  std::vector<int64_t> first_edge(n_nodes + 1, 0);
  for (int64_t i = 0; i < n_edges; ++i) ++first_edge[m.edges[2 * i] + 1];
  std::partial_sum(first_edge.begin(), first_edge.end(), first_edge.begin());
  auto find_edge = [&](int32_t u, int32_t v) -> int64_t {
    const int32_t a = std::min(u, v), b = std::max(u, v);
    if (a < 0 || b >= n_nodes) return -1;
    int64_t lo = first_edge[a], hi = first_edge[a + 1];
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (m.edges[2 * mid + 1] < b) lo = mid + 1; else hi = mid;
    }
    return (lo < first_edge[a + 1] && m.edges[2 * lo + 1] == b) ? lo : -1;
  };

  // Boundary classification (mesh.cpp:116-149).
  m.edge_kind.assign(n_edges, DGB_EDGE_INTERIOR);
  std::vector<uint8_t> tagged(n_edges, 0);
  auto classify = [&](const std::vector<int32_t>& list, uint8_t kind) {
    for (std::size_t i = 0; i + 1 < list.size(); i += 2) {
      const int64_t e = find_edge(list[i], list[i + 1]);
      if (e < 0) {
        throw dgb::Error(DGB_STATUS_INVALID_BOUNDARY_SPEC,
                         "boundary list names a node pair that is not a mesh edge");
      }
      if (m.edge_elements[2 * e + 1] >= 0) {
        throw dgb::Error(DGB_STATUS_INVALID_BOUNDARY_SPEC, "boundary list names an interior edge",
                         e);
      }
      if (tagged[e]) {
        throw dgb::Error(DGB_STATUS_INVALID_BOUNDARY_SPEC, "boundary edge tagged more than once",
                         e);
      }
      tagged[e] = 1;
      m.edge_kind[e] = kind;
    }
  };
  classify(m.raw_dirichlet, DGB_EDGE_DIRICHLET);
  classify(m.raw_neumann, DGB_EDGE_NEUMANN);
  m.n_interior = 0;
  for (int64_t e = 0; e < n_edges; ++e) {
    if (m.edge_elements[2 * e + 1] < 0 && !tagged[e]) {
      throw dgb::Error(DGB_STATUS_INVALID_BOUNDARY_SPEC,
                       "boundary edge missing from the Dirichlet/Neumann lists", e);
    }
    m.n_interior += m.edge_kind[e] == DGB_EDGE_INTERIOR;
  }
}

// splitmix64 (Steele, Lea, Flood 2014): the seeded stream behind every synthetic input.
struct SplitMix64 {
  uint64_t state;
  uint64_t next() {
    uint64_t z = (state += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

}  // namespace

extern "C" {

int dgb_mesh_build(const double* nodes_xy, int32_t n_nodes, const int32_t* elements,
                   int32_t n_elements, const int32_t* dirichlet_pairs, int32_t n_dirichlet,
                   const int32_t* neumann_pairs, int32_t n_neumann, dgb_mesh** out) {
  *out = nullptr;
  return dgb::guarded([&] {
    if (n_nodes < 0 || n_elements < 0 || n_dirichlet < 0 || n_neumann < 0) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "negative count");
    }
    auto* m = new dgb_mesh();
    try {
      m->raw_nodes.assign(nodes_xy, nodes_xy + 2 * static_cast<int64_t>(n_nodes));
      m->raw_elements.assign(elements, elements + 3 * static_cast<int64_t>(n_elements));
      m->raw_dirichlet.assign(dirichlet_pairs, dirichlet_pairs + 2 * n_dirichlet);
      m->raw_neumann.assign(neumann_pairs, neumann_pairs + 2 * n_neumann);
      build(*m);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int dgb_mesh_rectangle(int32_t nx, int32_t ny, double lx, double ly, double jitter,
                       uint64_t jitter_seed, int32_t permute, uint64_t permute_seed,
                       int32_t neumann_sides, dgb_mesh** out) {
  *out = nullptr;
  return dgb::guarded([&] {
    if (nx < 1 || ny < 1 || static_cast<int64_t>(nx) * ny > (int64_t{1} << 29)) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "grid size out of range", nx);
    }
    if (!(lx > 0.0 && ly > 0.0)) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "bad extent");
    if (!(jitter >= 0.0 && jitter < 0.5)) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "jitter must be in [0, 0.5)");
    }
    auto* m = new dgb_mesh();
    try {
      const int64_t px = static_cast<int64_t>(nx) + 1, py = static_cast<int64_t>(ny) + 1;
      auto node = [px](int64_t i, int64_t j) { return static_cast<int32_t>(j * px + i); };
      m->raw_nodes.resize(2 * px * py);
      const double hx = lx / nx, hy = ly / ny;
      SplitMix64 rng{jitter_seed};
      for (int64_t j = 0; j < py; ++j) {
        for (int64_t i = 0; i < px; ++i) {
          double x = lx * (static_cast<double>(i) / nx), y = ly * (static_cast<double>(j) / ny);
          if (jitter > 0.0 && i > 0 && i < nx && j > 0 && j < ny) {
            x += (2.0 * rng.uniform() - 1.0) * (jitter * hx);
            y += (2.0 * rng.uniform() - 1.0) * (jitter * hy);
          }
          m->raw_nodes[2 * node(i, j)] = x;
          m->raw_nodes[2 * node(i, j) + 1] = y;
        }
      }
      m->raw_elements.resize(6 * static_cast<int64_t>(nx) * ny);
      for (int64_t j = 0; j < ny; ++j) {
        for (int64_t i = 0; i < nx; ++i) {
          const int64_t c = j * nx + i;
          const int32_t v00 = node(i, j), v10 = node(i + 1, j), v01 = node(i, j + 1),
                        v11 = node(i + 1, j + 1);
          int32_t* lo = &m->raw_elements[6 * c];
          lo[0] = v00; lo[1] = v10; lo[2] = v11;  // lower triangle, CCW
          lo[3] = v00; lo[4] = v11; lo[5] = v01;  // upper triangle, CCW
        }
      }
      if (permute) {  // Fisher-Yates over the element list (config 4)
        SplitMix64 prng{permute_seed};
        const int64_t ne = 2 * static_cast<int64_t>(nx) * ny;
        for (int64_t i = ne - 1; i > 0; --i) {
          const int64_t k = static_cast<int64_t>(prng.next() % static_cast<uint64_t>(i + 1));
          for (int t = 0; t < 3; ++t) std::swap(m->raw_elements[3 * i + t], m->raw_elements[3 * k + t]);
        }
      }
      auto side = [&](int bit, int64_t i0, int64_t j0, int64_t di, int64_t dj, int64_t count) {
        auto& list = (neumann_sides & bit) ? m->raw_neumann : m->raw_dirichlet;
        for (int64_t s = 0; s < count; ++s) {
          list.push_back(node(i0 + s * di, j0 + s * dj));
          list.push_back(node(i0 + (s + 1) * di, j0 + (s + 1) * dj));
        }
      };
      side(4, 0, 0, 1, 0, nx);   // y = 0
      side(8, 0, ny, 1, 0, nx);  // y = ly
      side(1, 0, 0, 0, 1, ny);   // x = 0
      side(2, nx, 0, 0, 1, ny);  // x = lx
      build(*m);
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
  });
}

int dgb_mesh_unit_square(int32_t n, double jitter, uint64_t jitter_seed, int32_t permute,
                         uint64_t permute_seed, int32_t neumann_sides, dgb_mesh** out) {
  if (n < 1 || n > 16384) {
    *out = nullptr;
    return dgb::record_error(DGB_STATUS_INVALID_ARGUMENT, "InvalidArgument: n out of range", n);
  }
  return dgb_mesh_rectangle(n, n, 1.0, 1.0, jitter, jitter_seed, permute, permute_seed,
                            neumann_sides, out);
}

int dgb_mesh_view(const dgb_mesh* m, dgb_mesh_arrays* out) {
  if (!m || !out) return DGB_STATUS_INVALID_ARGUMENT;
  out->n_nodes = static_cast<int32_t>(m->nodes.size() / 2);
  out->n_elements = static_cast<int32_t>(m->elements.size() / 3);
  out->n_edges = static_cast<int32_t>(m->edges.size() / 2);
  out->n_interior_edges = m->n_interior;
  out->nodes = m->nodes.data();
  out->elements = m->elements.data();
  out->edges = m->edges.data();
  out->edge_kind = m->edge_kind.data();
  out->edge_elements = m->edge_elements.data();
  out->element_edges = m->element_edges.data();
  return DGB_OK;
}

int dgb_mesh_raw(const dgb_mesh* m, const double** nodes, int32_t* n_nodes,
                 const int32_t** elements, int32_t* n_elements, const int32_t** dirichlet,
                 int32_t* n_dirichlet, const int32_t** neumann, int32_t* n_neumann) {
  if (!m) return DGB_STATUS_INVALID_ARGUMENT;
  if (nodes) *nodes = m->raw_nodes.data();
  if (elements) *elements = m->raw_elements.data();
  if (dirichlet) *dirichlet = m->raw_dirichlet.data();
  if (neumann) *neumann = m->raw_neumann.data();
  if (n_nodes) *n_nodes = static_cast<int32_t>(m->raw_nodes.size() / 2);
  if (n_elements) *n_elements = static_cast<int32_t>(m->raw_elements.size() / 3);
  if (n_dirichlet) *n_dirichlet = static_cast<int32_t>(m->raw_dirichlet.size() / 2);
  if (n_neumann) *n_neumann = static_cast<int32_t>(m->raw_neumann.size() / 2);
  return DGB_OK;
}

void dgb_mesh_free(dgb_mesh* m) { delete m; }

}  // extern "C"
