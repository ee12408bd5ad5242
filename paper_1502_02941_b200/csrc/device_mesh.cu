// device_mesh.cu -- mesh topology built on the device.
//
// Replaces dgfem::build_mesh (mesh.cpp:51-151) and uniform_refine (mesh.cpp:153-187), whose
// std::map edge table dominates the reference's setup (9.1 s to reach refinement level 9,
// 42.2 s for level 10).  Sort-based instead:
//   1. per element: index range and degeneracy checks (the reference's order and error
//      details), CCW reorientation;
//   2. 3E half-edges keyed by the sorted node pair (a << 32 | b), stable radix sort --
//      ascending keys are the reference's lexicographic std::map order, and equal keys keep
//      element order, so adj[0] / adj[1] come out exactly as the reference pushes them;
//   3. run heads + inclusive scan number the edges; a run longer than 2 is NonManifold;
//   4. boundary lists classified by binary search over the unique keys; "tagged more than
//      once" is found by sorting (edge, list position); errors report the first offending
//      list entry in the reference's processing order.
// Every output array is bit-identical to build_mesh's (tests/test_gpu_device_mesh.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <mutex>
#include <set>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.hpp"
#include "device_math.cuh"

namespace dgb {
void cuda_check(cudaError_t err, const char* what);
}

struct dgb_device_mesh {
  int device = 0;
  int32_t n_nodes = 0, n_elements = 0, n_edges = 0, n_interior = 0;
  double* nodes = nullptr;
  int32_t* elements = nullptr;
  int32_t* edges = nullptr;
  uint8_t* edge_kind = nullptr;
  int32_t* edge_elements = nullptr;
  int32_t* element_edges = nullptr;
};

namespace {

using dgb::cuda_check;
constexpr int kT = 256;
constexpr unsigned long long kNone = ~0ull;

unsigned blocks(long long n) { return static_cast<unsigned>((n + kT - 1) / kT); }

// Element checks (mesh.cpp:55-73): the lowest offending element wins; within an element the
// index check comes first.  err = e << 2 | code (0 InvalidTopology, 1 DegenerateElement).
__global__ void validate_orient_kernel(const double* __restrict__ nodes, const int32_t* __restrict__ in,
                                       int E, int n_nodes, int32_t* __restrict__ out,
                                       unsigned long long* err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  int v[3];
  for (int k = 0; k < 3; ++k) v[k] = in[3 * e + k];
  for (int k = 0; k < 3; ++k) {
    if (v[k] < 0 || v[k] >= n_nodes) {
      atomicMin(err, static_cast<unsigned long long>(e) << 2 | 0ull);
      return;
    }
  }
  const double p0x = nodes[2 * v[0]], p0y = nodes[2 * v[0] + 1];
  const double p1x = nodes[2 * v[1]], p1y = nodes[2 * v[1] + 1];
  const double p2x = nodes[2 * v[2]], p2y = nodes[2 * v[2] + 1];
  // element_det (mesh.cpp:32-37), unfused
  const double det = __dsub_rn(__dmul_rn(__dsub_rn(p1x, p0x), __dsub_rn(p2y, p0y)),
                               __dmul_rn(__dsub_rn(p2x, p0x), __dsub_rn(p1y, p0y)));
  double diam = 0.0;  // longest_edge (mesh.cpp:39-47)
  const double px[3] = {p0x, p1x, p2x}, py[3] = {p0y, p1y, p2y};
  for (int l = 0; l < 3; ++l) {
    const int a = (l + 1) % 3, b = (l + 2) % 3;
    diam = fmax(diam, dgb::hypot_dd(__dsub_rn(px[b], px[a]), __dsub_rn(py[b], py[a])));
  }
  if (fabs(det) <= __dmul_rn(__dmul_rn(1e-14, diam), diam)) {
    atomicMin(err, static_cast<unsigned long long>(e) << 2 | 1ull);
    return;
  }
  if (det < 0.0) {
    const int t = v[1];
    v[1] = v[2];
    v[2] = t;
  }
  for (int k = 0; k < 3; ++k) out[3 * e + k] = v[k];
}

__global__ void halfedge_kernel(const int32_t* __restrict__ el, int E, unsigned long long* keys,
                                int32_t* vals) {
  const long long h = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (h >= 3LL * E) return;
  const int e = static_cast<int>(h / 3), l = static_cast<int>(h - 3LL * e);
  const unsigned a = static_cast<unsigned>(el[3 * e + (l + 1) % 3]);
  const unsigned b = static_cast<unsigned>(el[3 * e + (l + 2) % 3]);
  const unsigned lo = a < b ? a : b, hi = a < b ? b : a;
  keys[h] = static_cast<unsigned long long>(lo) << 32 | hi;
  vals[h] = static_cast<int32_t>(h);
}

__global__ void head_kernel(const unsigned long long* __restrict__ keys, long long M, int32_t* flags) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < M) flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

// Edge table from the sorted half-edges (mesh.cpp:85-111).
__global__ void edge_table_kernel(const unsigned long long* __restrict__ keys,
                                  const int32_t* __restrict__ vals, const int32_t* __restrict__ uid,
                                  long long M, int32_t* edges, int32_t* edge_elements,
                                  int32_t* element_edges, unsigned long long* ukeys,
                                  unsigned long long* nonmanifold) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= M) return;
  const int u = uid[i] - 1;
  element_edges[vals[i]] = u;
  const unsigned long long k = keys[i];
  if (i > 0 && keys[i - 1] == k) return;  // not a run head
  edges[2 * u] = static_cast<int32_t>(k >> 32);
  edges[2 * u + 1] = static_cast<int32_t>(k & 0xFFFFFFFFull);
  ukeys[u] = k;
  const bool two = i + 1 < M && keys[i + 1] == k;
  if (two && i + 2 < M && keys[i + 2] == k) atomicMin(nonmanifold, static_cast<unsigned long long>(u));
  edge_elements[2 * u] = vals[i] / 3;                     // adj[0]
  edge_elements[2 * u + 1] = two ? vals[i + 1] / 3 : -1;  // adj[1] (> adj[0]: element order)
}

// Boundary list entry p (dirichlet entries first, then neumann): its edge, or a status.
// status: err = p << 2 | code (1 not a mesh edge, 2 interior edge; duplicates found later).
__global__ void boundary_lookup_kernel(const int32_t* __restrict__ pairs, int n_pairs,
                                       const unsigned long long* __restrict__ ukeys, int n_edges,
                                       const int32_t* __restrict__ edge_elements, int32_t* edge_of,
                                       unsigned long long* dup_keys, int32_t* dup_vals,
                                       unsigned long long* err) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const unsigned a = static_cast<unsigned>(pairs[2 * p]), b = static_cast<unsigned>(pairs[2 * p + 1]);
  const unsigned lo = a < b ? a : b, hi = a < b ? b : a;
  const unsigned long long k = static_cast<unsigned long long>(lo) << 32 | hi;
  int l = 0, r = n_edges;  // lower_bound
  while (l < r) {
    const int m = (l + r) >> 1;
    if (ukeys[m] < k) l = m + 1; else r = m;
  }
  int u = -1;
  if (l < n_edges && ukeys[l] == k && pairs[2 * p] >= 0 && pairs[2 * p + 1] >= 0) u = l;
  edge_of[p] = u;
  dup_keys[p] = (static_cast<unsigned long long>(static_cast<unsigned>(u)) << 32) | static_cast<unsigned>(p);
  dup_vals[p] = p;
  if (u < 0) {
    atomicMin(err, static_cast<unsigned long long>(p) << 2 | 1ull);
  } else if (edge_elements[2 * u + 1] >= 0) {
    atomicMin(err, static_cast<unsigned long long>(p) << 2 | 2ull);
  }
}

// Sorted (edge, position): every entry after the first of its edge is "tagged more than once".
__global__ void duplicate_kernel(const unsigned long long* __restrict__ sorted, int n,
                                 unsigned long long* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 || i >= n) return;
  const unsigned long long k = sorted[i], prev = sorted[i - 1];
  if ((k >> 32) == 0xFFFFFFFFull) return;  // not an edge: reported by the lookup
  if ((k >> 32) == (prev >> 32)) {
    atomicMin(err, (k & 0xFFFFFFFFull) << 2 | 3ull);
  }
}

__global__ void classify_kernel(const int32_t* __restrict__ edge_of, int n_dirichlet, int n_pairs,
                                uint8_t* kind) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const int u = edge_of[p];
  if (u >= 0) kind[u] = p < n_dirichlet ? DGB_EDGE_DIRICHLET : DGB_EDGE_NEUMANN;
}

__global__ void missing_kernel(const int32_t* __restrict__ edge_elements, const uint8_t* __restrict__ kind,
                               int n_edges, unsigned long long* missing, unsigned long long* n_interior) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_edges) return;
  if (edge_elements[2 * u + 1] >= 0) {
    atomicAdd(n_interior, 1ull);
  } else if (kind[u] == DGB_EDGE_INTERIOR) {
    atomicMin(missing, static_cast<unsigned long long>(u));
  }
}

// uniform_refine (mesh.cpp:153-187): midpoint nodes, 4 children per element, split boundary
// lists in edge order.
__global__ void refine_nodes_kernel(const double* __restrict__ nodes, int n_nodes,
                                    const int32_t* __restrict__ edges, int n_edges, double* out) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < 2LL * n_nodes) out[i] = nodes[i];
  if (i < n_edges) {
    const int a = edges[2 * i], b = edges[2 * i + 1];
    out[2 * (n_nodes + i)] = 0.5 * (nodes[2 * a] + nodes[2 * b]);
    out[2 * (n_nodes + i) + 1] = 0.5 * (nodes[2 * a + 1] + nodes[2 * b + 1]);
  }
}

__global__ void refine_elements_kernel(const int32_t* __restrict__ el, const int32_t* __restrict__ ee,
                                       int E, int base, int32_t* out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  const int v0 = el[3 * e], v1 = el[3 * e + 1], v2 = el[3 * e + 2];
  const int m0 = base + ee[3 * e], m1 = base + ee[3 * e + 1], m2 = base + ee[3 * e + 2];
  int32_t* o = out + 12LL * e;
  const int c[12] = {v0, m2, m1, m2, v1, m0, m1, m0, v2, m2, m0, m1};
  for (int k = 0; k < 12; ++k) o[k] = c[k];
}

__global__ void boundary_flags_kernel(const uint8_t* __restrict__ kind, int n_edges, int32_t* fd, int32_t* fn) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_edges) return;
  fd[u] = kind[u] == DGB_EDGE_DIRICHLET;
  fn[u] = kind[u] == DGB_EDGE_NEUMANN;
}

__global__ void refine_boundary_kernel(const uint8_t* __restrict__ kind, const int32_t* __restrict__ edges,
                                       const int32_t* __restrict__ pd, const int32_t* __restrict__ pn,
                                       int n_edges, int base, int n_dir_entries, int32_t* pairs) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n_edges || kind[u] == DGB_EDGE_INTERIOR) return;
  const int mid = base + u;
  const int slot = kind[u] == DGB_EDGE_DIRICHLET ? 2 * pd[u] : n_dir_entries + 2 * pn[u];
  pairs[2 * slot] = edges[2 * u];
  pairs[2 * slot + 1] = mid;
  pairs[2 * slot + 2] = mid;
  pairs[2 * slot + 3] = edges[2 * u + 1];
}

// Stream-ordered allocations from the device's default pool, kept cached (release threshold
// raised once per device): a refine chain allocates and frees per level, and plain
// cudaMalloc / cudaFree made its wall time vary 47 ms .. 0.39 s from run to run.
void keep_mesh_pool_cached() {
  static std::mutex mu;
  static std::set<int> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (!done.insert(dev).second) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    unsigned long long keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
}
template <typename T>
void pool_alloc(T** x, size_t bytes, cudaStream_t s) {
  keep_mesh_pool_cached();
  cuda_check(cudaMallocAsync(reinterpret_cast<void**>(x), std::max<size_t>(bytes, 1), s),
             "cudaMallocAsync(mesh)");
}

struct Tmp {
  cudaStream_t s;
  std::vector<void*> p;
  explicit Tmp(cudaStream_t st) : s(st) {}
  ~Tmp() {
    for (void* x : p) cudaFreeAsync(x, s);
  }
  template <typename T>
  T* alloc(size_t n) {
    T* x = nullptr;
    pool_alloc(&x, n * sizeof(T), s);
    p.push_back(x);
    return x;
  }
};

template <typename T>
T read1(const T* d, cudaStream_t s) {
  T h;
  cuda_check(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s), "D2H(mesh)");
  cuda_check(cudaStreamSynchronize(s), "cudaStreamSynchronize(mesh)");
  return h;
}

// Builds from DEVICE arrays (nodes [2n], elements [3E], pairs: dirichlet then neumann [2(nd+nn)]).
// Takes ownership of `nodes` (a pool allocation on `s`).
dgb_device_mesh* build(double* nodes, int n_nodes, const int32_t* elements, int E,
                       const int32_t* pairs, int n_dir, int n_neu, int device, cudaStream_t s) {
  std::unique_ptr<dgb_device_mesh, void (*)(dgb_device_mesh*)> owner(new dgb_device_mesh(),
                                                                     dgb_device_mesh_free);
  dgb_device_mesh* m = owner.get();
  m->device = device;
  m->n_nodes = n_nodes;
  m->n_elements = E;
  m->nodes = nodes;  // owned from here on (freed with the mesh on any failure)
  auto fail = [&](int status, const char* msg, long long detail) {
    throw dgb::Error(status, msg, detail);
  };
  {
    Tmp t(s);
    unsigned long long* words = t.alloc<unsigned long long>(8);
    cuda_check(cudaMemsetAsync(words, 0xFF, 8 * sizeof(unsigned long long), s), "memset");
    cuda_check(cudaMemsetAsync(words + 7, 0, sizeof(unsigned long long), s), "memset");
    pool_alloc(&m->elements, std::max<size_t>(3ull * E, 1) * sizeof(int32_t), s);
    if (E > 0) {
      validate_orient_kernel<<<blocks(E), kT, 0, s>>>(nodes, elements, E, n_nodes, m->elements, words);
      cuda_check(cudaGetLastError(), "validate_orient_kernel");
    }
    const unsigned long long ve = read1(words, s);
    if (ve != kNone) {
      if ((ve & 3) == 0) fail(DGB_STATUS_INVALID_TOPOLOGY, "element references a node index outside the node table", static_cast<long long>(ve >> 2));
      fail(DGB_STATUS_DEGENERATE_ELEMENT, "element has (numerically) zero area", static_cast<long long>(ve >> 2));
    }
    const long long M = 3LL * E;
    unsigned long long* keys = t.alloc<unsigned long long>(M);
    unsigned long long* skeys = t.alloc<unsigned long long>(M);
    int32_t* vals = t.alloc<int32_t>(M);
    int32_t* svals = t.alloc<int32_t>(M);
    int32_t* uid = t.alloc<int32_t>(M);
    if (M > 0) {
      halfedge_kernel<<<blocks(M), kT, 0, s>>>(m->elements, E, keys, vals);
      size_t bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, skeys, vals, svals, static_cast<int>(M), 0, 64, s);
      void* scratch = t.alloc<char>(bytes);
      cub::DeviceRadixSort::SortPairs(scratch, bytes, keys, skeys, vals, svals, static_cast<int>(M), 0, 64, s);
      head_kernel<<<blocks(M), kT, 0, s>>>(skeys, M, uid);
      size_t sb = 0;
      cub::DeviceScan::InclusiveSum(nullptr, sb, uid, uid, static_cast<int>(M), s);
      void* ss = t.alloc<char>(sb);
      cub::DeviceScan::InclusiveSum(ss, sb, uid, uid, static_cast<int>(M), s);
      cuda_check(cudaGetLastError(), "edge sort");
      m->n_edges = read1(uid + M - 1, s);
    }
    const int NE = m->n_edges;
    pool_alloc(&m->edges, std::max<size_t>(2ull * NE, 1) * sizeof(int32_t), s);
    pool_alloc(&m->edge_elements, std::max<size_t>(2ull * NE, 1) * sizeof(int32_t), s);
    pool_alloc(&m->element_edges, std::max<size_t>(3ull * E, 1) * sizeof(int32_t), s);
    pool_alloc(&m->edge_kind, std::max<size_t>(NE, 1), s);
    cuda_check(cudaMemsetAsync(m->edge_kind, DGB_EDGE_INTERIOR, std::max<size_t>(NE, 1), s), "memset");
    unsigned long long* ukeys = t.alloc<unsigned long long>(NE);
    if (M > 0) {
      edge_table_kernel<<<blocks(M), kT, 0, s>>>(skeys, svals, uid, M, m->edges, m->edge_elements,
                                                 m->element_edges, ukeys, words + 1);
      cuda_check(cudaGetLastError(), "edge_table_kernel");
    }
    const unsigned long long nm = read1(words + 1, s);
    if (nm != kNone) fail(DGB_STATUS_NON_MANIFOLD, "edge is shared by more than two elements", static_cast<long long>(nm));
    const int NP = n_dir + n_neu;
    if (NP > 0) {
      int32_t* edge_of = t.alloc<int32_t>(NP);
      unsigned long long* dk = t.alloc<unsigned long long>(NP);
      unsigned long long* dks = t.alloc<unsigned long long>(NP);
      int32_t* dv = t.alloc<int32_t>(NP);
      int32_t* dvs = t.alloc<int32_t>(NP);
      boundary_lookup_kernel<<<blocks(NP), kT, 0, s>>>(pairs, NP, ukeys, NE, m->edge_elements, edge_of, dk, dv, words + 2);
      size_t bytes = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dks, dv, dvs, NP, 0, 64, s);
      void* scratch = t.alloc<char>(bytes);
      cub::DeviceRadixSort::SortPairs(scratch, bytes, dk, dks, dv, dvs, NP, 0, 64, s);
      duplicate_kernel<<<blocks(NP), kT, 0, s>>>(dks, NP, words + 2);
      cuda_check(cudaGetLastError(), "boundary lookup");
      const unsigned long long be = read1(words + 2, s);
      if (be != kNone) {
        const int p = static_cast<int>(be >> 2), code = static_cast<int>(be & 3);
        if (code == 1) fail(DGB_STATUS_INVALID_BOUNDARY_SPEC, "boundary list names a node pair that is not a mesh edge", -1);
        int32_t u = 0;
        cuda_check(cudaMemcpyAsync(&u, edge_of + p, sizeof u, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "sync");
        if (code == 2) fail(DGB_STATUS_INVALID_BOUNDARY_SPEC, "boundary list names an interior edge", u);
        fail(DGB_STATUS_INVALID_BOUNDARY_SPEC, "boundary edge tagged more than once", u);
      }
      classify_kernel<<<blocks(NP), kT, 0, s>>>(edge_of, n_dir, NP, m->edge_kind);
    }
    if (NE > 0) {
      missing_kernel<<<blocks(NE), kT, 0, s>>>(m->edge_elements, m->edge_kind, NE, words + 3, words + 7);
      cuda_check(cudaGetLastError(), "missing_kernel");
    }
    const unsigned long long miss = read1(words + 3, s);
    if (miss != kNone) fail(DGB_STATUS_INVALID_BOUNDARY_SPEC, "boundary edge missing from the Dirichlet/Neumann lists", static_cast<long long>(miss));
    m->n_interior = static_cast<int32_t>(read1(words + 7, s));
  }
  return owner.release();
}

struct Guard {
  int prev = -1;
  explicit Guard(int dev) {
    cudaGetDevice(&prev);
    cuda_check(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~Guard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int dgb_device_mesh_build(const double* nodes_xy, int32_t n_nodes, const int32_t* elements,
                          int32_t n_elements, const int32_t* dirichlet_pairs, int32_t n_dirichlet,
                          const int32_t* neumann_pairs, int32_t n_neumann, int32_t device,
                          dgb_device_mesh** out, void* stream) {
  if (out) *out = nullptr;
  return dgb::guarded([&] {
    if (!out || n_nodes < 0 || n_elements < 0 || n_dirichlet < 0 || n_neumann < 0) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "invalid argument");
    }
    if ((n_nodes && !nodes_xy) || (n_elements && !elements) || (n_dirichlet && !dirichlet_pairs) ||
        (n_neumann && !neumann_pairs)) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null array");
    }
    Guard g(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    double* nodes = nullptr;
    pool_alloc(&nodes, std::max<size_t>(2ull * n_nodes, 1) * sizeof(double), s);
    cuda_check(cudaMemcpyAsync(nodes, nodes_xy, 2ull * n_nodes * sizeof(double), cudaMemcpyDefault, s), "copy(nodes)");
    Tmp t(s);
    int32_t* pairs = t.alloc<int32_t>(2ull * (n_dirichlet + n_neumann));
    if (n_dirichlet) cuda_check(cudaMemcpyAsync(pairs, dirichlet_pairs, 8ull * n_dirichlet, cudaMemcpyDefault, s), "copy");
    if (n_neumann) cuda_check(cudaMemcpyAsync(pairs + 2 * n_dirichlet, neumann_pairs, 8ull * n_neumann, cudaMemcpyDefault, s), "copy");
    int32_t* el = t.alloc<int32_t>(3ull * n_elements);
    if (n_elements) cuda_check(cudaMemcpyAsync(el, elements, 12ull * n_elements, cudaMemcpyDefault, s), "copy");
    *out = build(nodes, n_nodes, el, n_elements, pairs, n_dirichlet, n_neumann, device, s);
  });
}

int dgb_device_mesh_refine(const dgb_device_mesh* in, dgb_device_mesh** out, void* stream) {
  if (out) *out = nullptr;
  return dgb::guarded([&] {
    if (!in || !out) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    Guard g(in->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int NN = in->n_nodes, NE = in->n_edges, E = in->n_elements;
    if (static_cast<long long>(NN) + NE > INT32_MAX || 4LL * E > INT32_MAX) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "refined mesh exceeds 32-bit indices");
    }
    double* nodes = nullptr;
    pool_alloc(&nodes, std::max<size_t>(2ull * (NN + NE), 1) * sizeof(double), s);
    const long long nmax = std::max<long long>(2LL * NN, NE);
    if (nmax > 0) refine_nodes_kernel<<<blocks(nmax), kT, 0, s>>>(in->nodes, NN, in->edges, NE, nodes);
    Tmp t(s);
    int32_t* el = t.alloc<int32_t>(12ull * E);
    if (E > 0) refine_elements_kernel<<<blocks(E), kT, 0, s>>>(in->elements, in->element_edges, E, NN, el);
    int32_t* fd = t.alloc<int32_t>(NE + 1);
    int32_t* fn = t.alloc<int32_t>(NE + 1);
    int nd = 0, nn = 0;
    if (NE > 0) {
      boundary_flags_kernel<<<blocks(NE), kT, 0, s>>>(in->edge_kind, NE, fd, fn);
      size_t b1 = 0;
      cub::DeviceScan::ExclusiveSum(nullptr, b1, fd, fd, NE + 1, s);
      void* sc = t.alloc<char>(b1);
      // the extra slot [NE] is scanned too: zero it so its exclusive sum is the total
      cuda_check(cudaMemsetAsync(fd + NE, 0, sizeof(int32_t), s), "memset");
      cuda_check(cudaMemsetAsync(fn + NE, 0, sizeof(int32_t), s), "memset");
      cub::DeviceScan::ExclusiveSum(sc, b1, fd, fd, NE + 1, s);
      cub::DeviceScan::ExclusiveSum(sc, b1, fn, fn, NE + 1, s);
      cuda_check(cudaGetLastError(), "boundary scan");
      nd = read1(fd + NE, s);
      nn = read1(fn + NE, s);
    }
    int32_t* pairs = t.alloc<int32_t>(4ull * (nd + nn));
    if (NE > 0) {
      refine_boundary_kernel<<<blocks(NE), kT, 0, s>>>(in->edge_kind, in->edges, fd, fn, NE, NN, 2 * nd, pairs);
      cuda_check(cudaGetLastError(), "refine kernels");
    }
    *out = build(nodes, NN + NE, el, 4 * E, pairs, 2 * nd, 2 * nn, in->device, s);
  });
}

int dgb_device_mesh_view(const dgb_device_mesh* m, dgb_mesh_arrays* out) {
  return dgb::guarded([&] {
    if (!m || !out) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null argument");
    out->n_nodes = m->n_nodes;
    out->n_elements = m->n_elements;
    out->n_edges = m->n_edges;
    out->n_interior_edges = m->n_interior;
    out->nodes = m->nodes;
    out->elements = m->elements;
    out->edges = m->edges;
    out->edge_kind = m->edge_kind;
    out->edge_elements = m->edge_elements;
    out->element_edges = m->element_edges;
  });
}

int dgb_device_mesh_copy_to_host(const dgb_device_mesh* m, double* nodes, int32_t* elements,
                                 int32_t* edges, uint8_t* edge_kind, int32_t* edge_elements,
                                 int32_t* element_edges) {
  return dgb::guarded([&] {
    if (!m) throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "null mesh");
    Guard g(m->device);
    auto get = [](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) cuda_check(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "D2H(mesh)");
    };
    get(nodes, m->nodes, 16ull * m->n_nodes);
    get(elements, m->elements, 12ull * m->n_elements);
    get(edges, m->edges, 8ull * m->n_edges);
    get(edge_kind, m->edge_kind, static_cast<size_t>(m->n_edges));
    get(edge_elements, m->edge_elements, 8ull * m->n_edges);
    get(element_edges, m->element_edges, 12ull * m->n_elements);
  });
}

void dgb_device_mesh_free(dgb_device_mesh* m) {
  if (!m) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(m->device);
  cudaFree(m->nodes);
  cudaFree(m->elements);
  cudaFree(m->edges);
  cudaFree(m->edge_kind);
  cudaFree(m->edge_elements);
  cudaFree(m->element_edges);
  if (prev >= 0) cudaSetDevice(prev);
  delete m;
}

}  // extern "C"
