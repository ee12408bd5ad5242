/*
 * dgfem_b200.h -- C-ABI of the B200-native interior-penalty DG assembly.
 *
 * This is the drop-in boundary for the reference library's hot path
 * `dgfem::assemble_all` (/root/reference/proj/src/assembly.cpp:725-737) followed by
 * `DgSystem::stiffness()` (assembly.cpp:508-510): mesh + reference tables + coefficients +
 * penalty parameters in, block-sparse stiffness K = (D + C) + R and load vector F out.
 *
 * Every signature uses plain pointers, sizes and POD structs (no C++ or torch types), so the
 * reference's C++ code (or any FFI) can bind it directly; INTEGRATION.md shows the binding.
 *
 * Status codes: 0 = success, otherwise 1 + the numeric value of the reference's
 * `dgfem::ErrorCode` enumerator (errors.hpp:9-27), so the C++ wrapper can rethrow
 * `dgfem::Error(code, message, detail)` 1:1.  CUDA runtime failures use DGB_STATUS_CUDA.
 * The message and the `detail` index of the last failure on the calling thread are available
 * from dgb_last_error_message()/dgb_last_error_detail().
 *
 * Arrays that describe a mesh, tables or outputs are either all HOST pointers (functions whose
 * name contains `host`, and the mesh/reference builders) or all DEVICE pointers (dgb_assemble,
 * dgb_spmv, dgb_bsr_pattern); each function says which.
 */
#ifndef DGFEM_B200_H
#define DGFEM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status codes */
/* 1 + dgfem::ErrorCode (errors.hpp:9-27), in declaration order. */
enum dgb_status {
  DGB_OK = 0,
  DGB_STATUS_INVALID_TOPOLOGY = 1,
  DGB_STATUS_INVALID_BOUNDARY_SPEC = 2,
  DGB_STATUS_NON_MANIFOLD = 3,
  DGB_STATUS_DEGENERATE_ELEMENT = 4,
  DGB_STATUS_UNSUPPORTED_DEGREE = 5,
  DGB_STATUS_INVALID_INDEX = 6,
  DGB_STATUS_DIMENSION_MISMATCH = 7,
  DGB_STATUS_SINGULAR_MATRIX = 8,
  DGB_STATUS_SOLVE_ACCURACY = 9,
  DGB_STATUS_INFLOW_ON_NEUMANN = 10,
  DGB_STATUS_NON_POSITIVE_DIFFUSION = 11,
  DGB_STATUS_INVALID_REACTION = 12,
  DGB_STATUS_NO_EXACT_SOLUTION = 13,
  DGB_STATUS_UNKNOWN_PROBLEM = 14,
  DGB_STATUS_UNKNOWN_METHOD = 15,
  DGB_STATUS_IO_FAILURE = 16,
  DGB_STATUS_INVALID_ARGUMENT = 17,
  DGB_STATUS_CUDA = 100 /* CUDA runtime / launch failure (no reference equivalent) */
};

/* Name of a status ("InflowOnNeumann", ...), matching dgfem::to_string(ErrorCode)
 * (errors.cpp:5-27). */
const char* dgb_status_name(int status);
/* Message / detail of the last failure on this thread (detail = -1 when none),
 * mirroring dgfem::Error::what()/detail() (errors.hpp:35-48). */
const char* dgb_last_error_message(void);
long long dgb_last_error_detail(void);
/* Library version string. */
const char* dgb_version(void);

/* ---------------------------------------------------------------- mesh */
/* Edge kinds, as dgfem::EdgeKind (mesh.hpp:12), stored as one byte per edge. */
enum dgb_edge_kind { DGB_EDGE_INTERIOR = 0, DGB_EDGE_DIRICHLET = 1, DGB_EDGE_NEUMANN = 2 };

/* Flat view of dgfem::Mesh (mesh.hpp:37-49). Same conventions: CCW elements; edges are sorted
 * node pairs (a < b) in lexicographic order; edge_elements = {left, right} with left the lower
 * element index and right = -1 on the boundary; local edge l of an element joins its local
 * vertices (l+1)%3 -> (l+2)%3.  Used with host pointers (mesh builders) and with device
 * pointers (dgb_assemble / dgb_bsr_pattern). */
typedef struct dgb_mesh_arrays {
  int32_t n_nodes;
  int32_t n_elements;
  int32_t n_edges;
  int32_t n_interior_edges;     /* count of DGB_EDGE_INTERIOR edges (sizes the BSR pattern) */
  const double* nodes;          /* [2*n_nodes] x,y interleaved       (Mesh::nodes)          */
  const int32_t* elements;      /* [3*n_elements]                    (Mesh::elements)       */
  const int32_t* edges;         /* [2*n_edges] sorted pairs          (Mesh::edges)          */
  const uint8_t* edge_kind;     /* [n_edges] dgb_edge_kind           (Mesh::edge_kind)      */
  const int32_t* edge_elements; /* [2*n_edges] left,right            (Mesh::edge_elements)  */
  const int32_t* element_edges; /* [3*n_elements]                    (Mesh::element_edges)  */
} dgb_mesh_arrays;

/* Opaque host-side mesh (owns its arrays). */
typedef struct dgb_mesh dgb_mesh;

/* Replaces dgfem::build_mesh (mesh.hpp:62-65, mesh.cpp:51-151): derives the sorted edge table,
 * adjacency and boundary classification, reorienting clockwise elements.  Same checks and
 * error codes: InvalidTopology, DegenerateElement, NonManifold, InvalidBoundarySpec.
 * All pointers are HOST pointers; boundary lists are node pairs (any order). */
int dgb_mesh_build(const double* nodes_xy, int32_t n_nodes, const int32_t* elements,
                   int32_t n_elements, const int32_t* dirichlet_pairs, int32_t n_dirichlet,
                   const int32_t* neumann_pairs, int32_t n_neumann, dgb_mesh** out);

/* The benchmark meshes (BASELINE.json configs): the unit square cut into n x n cells, each
 * split along its (0,0)-(1,1) diagonal into two CCW triangles; nodes numbered row-major.
 * jitter > 0 moves every interior node by independent U[-jitter*h, jitter*h] offsets per
 * coordinate (h = 1/n; config 3 uses 0.2); permute != 0 applies a Fisher-Yates shuffle to the
 * element list before the edge table is built (config 4).  neumann_sides is a bit mask of
 * sides tagged Neumann (1: x=0, 2: x=1, 4: y=0, 8: y=1); the rest is Dirichlet.  The random
 * stream is splitmix64(seed) (documented in DESIGN.md).  HOST.  Also returns the raw
 * (pre-build) arrays through dgb_mesh_raw so the reference build_mesh can be fed the same
 * input. */
int dgb_mesh_unit_square(int32_t n, double jitter, uint64_t jitter_seed, int32_t permute,
                         uint64_t permute_seed, int32_t neumann_sides, dgb_mesh** out);

/* The same construction on [0, lx] x [0, ly] with nx x ny cells (sides 1: x=0, 2: x=lx, 4: y=0,
 * 8: y=ly).  dgb_mesh_unit_square(n, ...) == dgb_mesh_rectangle(n, n, 1, 1, ...).  Used for the
 * weak-scaling global mesh of the multi-GPU benchmark (N x 1 strip of config-sized squares). */
int dgb_mesh_rectangle(int32_t nx, int32_t ny, double lx, double ly, double jitter,
                       uint64_t jitter_seed, int32_t permute, uint64_t permute_seed,
                       int32_t neumann_sides, dgb_mesh** out);

/* Pointers into the mesh's own storage (valid until dgb_mesh_free). */
int dgb_mesh_view(const dgb_mesh* mesh, dgb_mesh_arrays* out);
/* The input that produced the mesh: nodes, elements before reorientation, and the boundary
 * pair lists.  Any pointer may be NULL; counts are always written.  HOST. */
int dgb_mesh_raw(const dgb_mesh* mesh, const double** nodes, int32_t* n_nodes,
                 const int32_t** elements, int32_t* n_elements, const int32_t** dirichlet,
                 int32_t* n_dirichlet, const int32_t** neumann, int32_t* n_neumann);
void dgb_mesh_free(dgb_mesh* mesh);

/* ---------------------------------------------------------------- reference element */
/* Flat view of dgfem::ReferenceElement (reference.hpp:22-77) with the layouts of its public
 * accessors: phi(q,j) = phi[q*nl+j]; dphi(q,j,d) = dphi[(q*nl+j)*2+d];
 * edge_phi(l,o,q,j) = edge_phi[((l*2+o)*nq_edge+q)*nl+j];
 * edge_dphi(l,o,q,j,d) = edge_dphi[(((l*2+o)*nq_edge+q)*nl+j)*2+d]. */
typedef struct dgb_reference_tables {
  int32_t degree;
  int32_t n_local;
  int32_t nq_vol;
  int32_t nq_edge;
  const double* vol_x;      /* [nq_vol]  TriangleRule::x (quadrature.hpp:11-16) */
  const double* vol_y;      /* [nq_vol]  */
  const double* vol_w;      /* [nq_vol]  weights, sum 1/2 */
  const double* edge_t;     /* [nq_edge] Gauss1D::t on [0,1] (quadrature.hpp:26-30) */
  const double* edge_w;     /* [nq_edge] weights, sum 1 */
  const double* phi;        /* [nq_vol*nl]            */
  const double* dphi;       /* [nq_vol*nl*2]          */
  const double* edge_phi;   /* [3*2*nq_edge*nl]       */
  const double* edge_dphi;  /* [3*2*nq_edge*nl*2]     */
} dgb_reference_tables;

typedef struct dgb_reference dgb_reference;

/* Replaces dgfem::ReferenceElement(degree, quad_order) (reference.cpp:87-147): orthonormal
 * Dubiner basis, degree 1..4 (UnsupportedDegree otherwise); quad_order = 0 picks the default
 * rules (volume exact to 2k+2, k+1 edge points), quad_order > 0 a volume rule of that
 * exactness and (quad_order+1)/2 edge points.  HOST. */
int dgb_reference_create(int32_t degree, int32_t quad_order, dgb_reference** out);
int dgb_reference_view(const dgb_reference* ref, dgb_reference_tables* out);
void dgb_reference_free(dgb_reference* ref);

/* ---------------------------------------------------------------- coefficients */
/* Device-evaluable replacement of dgfem::ProblemSpec's std::function callbacks
 * (problems.hpp:19-68), which cannot cross to the device.  Each field is an enum-tagged
 * descriptor; oracle/dg_coeffs.h holds the host twins the oracle feeds to the reference. */
enum dgb_field_kind {
  DGB_FIELD_CONSTANT = 0,    /* value                                                        */
  DGB_FIELD_PER_ELEMENT = 1, /* per_element[e] (piecewise constant; config 5)                */
  DGB_FIELD_FUNCTION = 2     /* analytic family `fn` with parameters p[], evaluated as `mode` */
};
/* Analytic families u(x,y) (each with closed-form gradient and Laplacian). */
enum dgb_function {
  DGB_FN_SIN_SIN = 1,    /* u = p0 sin(pi x) sin(pi y)                                       */
  DGB_FN_TANH_LAYER = 2, /* u = 0.5 (1 - tanh((p0 x + p1 y + p2) / p3))                      */
  DGB_FN_GAUSSIAN = 3,   /* u = exp(-p0 ((x - p1)^2 + (y - p2)^2))                           */
  DGB_FN_AFFINE = 4,     /* u = p0 + p1 x + p2 y                                             */
  DGB_FN_STEP_Y = 5      /* u = (y < p0) ? p1 : p2            (value only)                   */
};
/* What a DGB_FIELD_FUNCTION field returns. */
enum dgb_function_mode {
  DGB_MODE_VALUE = 0,   /* u                                                                 */
  DGB_MODE_SOURCE = 1,  /* q0 u - q1 lap(u) + q2 du/dx + q3 du/dy  (manufactured source with
                           constant alpha = q0, eps = q1, b = (q2, q3))                      */
  DGB_MODE_FLUX_X = 2,  /* q1 du/dx  (conormal flux through x = const sides)                 */
  DGB_MODE_SOURCE_SQUARE = 3 /* the SOURCE value + u^2: the manufactured source of a problem
                           with the nonlinear reaction r(u) = u^2 (the reference's
                           "paper-boundary-layer", problems.cpp:113-118)                     */
};
typedef struct dgb_scalar_field {
  int32_t kind;               /* dgb_field_kind  */
  int32_t fn;                 /* dgb_function    */
  int32_t mode;               /* dgb_function_mode */
  int32_t pad_;
  double value;               /* DGB_FIELD_CONSTANT */
  double p[4];                /* function parameters */
  double q[4];                /* mode parameters     */
  const double* per_element;  /* DGB_FIELD_PER_ELEMENT: [n_elements] (device pointer for
                                 dgb_assemble, host pointer for the host entry points) */
} dgb_scalar_field;

enum dgb_vector_kind {
  DGB_VEC_CONSTANT = 0, /* b = (p0, p1)                                                     */
  DGB_VEC_AFFINE = 1,   /* b = (p0 + p2 x + p3 y, p1 + p4 x + p5 y)         (config 3)        */
  DGB_VEC_TRIG = 2      /* b = (cos(p0 y), sin(p1 x))                        (config 5)        */
};
typedef struct dgb_vector_field {
  int32_t kind;
  int32_t pad_;
  double p[6];
} dgb_vector_field;

/* The coefficient set of ProblemSpec (problems.hpp:52-68) that assemble_all reads.
 * diffusion and linear_reaction must be CONSTANT or PER_ELEMENT (every problem in the
 * reference registry and every BASELINE config is).  For a PER_ELEMENT diffusion the edge
 * value is 0.5 (eps_L + eps_R) on interior edges and eps_K on boundary edges (SURVEY.md §8
 * "Config-5 policy"). */
typedef struct dgb_problem {
  dgb_scalar_field diffusion;       /* eps   > 0 */
  dgb_vector_field advection;       /* b         */
  dgb_scalar_field linear_reaction; /* alpha >= 0 */
  dgb_scalar_field source;          /* f         */
  dgb_scalar_field dirichlet;       /* gD        */
  dgb_scalar_field neumann;         /* gN        */
} dgb_problem;

/* ---------------------------------------------------------------- parameters */
/* dgfem::DgMethod (assembly.hpp:15) and dgfem::DgParameters (assembly.hpp:29-35). */
enum dgb_method { DGB_SIPG = 0, DGB_NIPG = 1, DGB_IIPG = 2 };
/* What to do when b.n < -tol at a point of a Neumann edge (assembly.cpp:386-397). */
enum dgb_neumann_inflow {
  DGB_INFLOW_ERROR = 0, /* reference behaviour: InflowOnNeumann, detail = lowest edge index   */
  DGB_INFLOW_DROP = 1   /* Neumann boundary treated as outflow-only: no convection terms on it */
};
typedef struct dgb_params {
  int32_t method;         /* dgb_method            */
  int32_t degree;
  double kappa;           /* -1 SIPG, +1 NIPG, 0 IIPG */
  double sigma_interior;
  double sigma_boundary;
  int32_t neumann_inflow; /* dgb_neumann_inflow    */
  int32_t pad_;
} dgb_params;

/* Replaces dgfem::set_parameters (assembly.cpp:483-506): per-method defaults,
 * sigma_boundary = 2 sigma_interior; InvalidArgument for degree < 1. */
int dgb_set_parameters(int32_t method, int32_t degree, dgb_params* out);

/* ---------------------------------------------------------------- BSR output */
/* Block-sparse stiffness: block row e holds the diagonal block and one block per interior
 * edge neighbour, block columns sorted ascending, nl x nl row-major FP64 blocks.  Expands 1:1
 * to the reference's stiffness() CSR (sorted columns, explicit zeros included). */
typedef struct dgb_bsr {
  int32_t n_block_rows;   /* = n_elements */
  int32_t block_dim;      /* = n_local    */
  int64_t nnzb;           /* = n_elements + 2 * n_interior_edges */
  int32_t* row_ptr;       /* [n_block_rows + 1] */
  int32_t* col;           /* [nnzb]             */
  double* val;            /* [nnzb * block_dim * block_dim] */
} dgb_bsr;

/* Number of BSR blocks for a mesh. */
int64_t dgb_bsr_nnzb(int32_t n_elements, int32_t n_interior_edges);

/* ---------------------------------------------------------------- device plan */
/* A plan owns the device-resident reference-contraction tensors derived from one set of
 * reference tables, plus scratch (scan partials, error word).  Not re-entrant across host
 * threads; results are bitwise reproducible run to run (no floating-point atomics). */
typedef struct dgb_plan dgb_plan;

/* tables: HOST pointers (e.g. dgb_reference_view, or the reference's own ReferenceElement
 * accessors).  device: CUDA device ordinal.  Degrees 1..4. */
int dgb_plan_create(const dgb_reference_tables* tables, int32_t device, dgb_plan** out);
void dgb_plan_destroy(dgb_plan* plan);

/* Full assembly on `stream` (a cudaStream_t; NULL = legacy default stream): writes the BSR
 * pattern and values of K = (D + C) + R into `out` (DEVICE buffers sized by dgb_bsr_nnzb) and
 * F into rhs[n_elements * n_local] (DEVICE).  mesh and the per-element pointers of problem are
 * DEVICE pointers.  Asynchronous: returns after enqueueing; call dgb_plan_status to wait
 * and collect InflowOnNeumann (only possible with DGB_INFLOW_ERROR and Neumann edges). */
int dgb_assemble(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                 const dgb_params* params, dgb_bsr* out, double* rhs, void* stream);

/* Per-term assembly: the reference's assemble_diffusion / assemble_convection /
 * assemble_reaction (assembly.hpp:72-95, assembly.cpp:512-641) as matrices.  `terms` is a mask
 * of dgb_term; K gets exactly the selected terms' sum in K's full pattern: the coefficients of
 * the other terms are zeroed (eps = 0 removes every diffusion volume and face term, b = 0 every
 * transport and upwind term, alpha = 0 the reaction), so their entries are exact zeros and, e.g.,
 * DGB_TERM_DIFFUSION gives the reference's D on its own pattern.  F is the load vector of that
 * modified problem (not the reference's per-term F_D / F_C, which assemble_all discards).
 * Otherwise as dgb_assemble. */
enum dgb_term { DGB_TERM_DIFFUSION = 1, DGB_TERM_CONVECTION = 2, DGB_TERM_REACTION = 4, DGB_TERM_ALL = 7 };
int dgb_assemble_terms(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                       const dgb_params* params, int32_t terms, dgb_bsr* out, double* rhs,
                       void* stream);

/* Shard form of dgb_assemble: block rows [row_begin, row_end) only.  `out`
 * holds those rows (row_ptr relative to the shard, starting at 0; block columns global) and
 * rhs their F slices; out->nnzb from dgb_count_blocks_host.  The mesh arrays are the full mesh
 * (device).  No collective is needed: shards are independent and their global block offsets
 * are a prefix sum of the shard block counts. */
int dgb_assemble_rows(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                      const dgb_params* params, int32_t row_begin, int32_t row_end, dgb_bsr* out,
                      double* rhs, void* stream);

/* Number of BSR blocks of block rows [row_begin, row_end) of a HOST mesh (-1 on bad input). */
int64_t dgb_count_blocks_host(const dgb_mesh_arrays* mesh, int32_t row_begin, int32_t row_end);

/* Waits for the plan's last dgb_assemble on `stream` and returns its status
 * (DGB_STATUS_INFLOW_ON_NEUMANN with detail = lowest offending edge, as the reference's
 * deterministic chunk merge reports it). */
int dgb_plan_status(dgb_plan* plan, void* stream);

/* Measurement hook: the next dgb_assemble calls record `start` / `stop` (cudaEvent_t, NULL
 * to disable) on their stream immediately before / after the block-row kernel, so a caller
 * can time that kernel with CUDA events on the launching stream (bench.py's roofline). */
int dgb_plan_set_kernel_events(dgb_plan* plan, void* start, void* stop);

/* Plan options.  DGB_OPTION_FORCE_GENERIC_KERNEL = 1: run the generic (any quadrature) block-row
 * kernel even where a specialised one exists (used by the tests to check both). */
enum dgb_plan_option {
  DGB_OPTION_FORCE_GENERIC_KERNEL = 1,
  DGB_OPTION_MIN_BLOCKS = 2, /* tuning knob: register budget of the P2 kernel (CTAs per SM) */
  DGB_OPTION_L2_POLICY = 3,  /* bit 0: keep node coordinates persisting in L2 (access-policy
                                window, carve-out sized to the node array at bind time);
                                bit 1: evict-first L2 hint on the output stream;
                                bit 2: L2 hints on the P1 kernel's loads (node gathers
                                evict-last, per-element records evict-first);
                                -1 (default): evict-first for odd block sizes only; the
                                P1 persistent kernel on a bound mesh instead keeps its node
                                gathers evict-last in a persisting carve-out of at most 56 MiB
                                (a process-wide device limit set at bind time, released when
                                the plan is destroyed) */
  DGB_OPTION_BATCH_FUSE = 4, /* dgb_assemble_batch on the tensor-core kernels (default 1): sets
                                with equal penalties share the per-element work and each CTA
                                writes every set; 0 = one CTA row per set (grid.y = n) */
  DGB_OPTION_WARP_SPECIALIZED = 5, /* P-form tensor-core kernels on a bound mesh (default 1:
                                      8 producer + 4 consumer warps for config 2's kernel);
                                      0 = the monolithic kernel; 4..12 = producer warps of 16,
                                      100 p + c = p producers and c consumers (tuning) */
  DGB_OPTION_P1_PIPELINE = 6, /* P1 kernels on a bound mesh (default 1): persistent kernel with
                                 the record and node gathers in flight one chunk ahead
                                 (asynchronous copies), 12 warps per SM at 166 registers;
                                 0 = the one-shot kernel */
  DGB_OPTION_L2_CARVEOUT_MB = 7, /* cap (MiB) on the persisting-L2 carve-out that L2 policy bits
                                    0 / 2 set up at bind time; 0 = the node array (tuning) */
  DGB_OPTION_GEOMETRY_CACHE = 8, /* P1 persistent kernel (default 1): dgb_plan_bind_mesh also
                                    builds the bound rows' geometry record (own vertices and,
                                    per edge, the neighbour's G^T n; 96 B per element, in
                                    32-row chunks) so that an assembly reads its geometry with
                                    coalesced 16-byte copies: no node gathers or neighbour
                                    Jacobians per assembly (the same expressions; results
                                    agree to the last bits); 0 = gather from mesh->nodes at
                                    every assembly.  With 1, rebind after changing mesh->nodes */
  DGB_OPTION_PROFILE_ABLATE = 1000 /* DIAGNOSTICS ONLY -- RESULTS ARE WRONG while nonzero: skip
                                      kernel parts to attribute time (bits: 1 block stores,
                                      2 source evaluation, 4 neighbour blocks, 8 diagonal
                                      block, 16 exit after the prologue, 32 after own geometry) */
};
int dgb_plan_set_option(dgb_plan* plan, int32_t option, int32_t value);

/* Binds block rows [row_begin, row_end) of `mesh` (DEVICE arrays) to the plan, computing once
 * (on `stream`) what depends only on the mesh: the BSR row_ptr (count + scan) and an element
 * adjacency record (neighbour per local edge, its vertex opposite the shared edge, edge kinds,
 * orientations and block slots; 32 B per element).  Later dgb_assemble / dgb_assemble_rows calls on the same mesh arrays and
 * rows run as one kernel that reads the record with coalesced loads instead of the dependent
 * element_edges -> edge_elements -> elements gathers, and copy the bound row_ptr into their
 * output.  For P1 the bind also builds the rows' geometry record (DGB_OPTION_GEOMETRY_CACHE).
 * Rebind (or unbind) if elements / element_edges / edge_kind / edge_elements change, or, for
 * P1, if the node coordinates change (a plan bound to another `nodes` pointer gathers from
 * mesh->nodes as before). */
int dgb_plan_bind_mesh(dgb_plan* plan, const dgb_mesh_arrays* mesh, int32_t row_begin,
                       int32_t row_end, void* stream);
int dgb_plan_unbind_mesh(dgb_plan* plan);

/* Several assemblies of block rows [row_begin, row_end) of the same mesh and problem with
 * different parameter sets (SIPG / NIPG / IIPG, penalty sweeps): outs[i], rhs[i] receive the
 * system of params[i], exactly as n calls of dgb_assemble_rows would.  With the rows bound
 * (dgb_plan_bind_mesh), the P2 tensor-core kernel and n <= 4 this is ONE launch (grid.y = n:
 * no per-launch tail or launch gap between the assemblies); otherwise n calls.  DEVICE. */
int dgb_assemble_batch(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_problem* problem,
                       const dgb_params* params, int32_t n, int32_t row_begin, int32_t row_end,
                       dgb_bsr* outs, double* const* rhs, void* stream);

/* Device operations (kernels, CUB scan kernels) the plan's last dgb_assemble* call launched:
 * 1 with a bound pattern, 4 without (bench.py's gpu_launches). */
int32_t dgb_plan_launch_count(const dgb_plan* plan);

/* y = K x with the BSR from dgb_assemble (DEVICE pointers), on `stream`.  Replaces
 * dgfem::matvec(stiffness(), x) (sparse.cpp:116-129). */
int dgb_spmv(const dgb_bsr* a, const double* x, double* y, void* stream);

/* One-shot drop-in for `assemble_all(mesh, ref, problem, params)` + `stiffness()` with HOST
 * buffers in and out: uploads the mesh, tables and per-element coefficients, assembles on
 * `device`, downloads K (BSR) and F.  Output buffers are caller-allocated host memory sized
 * by dgb_bsr_nnzb.  Synchronous; returns the reference's error code on failure. */
int dgb_assemble_all_host(const dgb_mesh_arrays* mesh, const dgb_reference_tables* tables,
                          const dgb_problem* problem, const dgb_params* params, int32_t device,
                          dgb_bsr* out, double* rhs);

/* ---- Nonlinear reaction ------------------------------------------
 * The reaction r(u) of `alpha u - div(eps grad u) + b.grad u + r(u) = f`
 * (ProblemSpec::nonlinear_reaction, problems.hpp:38-41, 62).  std::function callbacks cannot
 * run on the device, so the reference's reactions are enumerated with their exact
 * expressions:
 *   ZERO    r = 0,          r' = 0            (test_nonlinear.cpp zero_reaction)
 *   LINEAR  r = u,          r' = 1            (test_nonlinear.cpp "linear reaction")
 *   SQUARE  r = u * u,      r' = 2.0 * u      (problems.cpp:125-127, paper-boundary-layer)
 *   CUBIC   r = u * u * u,  r' = 3.0 * u * u  (test_nonlinear.cpp cubic_reaction)       */
enum {
  DGB_REACTION_ZERO = 0,
  DGB_REACTION_LINEAR = 1,
  DGB_REACTION_SQUARE = 2,
  DGB_REACTION_CUBIC = 3
};

typedef struct dgb_reaction {
  int32_t kind;
  int32_t pad_;
} dgb_reaction;

/* Replaces dgfem::assemble_nonlinear(coef, mesh, ref, reaction) (nonlinear.cpp:11-107):
 *   H_i   = sum_q det w_q r(u_h(x_q)) phi_i(x_q)            -> h[n_elements * nl]
 *   HJ_ij = sum_q det w_q r'(u_h(x_q)) phi_j phi_i           -> hj, block-diagonal BSR
 * with u_h = sum_j coef[e*nl + j] phi_j.  HJ has one nl x nl block per element: on return
 * hj->row_ptr[e] = e and hj->col[e] = e (the reference's CSR expands 1:1 from it).
 * DEVICE pointers (mesh arrays, coef, h, hj arrays), asynchronous on `stream`.
 * hj->n_block_rows must equal n_elements, hj->nnzb == n_elements, hj->block_dim == nl
 * (else DGB_STATUS_DIMENSION_MISMATCH, like the reference's coefficient-length check).   */
int dgb_assemble_nonlinear(dgb_plan* plan, const dgb_mesh_arrays* mesh, const double* coef,
                           int64_t n_coef, const dgb_reaction* reaction, double* h,
                           dgb_bsr* hj, void* stream);

/* The same with HOST buffers in and out (synchronous): uploads mesh and coef, downloads H and
 * HJ.  n_coef must equal n_elements * nl (DGB_STATUS_DIMENSION_MISMATCH otherwise). */
int dgb_assemble_nonlinear_host(const dgb_mesh_arrays* mesh, const dgb_reference_tables* tables,
                                const double* coef, int64_t n_coef,
                                const dgb_reaction* reaction, int32_t device, double* h,
                                dgb_bsr* hj);

/* ---- Solve of the assembled system and the Newton driver ----------
 * The reference solves with Eigen's SparseLU (direct_solve, sparse.cpp:154-217).  Here the
 * BSR system is solved on the device by restarted GMRES(m) with a block-Jacobi
 * preconditioner (the inverses of the nl x nl diagonal blocks), accepted under the
 * reference's own accuracy contract:
 *     ||A x - b||_2 <= 1e-10 (||A||_F ||x||_2 + ||b||_2)      (sparse.cpp:201-214)
 * and the same errors: DimensionMismatch, SingularMatrix (a zero pivot in a diagonal block;
 * detail = the scalar row), SolveAccuracy (the bound is not met within max_iterations).  */
typedef struct dgb_solve_options {
  double tolerance_scale;  /* stop at tolerance_scale * the contract bound (default 0.1)   */
  int32_t max_iterations;  /* total Krylov iterations (default 20000)                     */
  int32_t restart;         /* GMRES(m) restart length m (default 30, <= 200)              */
  int32_t preconditioner;  /* DGB_PRECOND_*: right preconditioner (default: block SGS)        */
  int32_t pad_;
} dgb_solve_options;
/* Right preconditioners of dgb_solve: block Jacobi (the inverses of the diagonal blocks), or one
 * symmetric block Gauss-Seidel sweep in a multicolour order of the block rows (a greedy colouring
 * of the BSR graph: rows of one colour are independent, so each colour is one parallel step). */
enum dgb_preconditioner { DGB_PRECOND_BLOCK_JACOBI = 0, DGB_PRECOND_BLOCK_SGS = 1 };

typedef struct dgb_solve_info { /* SolveInfo (sparse.hpp:55-59) + the Krylov counters      */
  double defect_norm2;
  double defect_norm_inf;
  double bound;
  int32_t iterations;
  int32_t restarts;
} dgb_solve_info;

/* Fills the defaults above. */
void dgb_solve_options_default(dgb_solve_options* opt);

/* Replaces direct_solve(a, rhs, &info) (sparse.cpp:154-217): solves A x = b for the BSR `a`
 * from dgb_assemble (DEVICE pointers; sorted block columns with a diagonal block in every
 * row).  x (device, n = n_block_rows * block_dim) holds the initial guess on entry (zeros
 * are fine) and the solution on return.  Synchronises `stream`.  opt may be NULL. */
int dgb_solve(const dgb_bsr* a, const double* b, double* x, const dgb_solve_options* opt,
              dgb_solve_info* info, void* stream);

typedef struct dgb_newton_config { /* NewtonConfig (nonlinear.hpp:16-26)                   */
  int32_t max_iterations;          /* 50                                                   */
  int32_t use_legacy_check;        /* 0: legacy_check unset                                */
  double residual_tolerance;       /* 1e-10 on ||Res||_2                                   */
  double step_tolerance;           /* 1e-12 on ||w||_2                                     */
  double legacy_check;             /* the bound on ||J w + Res||_2 when use_legacy_check    */
} dgb_newton_config;

typedef struct dgb_newton_report { /* NewtonReport (nonlinear.hpp:28-33)                   */
  int32_t iterations;
  int32_t converged;
  double final_residual;
  double* residual_history;        /* HOST array, capacity max_iterations (may be NULL)    */
  int32_t linear_iterations;       /* Krylov iterations over all Newton steps              */
  int32_t pad_;
} dgb_newton_report;

void dgb_newton_config_default(dgb_newton_config* cfg);

/* Replaces newton_solve(system, mesh, ref, reaction, config, initial_guess)
 * (nonlinear.cpp:109-176) for K = stiffness() and F of dgb_assemble (DEVICE pointers) on the
 * mesh the plan was built for: J w = -Res, u <- u + w, Res = K u + H(u) - F, J = K + HJ(u),
 * with the inner solves of dgb_solve.  coef (device, n) holds the initial guess (zeros = the
 * reference's empty guess) and returns the iterate.  Synchronises `stream`. */
int dgb_newton_solve(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_bsr* k,
                     const double* f, const dgb_reaction* reaction,
                     const dgb_newton_config* config, const dgb_solve_options* inner,
                     double* coef, dgb_newton_report* report, void* stream);

/* ---- Postprocessing --------------------------------------------- */

/* The quadrature order l2_error integrates with for ReferenceElement(degree, quad_order):
 * max(2k + 3, volume_rule().degree + 1) (postprocess.cpp:22-23; rule degrees as
 * triangle_rule, quadrature.cpp:46-154).  Create the plan for dgb_l2_error from
 * dgb_reference_create(degree, dgb_l2_quad_order(degree, quad_order)). */
int32_t dgb_l2_quad_order(int32_t degree, int32_t quad_order);

/* Replaces l2_error(coef, mesh, ref, exact) (postprocess.cpp:14-50): out[0] = ||u_h - u||_L2,
 * out[1] = max_element_diameter(mesh) (mesh.cpp:259-265).  `plan` carries the sharper rule
 * (dgb_l2_quad_order); exact = the exact solution's value as a scalar field.  DEVICE mesh
 * and coef, HOST out[2]; synchronises `stream`.  n_coef != n_elements * nl ->
 * DGB_STATUS_DIMENSION_MISMATCH. */
int dgb_l2_error(dgb_plan* plan, const dgb_mesh_arrays* mesh, const double* coef, int64_t n_coef,
                 const dgb_scalar_field* exact, double* out, void* stream);

/* Replaces project(mesh, ref, f) (postprocess.cpp:56-81): coef[e*nl + j] =
 * sum_q w_q f(x_q) phi_qj with the plan's volume rule.  DEVICE pointers, asynchronous. */
int dgb_project(dgb_plan* plan, const dgb_mesh_arrays* mesh, const dgb_scalar_field* f,
                double* coef, void* stream);

/* Replaces eval_solution(coef, ref, element, xhat, yhat) (postprocess.cpp:83-93) for a batch
 * of n points: values[i] = u_h(element[i]; xhat[i], yhat[i]).  DEVICE pointers; synchronises
 * `stream`.  An element outside [0, n_elements) -> DGB_STATUS_INVALID_INDEX, detail = the
 * first offending point. */
int dgb_eval_solution(const double* coef, int32_t degree, int32_t n_elements, int64_t n,
                      const int32_t* elements, const double* xhat, const double* yhat,
                      double* values, void* stream);

/* ---- Mesh topology on the device -------------------------------- */
typedef struct dgb_device_mesh dgb_device_mesh;

/* Replaces build_mesh(nodes, elements, dirichlet, neumann) (mesh.cpp:51-151) on `device`:
 * the same validation (InvalidTopology / DegenerateElement / NonManifold /
 * InvalidBoundarySpec with the reference's details), CCW reorientation, lexicographic edge
 * numbering, edge_elements, element_edges and edge kinds -- bit-identical arrays, resident in
 * HBM (view them with dgb_device_mesh_view and pass the view to dgb_assemble).  Inputs may be
 * HOST or DEVICE pointers (copied; cudaMemcpyDefault).  Synchronises `stream`. */
int dgb_device_mesh_build(const double* nodes_xy, int32_t n_nodes, const int32_t* elements,
                          int32_t n_elements, const int32_t* dirichlet_pairs, int32_t n_dirichlet,
                          const int32_t* neumann_pairs, int32_t n_neumann, int32_t device,
                          dgb_device_mesh** out, void* stream);

/* Replaces uniform_refine(mesh) (mesh.cpp:153-187): midpoint refinement (4 children per
 * element, boundary edges split in edge order), then the device build_mesh above. */
int dgb_device_mesh_refine(const dgb_device_mesh* in, dgb_device_mesh** out, void* stream);

/* DEVICE-pointer view (valid until dgb_device_mesh_free). */
int dgb_device_mesh_view(const dgb_device_mesh* mesh, dgb_mesh_arrays* out);
/* Copies the arrays into HOST buffers sized by the view's counts (any pointer may be NULL). */
int dgb_device_mesh_copy_to_host(const dgb_device_mesh* mesh, double* nodes, int32_t* elements,
                                 int32_t* edges, uint8_t* edge_kind, int32_t* edge_elements,
                                 int32_t* element_edges);
void dgb_device_mesh_free(dgb_device_mesh* mesh);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* DGFEM_B200_H */
