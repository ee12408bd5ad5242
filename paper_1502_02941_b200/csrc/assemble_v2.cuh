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

// Profiling ablations (dgb_plan_set_option(DGB_OPTION_PROFILE_ABLATE), results WRONG while
// set) exist only in a tuning build (-DDGB_TUNING, see tools/README.md); in the shipped library
// every ablation test is the constant 0 and compiles away.
#ifdef DGB_TUNING
#define DGB_ABLATE(bits) (P.ablate & (bits))
#else
#define DGB_ABLATE(bits) 0
#endif

namespace dgb {
namespace v2 {

// Flat layout of the tensor parameter block (offsets in doubles, all compile-time).  FULL =
// false (the tensor-core P2 kernel): the element-matrix tensors S .. P live in the B-operand
// table instead, and the parameter block keeps only the basis / quadrature tables -- a large
// __grid_constant__ block is re-read at every CTA launch (tools/microbench/launch_cost.cu).
template <int NL, int NQV, int NQE, bool TRIG, bool FULL = true>
struct Lay {
  static constexpr int N2 = NL * NL;
  static constexpr bool kHasP = FULL && !TRIG && NL <= 10;   // face mass tensors (constant b)
  static constexpr bool kHasTA = FULL && !TRIG && NL <= 10;  // affine transport tensors
  static constexpr int S = 0;                                   // 3: S00, S01 + S10, S11
  static constexpr int M = S + (FULL ? 3 : 0) * N2;             // 1: mass
  static constexpr int W = M + (FULL ? 1 : 0) * N2;             // 6: kappa Q^T - Q  [l][a]
  static constexpr int T = W + (FULL ? 6 : 0) * N2;             // 2: transport (constant b)
  static constexpr int TA = T + (FULL && !TRIG ? 2 : 0) * N2;   // 4: affine transport [a][c]
  static constexpr int P = TA + (kHasTA ? 4 : 0) * N2;          // 3: face mass [l]
  static constexpr int PHI = P + (kHasP ? 3 : 0) * N2;          // [q][i]
  static constexpr int DPHI = PHI + NQV * NL;               // [q][a][i]      (TRIG only)
  static constexpr int EPHI = DPHI + (TRIG ? NQV * 2 * NL : 0);  // [l][p][i]
  static constexpr int EDPHI = EPHI + 3 * NQE * NL;         // [l][p][a][i]
  static constexpr int EDW = EDPHI + 3 * NQE * 2 * NL;        // [l][p][a][i] w_p-scaled
  static constexpr int VX = EDW + 3 * NQE * 2 * NL;
  static constexpr int VY = VX + NQV;
  static constexpr int VW = VY + NQV;
  static constexpr int ET = VW + NQV;
  static constexpr int EW = ET + NQE;
  static constexpr int TOTAL = EW + NQE;
};

template <int NL, int NQV, int NQE, bool TRIG, bool FULL>
struct Tab {
  double x[Lay<NL, NQV, NQE, TRIG, FULL>::TOTAL];
};

// The tensor-core kernel (P2, constant velocity) takes the compact parameter block.
constexpr bool full_tensors(int NL, int BK) {
  return !((NL == 6 && BK == 0) || (NL == 10 && (BK == 0 || BK == 1)) || (NL == 15 && BK == 2));
}

// One assembly of a launch: its penalty parameters and its outputs.  A launch assembles
// n_batch parameter sets of the same mesh and problem (grid.y = n_batch; the tensor-core
// kernel only, whose kappa-dependent terms live in the per-set B operand `bfrag`).
constexpr int kMaxBatch = 4;
struct MethodOut {
  int32_t* row_ptr;              // output row pointer of the launch's rows
  int32_t* col;
  double* val;
  double* rhs;
  const double* bfrag;           // DMMA B fragments (diagonal: kappa-folded W) [ks][nt][lane]
  double kappa, sigma_i, sigma_b;
};

template <int NL, int NQV, int NQE, bool TRIG, bool FULL>
struct Params2 {
  const double* nodes;
  const int32_t* elements;
  const uint8_t* edge_kind;
  const int32_t* edge_elements;
  const int32_t* element_edges;
  const int32_t* row_ptr_src;    // bound pattern (dgb_plan_bind_mesh) copied to row_ptr, or null
  const int4* adj_nb;            // bound adjacency: neighbour per local edge, .w = kinds | lf << 2
  const int4* adj_op;            // bound adjacency: neighbour's vertex opposite the shared edge
  const double2* geo;            // bound vertex coordinates per 32-row chunk [chunk][6][32]: own
                                 // vertices 0..2, the neighbours' opposite vertices 3..5; or null
  unsigned long long* err_edge;  // epoch << 32 | ~edge, max-reduced (lowest edge wins)
  unsigned long long* diag;      // tuning builds: per-warp timing record, or null
  unsigned long long epoch;
  int32_t n_elements;
  int32_t row_begin, row_end;  // block rows [row_begin, row_end) of this launch (a shard)
  int32_t drop_neumann;
  int32_t evict_first;           // L2 evict-first hint on the output stream
  int32_t ablate;                // profiling diagnostics only (wrong results): see dg_assembly.cu
  int32_t load_hints;            // L2 hints on loads: gathers evict-last, streamed records evict-first
  const double* tr_src;          // the plan's neighbour trace table (the kernel's `tr`), or null
  int32_t n_batch;
  MethodOut bt[kMaxBatch];
  dgb_problem prob;
  Tab<NL, NQV, NQE, TRIG, FULL> t;
};

// Staging stride (doubles) per lane: even, so 16-byte chunks stay aligned.
template <int N2>
struct Stage {
  static constexpr int kStride = (N2 % 2 == 0) ? N2 + 2 : N2 + 1;
};

// Bulk asynchronous shared -> global copies (the TMA engine; SASS UBLKCP).  Each lane hands
// its own contiguous staged block to the copy engine and later waits only on its own group.
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
// L2 policy for the output stream: written once, never re-read by the kernel -> evict first,
// so the stream does not push the mesh arrays (gathered again by neighbours) out of L2.
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long evict_last_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
// Loads with an L2 eviction-priority hint.  Gathered data (node coordinates, read by several
// elements in random order on a permuted mesh) is kept with evict-last; records read once per
// element (connectivity, adjacency, row pointers) go evict-first without an L1 allocation.
__device__ __forceinline__ double2 ld_hint(const double2* p, unsigned long long pol) {
  double2 r;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;\n" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int4 ld_stream(const int4* p, unsigned long long pol) {
  int4 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;\n"
      : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_stream(const int* p, unsigned long long pol) {
  int r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;\n" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void bulk_store(void* g, const void* sm, unsigned bytes,
                                           bool evict_first = false) {
  if (evict_first) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;\n"
                 :: "l"(g), "r"(smem_addr(sm)), "r"(bytes), "l"(evict_first_policy()) : "memory");
  } else {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n"
                 :: "l"(g), "r"(smem_addr(sm)), "r"(bytes) : "memory");
  }
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// Per-lane asynchronous global -> shared copies (LDGSTS): the persistent kernels land the next
// chunk's records and node coordinates in shared memory without holding registers.
__device__ __forceinline__ void cp_async16(void* sm, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(smem_addr(sm)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(void* sm, const void* g, unsigned long long pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" :: "r"(smem_addr(sm)), "l"(g), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async4(void* sm, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" :: "r"(smem_addr(sm)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// One 32-element chunk's bound-mesh records and gathered node coordinates, as landed in shared
// memory by the persistent kernels: adj_nb [32] int4, adj_op [32] int4, elements [96],
// row_ptr [32], row_ptr + 1 [32] (ints), then the nodes [6][32] double2 (own vertices 0..2,
// the neighbours' opposite vertices 3..5).
// 16-byte rows of the bound geometry record per element (dg_assembly.cu geometry_kernel): the
// vertices (3) and the neighbours' G^T n (3); with DGB_GEO_RECIPROCALS also (1/det, 1/h_0),
// (1/h_1, 1/h_2).  Measured on config 4 (same-box A/B): with the reciprocals in the record the
// kernel moves 5.98 TB/s of DRAM traffic, 92% of the copy bandwidth, at 0.660 ms; recomputing
// them (one rcp and three rsqrt Newton chains per element) for 32 B per element less takes
// 0.637 ms.  The bytes are worth more than the instructions, so they are recomputed.
#ifndef DGB_GEO_RECIPROCALS
#define DGB_GEO_RECIPROCALS 0
#endif
constexpr int kGeoRows = DGB_GEO_RECIPROCALS ? 8 : 6;

struct ChunkRec {
  static constexpr int kNb = 0, kOp = 128, kV = 256, kRp = 352, kRpn = 384, kIdxInts = 416;
  static constexpr int kIdx = kIdxInts / 2;      // doubles
  static constexpr int kNode = 32 * 6 * 2;       // doubles
  static constexpr int kNode2 = 32 * kGeoRows * 2;  // doubles (geometry record)
};

__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void fence_smem_to_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// Writes this lane's staged block (N2 doubles at `st`) to val[base ..] (base < 0: none).
// Even N2: one bulk copy per lane (block starts are 16-byte aligned: N2 * 8 % 16 == 0);
// odd N2: the warp-cooperative flush below.
template <int N2>
__device__ __forceinline__ void write_block(const double* stw, const double* st, long long base,
                                            double* val, int lane);

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

// Per-warp shared-memory layout of the block-row kernel (doubles).
template <int N2>
__device__ __forceinline__ void write_block(const double* stw, const double* st, long long base,
                                            double* val, int lane, bool ef = false) {
  if constexpr (N2 % 2 == 0) {
    fence_smem_to_async();
    if (base >= 0) bulk_store(val + base, st, N2 * sizeof(double), ef);
  } else {
    flush_blocks<N2>(stw, base, val, lane);
  }
}

template <int NL, int NQV, int NQE, int BK>
struct Smem {
  static constexpr int N2 = NL * NL;
  static constexpr int SS = Stage<N2>::kStride;               // staging stride per lane
  static constexpr int NF = BK == 0 ? 8 : 7 + 2 * NQE;         // stashed coefficients per edge
  // even N2: one staged block per lane (bulk-copied per lane); odd N2 (P1): the warp's whole
  // contiguous row range (<= 4 blocks per lane), bulk-copied once per warp
  // (the tensor-core path writes from fragments: never row mode, whatever N2's parity)
  static constexpr bool kRowMode = N2 % 2 == 1 &&
                                   !((NL == 6 && BK == 0) || (NL == 10 && (BK == 0 || BK == 1)) ||
                                     (NL == 15 && BK == 2));
  // FP64 tensor-core (DMMA m8n8k4) path for P2 with constant velocity: every block (diagonal:
  // 15 terms; neighbour: 5 terms x 3 possible lf, zero-padded) is one [32 x 16] . [16 x 36]
  // product whose fragments are stored straight to global -- no block staging at all
  // Tensor-core path: P2 with constant velocity, P3 with constant or affine velocity.
  //  P-form (constant b): diagonal S0 S1 S2 M T0 T1 W[6] P[3] (15), neighbour X Y0 Y1 Z0 Z1 (5)
  //  U-form (affine b):   diagonal S0 S1 S2 M T0 T1 TA[4] W[6] U[3][NQE] (22 + 3 NQE),
  //                       neighbour X[NQE] Y0 Y1 Z0 Z1 (4 + NQE) -- per-point upwind terms
  //  T-form (trigonometric b, P4): diagonal S0 S1 S2 M TQ[NQV][2] W[6] U[3][NQE], the
  //                       per-point transport phi_q (x) d_a phi_q as 2 NQV rank-1 operands
  // (P1 on this path, through the warp-specialised kernel, measured 1.90 ms on config 4 vs the
  // CUDA-core P1 kernel's 1.16 ms: 9-entry blocks pad to 16 columns and store 8 bytes at a time)
  static constexpr bool kMma = (NL == 6 && BK == 0) || (NL == 10 && (BK == 0 || BK == 1)) ||
                               (NL == 15 && BK == 2);
  static constexpr bool kTForm = BK == 2;
  static constexpr bool kUForm = BK == 1 || BK == 2;            // per-point upwind terms
  static constexpr int kTerms = kTForm ? 4 + 2 * NQV + 6 + 3 * NQE : (kUForm ? 16 + 3 * NQE : 15);
  static constexpr int kOffT = kUForm ? 4 + NQE : 5;            // neighbour terms
  static constexpr int kWRow = kTForm ? 4 + 2 * NQV : (kUForm ? 10 : 6);  // first W row
  static constexpr int kURow = kWRow + 6;                       // first U row (U-/T-form)
  static constexpr int kKS = (kTerms + 3) / 4, kNT = (N2 + 7) / 8;
  static constexpr int kKO = (kOffT + 3) / 4;                   // neighbour k-steps
  static constexpr int kDRows = 4 * kKS;                         // diagonal rows (zero padded)
  static constexpr int kCT = 36;                                 // coefficient table stride [k][lane]
  static constexpr int kStage = kMma ? 0 : (kRowMode ? ((32 * 4 * N2 + 2 + 1) & ~1) : 32 * SS);
  // MMA path: the stash is the A operand itself, [term][lane] rows of stride kCT: diagonal
  // terms 0..15 (15 = zero pad), then the neighbour terms [l][X Y0 Y1 Z0 Z1]
  static constexpr int kStash = kMma ? (kDRows + 3 * kOffT) * kCT : 3 * NF * 32;
  static constexpr int kMeta = (3 * 32 + (kMma ? 48 : 0)) / 2; // 3 ints per lane (+ MMA row map)
  static constexpr int kTrig = BK == 2 && !kMma ? 2 * NQV * 32 : 0;  // pointwise transport weights
  static constexpr int kRhs = (32 * NL + 1) & ~1;               // packed RHS slice of the warp
  static constexpr int kWarp = kStage + kStash + kMeta + kTrig + kRhs;
  static constexpr int kTr = (3 * NQE * 3 * NL + 1) & ~1;      // trace table (per CTA)
  static constexpr int kFragTile = kKS * kNT * 32;               // one B operand, fragment order
  // neighbour operands per (l, lf): K = 4 kKO (kOffT terms), fragment order [ks][nt][lane]
  static constexpr int kOffTile = kKO * kNT * 32;
  static constexpr int kBt = kMma ? kFragTile + 9 * kOffTile : 0;
};

// Offset (doubles) of diagonal term k in the tensor parameter block (MMA path, P2, const b).
template <typename L>
__device__ __forceinline__ int diag_term_offset(int k) {
  constexpr int N2 = L::N2;
  if (k < 3) return L::S + k * N2;
  if (k == 3) return L::M;
  if (k < 6) return L::T + (k - 4) * N2;
  if (k < 12) return L::W + (k - 6) * N2;
  return L::P + (k - 12) * N2;
}

__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned long long output_policy(bool evict_first) {
  unsigned long long pol;
  if (evict_first) {
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(pol));
  } else {
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(pol));
  }
  return pol;
}
__device__ __forceinline__ void store_pair(double* g, double a, double b, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n"
               :: "l"(g), "d"(a), "d"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void store_one(double* g, double a, unsigned long long pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.f64 [%0], %1, %2;\n"
               :: "l"(g), "d"(a), "l"(pol) : "memory");
}
// Entries n0, n0 + 1 of an element block at `blk`: one 16-byte store when N2 is even (block
// starts 16-byte aligned), two 8-byte stores otherwise; entries past N2 are padding.
template <int N2>
__device__ __forceinline__ void store_entries(double* blk, int n0, double a, double b,
                                              unsigned long long pol) {
  if constexpr (N2 % 2 == 0) {
    if (N2 % 8 == 0 || n0 < N2) store_pair(blk + n0, a, b, pol);
  } else {
    if (n0 < N2) store_one(blk + n0, a, pol);
    if (n0 + 1 < N2) store_one(blk + n0 + 1, b, pol);
  }
}

// One warp-wide block product on the FP64 tensor cores: D[32 elements x N2] = C . B, where
// a_at(m, ks) returns C[8 m + g][4 ks + t] for this lane (g, t) and B is a fragment-ordered
// table in global memory ([ks][nt][lane], lane (g, t) holding B[4 ks + t][8 nt + g]).  Lane
// (g, t) ends up with D[8 m + g][8 nt + 2 t .. +1] and stores that 16-byte pair straight to
// val[base(8 m + g) + 8 nt + 2 t]: each store instruction writes 64 contiguous bytes of eight
// element blocks.  base < 0: the element has no such block.
template <int KS, int NT, int N2, class AF>
__device__ __forceinline__ void mma_block_store(AF a_at, const double* __restrict__ frag,
                                                long long base, double* val, int lane,
                                                unsigned long long pol) {
  const int g = lane >> 2, t = lane & 3;
  // small K: the A fragments stay in registers across the n-tiles; large K (P4): re-read
  constexpr bool kKeepA = KS <= 7;
  double af[4][kKeepA ? KS : 1];
  if constexpr (kKeepA) {
#pragma unroll
    for (int m = 0; m < 4; ++m) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) af[m][ks] = a_at(m, ks);
    }
  }
  long long bm[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) bm[m] = __shfl_sync(0xffffffffu, base, 8 * m + g);
  if constexpr (kKeepA) {
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      double bf[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) bf[ks] = __ldg(frag + (ks * NT + nt) * 32 + lane);
      const int n0 = 8 * nt + 2 * t;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) dmma_8x8x4(d0, d1, af[m][ks], bf[ks]);
        if (bm[m] >= 0) store_entries<N2>(val + bm[m], n0, d0, d1, pol);
      }
    }
  } else {
    // large K (P4): the B fragments of the next n-tile are loaded (from L2) while this one's
    // products run, and each product splits its K chain over two accumulators
    double bq[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bq[ks] = __ldg(frag + ks * NT * 32 + lane);
#pragma unroll 1
    for (int nt = 0; nt < NT; ++nt) {
      double bf[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) bf[ks] = bq[ks];
      if (nt + 1 < NT) {
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) bq[ks] = __ldg(frag + (ks * NT + nt + 1) * 32 + lane);
      }
      const int n0 = 8 * nt + 2 * t;
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ks += 2) {
          dmma_8x8x4(d0, d1, a_at(m, ks), bf[ks]);
          if (ks + 1 < KS) dmma_8x8x4(e0, e1, a_at(m, ks + 1), bf[ks + 1]);
        }
        if (bm[m] >= 0) store_entries<N2>(val + bm[m], n0, d0 + e0, d1 + e1, pol);
      }
    }
  }
}

// Split form of a fused batch (P-form, sets differing only in kappa): D_s = C . Bc + kappa_s
// (C . Bq), where Bc is the kappa = 0 table and Bq holds the kappa coefficient of the W rows
// (Q^T, k-steps 1 and 2: rows 4..11, rows 4 and 5 zero).  Each product runs once; every set
// costs two DFMAs and a store per fragment.
template <int KS, int NT, int N2, class AF>
__device__ __forceinline__ void mma_block_store_split(AF a_at, const double* __restrict__ frag,
                                                      long long base, const MethodOut* bt,
                                                      int n_sets, int lane,
                                                      unsigned long long pol) {
  static_assert(KS >= 3 && KS <= 7, "split form: W rows in k-steps 1 and 2, A in registers");
  const int g = lane >> 2, t = lane & 3;
  double af[4][KS];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) af[m][ks] = a_at(m, ks);
  }
  long long bm[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) bm[m] = __shfl_sync(0xffffffffu, base, 8 * m + g);
  const double* fq = frag + KS * NT * 32;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    double bf[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) bf[ks] = __ldg(frag + (ks * NT + nt) * 32 + lane);
    const double bq0 = __ldg(fq + nt * 32 + lane), bq1 = __ldg(fq + (NT + nt) * 32 + lane);
    const int n0 = 8 * nt + 2 * t;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      double d0 = 0.0, d1 = 0.0, q0 = 0.0, q1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) dmma_8x8x4(d0, d1, af[m][ks], bf[ks]);
      dmma_8x8x4(q0, q1, af[m][1], bq0);
      dmma_8x8x4(q0, q1, af[m][2], bq1);
      if (bm[m] >= 0) {
#pragma unroll
        for (int s = 0; s < kMaxBatch; ++s) {
          if (s < n_sets) {
            const double k = bt[s].kappa;
            store_entries<N2>(bt[s].val + bm[m], n0, fma(k, q0, d0), fma(k, q1, d1), pol);
          }
        }
      }
    }
  }
}

// Velocity of the kernel's specialised kind (BK = dgb_vector_field kind): no dead branches,
// so a constant-velocity kernel carries no call into the trigonometric form.
template <int BK>
__device__ __forceinline__ void velocity_k(const dgb_vector_field& b, double x, double y,
                                           double& bx, double& by) {
  if constexpr (BK == DGB_VEC_CONSTANT) {
    bx = b.p[0];
    by = b.p[1];
  } else if constexpr (BK == DGB_VEC_AFFINE) {
    bx = FADD(FADD(b.p[0], FMUL(b.p[2], x)), FMUL(b.p[3], y));
    by = FADD(FADD(b.p[1], FMUL(b.p[4], x)), FMUL(b.p[5], y));
  } else {
    velocity_trig(b.p[0], b.p[1], x, y, bx, by);
  }
}

// Stash field indices (per edge l, per lane): see the diagonal / neighbour passes.
enum { F_W0 = 0, F_W1, F_P, F_Y0, F_Y1, F_Z0, F_Z1, F_X, F_U = 7 };

// FUSE (tensor-core kernels, n_batch > 1 sets with equal penalties): one CTA assembles its
// rows for EVERY set.  The A operand (the per-element stash) does not depend on kappa --
// kappa lives in the B fragments (W = kappa Q^T - Q, kappa Z) and in one RHS term, kept apart
// (F = F0 + kappa Fk) -- so the gathers, geometry, source and edge terms run once and only the
// products and stores repeat per set.
template <int NL, int NQV, int NQE, int BK, int THREADS, int MINB, bool FUSE = false>
__global__ void __launch_bounds__(THREADS, MINB) assemble_kernel(
    const __grid_constant__ Params2<NL, NQV, NQE, BK == 2, full_tensors(NL, BK)> P) {
  constexpr bool TRIG = BK == 2;
  constexpr int N2 = NL * NL;
  using L = Lay<NL, NQV, NQE, TRIG, full_tensors(NL, BK)>;
  using SM = Smem<NL, NQV, NQE, BK>;
  constexpr int SS = SM::SS, NF = SM::NF;
  extern __shared__ double smem[];
  double* tr = smem;  // [3][NQE][3][NL]: phi, w d0 phi, w d1 phi of each local edge's points
  if (P.tr_src) {     // built once per plan (dgb_plan_create), the same values as below
    for (int i = threadIdx.x; i < 3 * NQE * 3 * NL; i += blockDim.x) tr[i] = __ldg(P.tr_src + i);
  } else
  for (int i = threadIdx.x; i < 3 * NQE * 3 * NL; i += blockDim.x) {
    const int j = i % NL, c = (i / NL) % 3, p = (i / (3 * NL)) % NQE, l = i / (3 * NL * NQE);
    // gradients rotated to the neighbour's (opposite, b, a) vertex order (p1_tables)
    const double g0 = P.t.x[L::EDW + ((l * NQE + p) * 2) * NL + j];
    const double g1 = P.t.x[L::EDW + ((l * NQE + p) * 2 + 1) * NL + j];
    tr[i] = c == 0 ? P.t.x[L::EPHI + (l * NQE + p) * NL + j]
            : l == 0 ? (c == 1 ? g0 : g1)
            : l == 1 ? (c == 1 ? g1 - g0 : -g0)
                     : (c == 1 ? -g1 : g0 - g1);
  }
  __syncthreads();
  if (DGB_ABLATE(16)) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // this CTA's parameter set (grid.y) and its outputs
  // split form (fused P-form batch): shared products, kappa applied per set at the store
  constexpr bool kSplit = FUSE && SM::kMma && !SM::kUForm;
  const int mset = FUSE ? 0 : blockIdx.y;
  const int n_sets = FUSE ? P.n_batch : 1;  // sets this CTA writes: bt[mset .. mset + n_sets)
  const double kappa = P.bt[mset].kappa, sigma_i = P.bt[mset].sigma_i, sigma_b = P.bt[mset].sigma_b;
  int32_t* const o_row_ptr = P.bt[mset].row_ptr;
  int32_t* const o_col = P.bt[mset].col;
  double* const o_val = P.bt[mset].val;
  double* const o_rhs = P.bt[mset].rhs;
  const double* const o_bfrag = P.bt[mset].bfrag;
  double* stw = smem + SM::kTr + warp * SM::kWarp;  // staging [32][SS]
  double* st = stw + lane * SS;  // (even N2) this lane's block
  double* sk = stw + SM::kStage;                     // stash [NF][3][32]
  int* mk = reinterpret_cast<int*>(sk + SM::kStash); // meta [3][32]: kind | lf << 2 | slot << 4
  double* sq = sk + SM::kStash + SM::kMeta;          // TRIG: [NQV][2][32]
  double* srhs = sq + SM::kTrig;                     // [32][NL] packed RHS
  auto K = [&](int f, int l) -> double& {
    if constexpr (SM::kMma) {
      constexpr int CT = SM::kCT, OB = SM::kDRows;  // OB: first neighbour row
      int row;
      if constexpr (SM::kUForm) {
        // F_U + p: diagonal point term U[l][p]; F_U + NQE + p: neighbour point term X[p]
        row = f == F_W0 ? SM::kWRow + 2 * l : f == F_W1 ? SM::kWRow + 1 + 2 * l
            : (f >= F_U && f < F_U + NQE) ? SM::kURow + l * NQE + (f - F_U)
            : f >= F_U + NQE ? OB + SM::kOffT * l + (f - F_U - NQE)
            : OB + SM::kOffT * l + NQE + (f - F_Y0);
      } else {
        row = f == F_W0 ? 6 + 2 * l : f == F_W1 ? 7 + 2 * l : f == F_P ? 12 + l
            : OB + 5 * l + (f == F_X ? 0 : f - F_Y0 + 1);
      }
      return sk[row * CT + lane];
    } else {
      return sk[(f * 3 + l) * 32 + lane];
    }
  };

  if constexpr (FUSE) {
#pragma unroll
    for (int i = 0; i < NL; ++i) srhs[lane * NL + i] = 0.0;  // Fk: this lane's row
  }
  const int e = P.row_begin + blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = e < P.row_end;
  const int ee = active ? e : P.row_end - 1;  // inactive lanes mirror a valid element
  const dgb_vector_field& bf = P.prob.advection;

  // ---- phase A0: own geometry; every gather issued up front (two dependent levels) -------------
  int v[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) v[k] = __ldg(P.elements + 3 * ee + k);
  int4 anb = make_int4(0, 0, 0, 0), aop = make_int4(0, 0, 0, 0);
  if (P.adj_nb) {  // bound adjacency record: two coalesced 16-byte loads per element
    anb = __ldg(P.adj_nb + (ee - P.row_begin));
    aop = __ldg(P.adj_op + (ee - P.row_begin));
  }
  double2 pv[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) pv[k] = __ldg(reinterpret_cast<const double2*>(P.nodes) + v[k]);
  double2 po[3];  // bound path: the neighbours' vertices opposite the shared edges
  if (P.adj_nb) {
    po[0] = __ldg(reinterpret_cast<const double2*>(P.nodes) + max(aop.x, 0));
    po[1] = __ldg(reinterpret_cast<const double2*>(P.nodes) + max(aop.y, 0));
    po[2] = __ldg(reinterpret_cast<const double2*>(P.nodes) + max(aop.z, 0));
  }
  const double B00 = FSUB(pv[1].x, pv[0].x), B01 = FSUB(pv[2].x, pv[0].x);
  const double B10 = FSUB(pv[1].y, pv[0].y), B11 = FSUB(pv[2].y, pv[0].y);
  const double det = FSUB(FMUL(B00, B11), FMUL(B01, B10));
  const double rdet = rcp_nr(det);
  const double G00 = B11 * rdet, G01 = -B10 * rdet;
  const double G10 = -B01 * rdet, G11 = B00 * rdet;
  const double eps = scalar_element(P.prob.diffusion, ee);
  if (DGB_ABLATE(32)) {
    if (active) o_rhs[ee - P.row_begin] = det;
    return;
  }

  // ---- phase A1: RHS volume term and pointwise transport weights (few live registers) -------
  double F[NL];
#pragma unroll
  for (int i = 0; i < NL; ++i) F[i] = 0.0;
  {
    source_points<NQV, TRIG>(
        P.prob.source, ee, DGB_ABLATE(2),
        [&](int q, double& px, double& py) {
          // volume points only evaluate coefficients (no term selection): fused
          px = fma(B01, P.t.x[L::VY + q], fma(B00, P.t.x[L::VX + q], pv[0].x));
          py = fma(B11, P.t.x[L::VY + q], fma(B10, P.t.x[L::VX + q], pv[0].y));
        },
        [&](int q, double f, double px, double py) {
          const double dw = det * P.t.x[L::VW + q];
          const double c = dw * f;
#pragma unroll
          for (int i = 0; i < NL; ++i) F[i] = fma(c, P.t.x[L::PHI + q * NL + i], F[i]);
          if constexpr (TRIG) {
            // volume points only scale the transport terms (no upwind decision is taken here):
            // b = (cos(w0 y), sin(w1 x)) through cospi / sinpi of (w / pi) y -- a cheaper
            // reduction than cos / sin of the rounded product w y, equal to ~1e-15 absolute.
            // Edge points keep the reference's expressions (they decide the upwind side).
            constexpr double kInvPi = 0.318309886183790671538;
            const double bx = cospi((bf.p[0] * kInvPi) * py), by = sinpi((bf.p[1] * kInvPi) * px);
            if constexpr (SM::kMma) {  // T-form: the transport coefficients are A-operand rows
              sk[(4 + 2 * q) * SM::kCT + lane] = dw * (G00 * bx + G10 * by);
              sk[(4 + 2 * q + 1) * SM::kCT + lane] = dw * (G01 * bx + G11 * by);
            } else {
              sq[(2 * q) * 32 + lane] = dw * (G00 * bx + G10 * by);
              sq[(2 * q + 1) * 32 + lane] = dw * (G01 * bx + G11 * by);
            }
          }
        });
  }

  // ---- phase A2: per local edge -> stashed coefficient record, boundary RHS --------------------
  int fcol[3] = {-1, -1, -1};  // neighbour across local edge l (interior edges only)
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    const int a = v[(l + 1) % 3], b = v[(l + 2) % 3];
    const int o = a < b ? 0 : 1;  // make_side orientation (assembly.cpp:125-126)
    const double2 A = o == 0 ? pv[(l + 1) % 3] : pv[(l + 2) % 3];
    const double2 Bn = o == 0 ? pv[(l + 2) % 3] : pv[(l + 1) % 3];
    const double dx = FSUB(Bn.x, A.x), dy = FSUB(Bn.y, A.y);
    const double h = hypot_fast(dx, dy);  // edge_geometry (mesh.cpp:232-257)
    const double rh = rcp_nr(h);
    const double tx = dx * rh, ty = dy * rh;
    const double nx = o == 0 ? ty : -ty, ny = o == 0 ? -tx : tx;  // outward normal of e
    const double ge0 = G00 * nx + G10 * ny, ge1 = G01 * nx + G11 * ny;
    int edge = -1, kind, lf = 0, f = -1, vf[3];
    if (P.adj_nb) {
      kind = (anb.w >> (4 * l)) & 3;
      lf = (anb.w >> (4 * l + 2)) & 3;
      f = l == 0 ? anb.x : (l == 1 ? anb.y : anb.z);
      const int opp = l == 0 ? aop.x : (l == 1 ? aop.y : aop.z);
      // f traverses the shared edge the other way: vf[lf] = opp, vf[lf+1] = b, vf[lf+2] = a
#pragma unroll
      for (int k = 0; k < 3; ++k) vf[k] = k == lf ? opp : (k == (lf + 1) % 3 ? b : a);
    } else {
      edge = __ldg(P.element_edges + 3 * ee + l);
      kind = __ldg(P.edge_kind + edge);
      if (kind == DGB_EDGE_INTERIOR) {
        const int2 lr = __ldg(reinterpret_cast<const int2*>(P.edge_elements) + edge);
        f = lr.x == ee ? lr.y : lr.x;
#pragma unroll
        for (int k = 0; k < 3; ++k) vf[k] = __ldg(P.elements + 3 * f + k);
#pragma unroll
        for (int k = 0; k < 3; ++k) if (vf[k] != a && vf[k] != b) lf = k;
      }
    }
    double w0 = 0.0, w1 = 0.0, cp = 0.0, y0 = 0.0, y1 = 0.0, z0 = 0.0, z1 = 0.0, cx = 0.0;
    if (kind == DGB_EDGE_INTERIOR) {
      Geo gf;
      if (P.adj_nb) {  // coordinates in registers: q[lf] = opposite, q[lf+1] = b, q[lf+2] = a
        const double2 qo = l == 0 ? po[0] : (l == 1 ? po[1] : po[2]);
        const double2 qa = l == 0 ? pv[1] : (l == 1 ? pv[2] : pv[0]);
        const double2 qb = l == 0 ? pv[2] : (l == 1 ? pv[0] : pv[1]);
        gf = element_geo_coords(qo, qb, qa);  // rotated order (opposite, b, a): see tr
      } else {
        const int vr[3] = {lf == 0 ? vf[0] : (lf == 1 ? vf[1] : vf[2]), b, a};
        gf = element_geo_fast(P.nodes, vr);
      }
      double eps_e = eps;
      if (P.prob.diffusion.kind == DGB_FIELD_PER_ELEMENT) {
        const double ef = __ldg(P.prob.diffusion.per_element + f);
        eps_e = ee < f ? 0.5 * (eps + ef) : 0.5 * (ef + eps);
      }
      fcol[l] = f;
      const double base = 0.5 * h * eps_e;  // avg * h * eps
      w0 = base * ge0;
      w1 = base * ge1;
      y0 = -base * (gf.G00 * nx + gf.G10 * ny);
      y1 = -base * (gf.G01 * nx + gf.G11 * ny);
      // tensor-core path: kappa is folded into the Z rows of the B operand
      const double kz = SM::kMma ? 1.0 : kappa;
      z0 = -kz * base * ge0;
      z1 = -kz * base * ge1;
      const double sh = sigma_i * rh;
      if constexpr (BK == 0) {
        // constant b: every point has the same flux, so the point weights factor out
        const double fl = FADD(FMUL(bf.p[0], nx), FMUL(bf.p[1], ny));
        const double up = fl < 0.0 ? FMUL(h, fl) : 0.0;
        cp = sh * (h * eps_e) - up;  // diag: penalty + (-h b.n) on inflow
        cx = up - sh * (h * eps_e);  // off : -penalty + (h b.n) on inflow
      } else {
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          // physical point q = o ? n-1-p : p; the mirrored rule gives t_q = 1 - t_p and
          // w_q = w_p bitwise (quadrature.cpp:185-192), so the loads stay warp-uniform
          const double w = FMUL(P.t.x[L::EW + p], h);
          const double tq = o == 0 ? P.t.x[L::ET + p] : 1.0 - P.t.x[L::ET + p];
          const double px = FADD(A.x, FMUL(tq, dx));
          const double py = FADD(A.y, FMUL(tq, dy));
          double bx, by;
          velocity_k<BK>(bf, px, py, bx, by);
          const double fl = FADD(FMUL(bx, nx), FMUL(by, ny));
          const double up = fl < 0.0 ? FMUL(w, fl) : 0.0;
          const double pen = FMUL(sh, FMUL(w, eps_e));
          K(F_U + p, l) = pen - up;
          K(F_U + NQE + p, l) = up - pen;
        }
      }
    } else {
      // boundary edge: diffusion (Dirichlet), inflow upwind, and the boundary RHS terms
      double fls[NQE], gb[NQE];
      bool inflow = false;
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double tq = o == 0 ? P.t.x[L::ET + p] : 1.0 - P.t.x[L::ET + p];
        const double px = FADD(A.x, FMUL(tq, dx));
        const double py = FADD(A.y, FMUL(tq, dy));
        double bx, by;
        velocity_k<BK>(bf, px, py, bx, by);
        fls[p] = FADD(FMUL(bx, nx), FMUL(by, ny));
        if (fls[p] < -1e-12 * fmax(1.0, hypot_dd(bx, by))) inflow = true;  // assembly.cpp:324-401
        gb[p] = scalar_point(kind == DGB_EDGE_NEUMANN ? P.prob.neumann : P.prob.dirichlet, px, py);
      }
      double cG[NQE], cH[NQE];
      if (kind == DGB_EDGE_NEUMANN) {
        if (edge < 0) edge = __ldg(P.element_edges + 3 * ee + l);
        if (inflow && !P.drop_neumann && active) atomicMax(P.err_edge, (P.epoch << 32) | (0xFFFFFFFFull - static_cast<unsigned>(edge)));
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          cG[p] = FMUL(FMUL(P.t.x[L::EW + p], h), gb[p]);  // neumann_rhs (assembly.cpp:427-442)
          cH[p] = 0.0;
          if constexpr (BK != 0) K(F_U + p, l) = 0.0;
        }
      } else {
        const double base = h * eps;  // avg = 1
        w0 = base * ge0;
        w1 = base * ge1;
        const double sh = sigma_b * rh;
        if constexpr (BK == 0) {
          cp = sh * (h * eps) - ((inflow && fls[0] < 0.0) ? FMUL(h, fls[0]) : 0.0);
        }
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double w = FMUL(P.t.x[L::EW + p], h);
          const double win = (inflow && fls[p] < 0.0) ? -FMUL(w, fls[p]) : 0.0;
          const double wgd = w * gb[p];
          cG[p] = wgd * (sh * eps) + win * gb[p];  // emit_dirichlet_rhs + inflow data term
          cH[p] = FUSE ? wgd * eps : wgd * (kappa * eps);  // FUSE: into Fk, kappa per set
          if constexpr (BK != 0) K(F_U + p, l) = FMUL(sh, FMUL(w, eps)) + win;
        }
      }
#pragma unroll
      for (int p = 0; p < NQE; ++p) {
        const double h0 = cH[p] * ge0, h1 = cH[p] * ge1;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
          if constexpr (FUSE) {
            F[i] = fma(cG[p], P.t.x[L::EPHI + (l * NQE + p) * NL + i], F[i]);
            srhs[lane * NL + i] =
                fma(h0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i],
                    fma(h1, P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], srhs[lane * NL + i]));
          } else {
            F[i] = fma(cG[p], P.t.x[L::EPHI + (l * NQE + p) * NL + i],
                       fma(h0, P.t.x[L::EDPHI + ((l * NQE + p) * 2) * NL + i],
                           fma(h1, P.t.x[L::EDPHI + ((l * NQE + p) * 2 + 1) * NL + i], F[i])));
          }
        }
      }
    }
    K(F_W0, l) = w0;
    K(F_W1, l) = w1;
    if constexpr (!SM::kUForm) K(F_P, l) = cp;  // U-form: per-point terms instead
    K(F_Y0, l) = y0;
    K(F_Y1, l) = y1;
    K(F_Z0, l) = z0;
    K(F_Z1, l) = z1;
    if constexpr (BK == 0) K(F_X, l) = cx;
    mk[l * 32 + lane] = kind | (lf << 2);
  }
  // sorted block columns -> slots (CSR order of the reference's stiffness()): each block's
  // slot is its rank among the row's columns (all distinct), computed without indexed arrays
  int slot_of[4], nb = 1;
  {
    const int cx[4] = {ee, fcol[0], fcol[1], fcol[2]};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int r = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) r += (j != i && cx[j] >= 0 && cx[j] < cx[i]) ? 1 : 0;
      slot_of[i] = r;
    }
#pragma unroll
    for (int l = 0; l < 3; ++l) nb += fcol[l] >= 0 ? 1 : 0;
  }
  int rp;
  if (P.row_ptr_src) {  // pattern computed once per mesh: copy this element's entry
    rp = __ldg(P.row_ptr_src + (ee - P.row_begin));
    if (active) {
      const int rp1 = __ldg(P.row_ptr_src + (ee - P.row_begin + 1));
#pragma unroll 1
      for (int s = 0; s < n_sets; ++s) {
        int32_t* rpo = P.bt[mset + s].row_ptr;
        rpo[ee - P.row_begin + 1] = rp1;
        if (ee == P.row_begin) rpo[0] = 0;
      }
    }
  } else {
    rp = o_row_ptr[ee - P.row_begin];
  }
  const int diag_slot = slot_of[0];
#pragma unroll 1
  for (int s = 0; s < n_sets; ++s) {
    int32_t* co = FUSE ? P.bt[mset + s].col : o_col;
    if (active) co[rp + diag_slot] = ee;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
      if (active && fcol[l] >= 0) co[rp + slot_of[1 + l]] = fcol[l];
    }
  }
#pragma unroll
  for (int l = 0; l < 3; ++l) {
    if (fcol[l] >= 0) mk[l * 32 + lane] |= slot_of[1 + l] << 4;
  }

  // odd N2: this lane's row inside the warp's contiguous staged row range
  int rp_first = 0, rp_last = 0;
  double* srow = stw;
  if constexpr (SM::kRowMode) {
    rp_first = __shfl_sync(0xffffffffu, rp, 0);
    rp_last = __reduce_max_sync(0xffffffffu, active ? rp + nb : 0);
    srow = stw + (rp_first & 1);  // same 16-byte phase as val + rp_first * N2
  }
  auto block_at = [&](int slot) -> double* {
    if constexpr (SM::kRowMode) return srow + (rp - rp_first + slot) * N2;
    else return st;
  };

  const unsigned long long pol = output_policy(P.evict_first);
  // ---- RHS: the warp's contiguous slice, packed in shared memory and written in one go ------
  if constexpr (FUSE) {
    // per set: F0 + kappa_s Fk staged, then coalesced 16-byte stores (slices 16-B aligned)
    double fk[NL];
#pragma unroll
    for (int i = 0; i < NL; ++i) fk[i] = srhs[lane * NL + i];
    const int e_first = blockIdx.x * blockDim.x + warp * 32;  // relative to row_begin
    const int n_here = min(32, P.row_end - P.row_begin - e_first);
    const int n = n_here * NL;
#pragma unroll 1
    for (int s = 0; s < n_sets; ++s) {
      const double ks = P.bt[mset + s].kappa;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < NL; ++i) srhs[lane * NL + i] = fma(ks, fk[i], F[i]);
      __syncwarp();
      double* dst = P.bt[mset + s].rhs + static_cast<long long>(e_first) * NL;
      for (int idx = 2 * lane; idx + 1 < n; idx += 64) {
        store_pair(dst + idx, srhs[idx], srhs[idx + 1], pol);
      }
      if (n > 0 && (n & 1) && lane == 0) store_one(dst + n - 1, srhs[n - 1], pol);
    }
  } else {
#pragma unroll
    for (int i = 0; i < NL; ++i) srhs[lane * NL + i] = F[i];
    fence_smem_to_async();  // every writer: its shared-memory stores -> the async (TMA) proxy
    __syncwarp();
    const int e_first = blockIdx.x * blockDim.x + warp * 32;  // relative to row_begin
    const int n_here = min(32, P.row_end - P.row_begin - e_first);
    double* dst = o_rhs + static_cast<long long>(e_first) * NL;
    const int bulk = (n_here * NL) & ~1;  // 16-byte multiple (warp slices start 16-B aligned)
    if (lane == 0 && bulk > 0) bulk_store(dst, srhs, bulk * sizeof(double), P.evict_first);
    for (int idx = bulk + lane; idx < n_here * NL; idx += 32) dst[idx] = srhs[idx];
  }

  // ---- diagonal block ----------------------------------------------------------------------
  {
    const double alpha = scalar_element(P.prob.linear_reaction, ee);
    const double de = det * eps;
    const double cD0 = de * (G00 * G00 + G10 * G10);
    const double cD1 = de * (G00 * G01 + G10 * G11);
    const double cD2 = de * (G01 * G01 + G11 * G11);
    const double cR = det * alpha;
    double cC0 = 0.0, cC1 = 0.0, cA[4] = {0.0, 0.0, 0.0, 0.0};
    if constexpr (BK == 0) {
      cC0 = det * (G00 * bf.p[0] + G10 * bf.p[1]);
      cC1 = det * (G01 * bf.p[0] + G11 * bf.p[1]);
    } else if constexpr (BK == 1) {
      // b(o + B xhat) = (c + A o) + (A B) xhat  (affine velocity, config 3)
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
    if constexpr (SM::kMma) {
      // D[32 elements x 36 entries] = C[32 x 16 coefficients] . T[16 x 36] on the FP64 tensor
      // cores, stored from the fragments
      const double cv[10] = {cD0, cD1, cD2, cR, cC0, cC1, cA[0], cA[1], cA[2], cA[3]};
#pragma unroll
      for (int k = 0; k < (SM::kTForm ? 4 : (SM::kUForm ? 10 : 6)); ++k) sk[k * SM::kCT + lane] = cv[k];
#pragma unroll
      for (int k = SM::kTerms; k < SM::kDRows; ++k) sk[k * SM::kCT + lane] = 0.0;  // K padding
      __syncwarp();
      const int g = lane >> 2, t = lane & 3;
      if constexpr (kSplit) {
        if (!(DGB_ABLATE(8))) {
          mma_block_store_split<SM::kKS, SM::kNT, N2>(
              [&](int m, int ks) { return sk[(4 * ks + t) * SM::kCT + 8 * m + g]; }, o_bfrag,
              (active && !(DGB_ABLATE(1))) ? static_cast<long long>(rp + diag_slot) * N2 : -1LL,
              P.bt + mset, n_sets, lane, pol);
        }
      } else if (!(DGB_ABLATE(8))) {
#pragma unroll 1
        for (int s = 0; s < n_sets; ++s) {
          mma_block_store<SM::kKS, SM::kNT, N2>(
              [&](int m, int ks) { return sk[(4 * ks + t) * SM::kCT + 8 * m + g]; },
              P.bt[mset + s].bfrag,
              (active && !(DGB_ABLATE(1))) ? static_cast<long long>(rp + diag_slot) * N2 : -1LL,
              P.bt[mset + s].val, lane, pol);
        }
      }
    } else {
    constexpr int RC = NL <= 6 ? NL : (NL <= 10 ? 2 : 1);  // rows per register chunk
    double* blk = block_at(diag_slot);
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
          if constexpr (!TRIG) {
            x = fma(cC0, P.t.x[L::T + k], x);
            x = fma(cC1, P.t.x[L::T + N2 + k], x);
          }
          if constexpr (BK == 1 && L::kHasTA) {
#pragma unroll
            for (int a = 0; a < 4; ++a) x = fma(cA[a], P.t.x[L::TA + a * N2 + k], x);
          }
          acc[r][j] = x;
        }
      }
#pragma unroll(NL <= 6 ? 3 : 1)
      for (int l = 0; l < 3; ++l) {
        const double w0 = K(F_W0, l), w1 = K(F_W1, l);
#pragma unroll
        for (int r = 0; r < RC; ++r) {
#pragma unroll
          for (int j = 0; j < NL; ++j) {
            const int k = (i0 + r) * NL + j;
            acc[r][j] = fma(w0, P.t.x[L::W + 2 * l * N2 + k],
                            fma(w1, P.t.x[L::W + (2 * l + 1) * N2 + k], acc[r][j]));
          }
        }
        if constexpr (BK == 0 && L::kHasP) {
          const double cp = K(F_P, l);
#pragma unroll
          for (int r = 0; r < RC; ++r) {
#pragma unroll
            for (int j = 0; j < NL; ++j) {
              acc[r][j] = fma(cp, P.t.x[L::P + l * N2 + (i0 + r) * NL + j], acc[r][j]);
            }
          }
        } else {
          // per-point face weights: acc += sum_p cU_p phi^l_p phi^l_p^T
#pragma unroll
          for (int p = 0; p < NQE; ++p) {
            double cu;
            if constexpr (BK == 0) {
              cu = K(F_P, l) * P.t.x[L::EW + p];
            } else {
              cu = K(F_U + p, l);
            }
#pragma unroll
            for (int r = 0; r < RC; ++r) {
              const double u = cu * P.t.x[L::EPHI + (l * NQE + p) * NL + i0 + r];
#pragma unroll
              for (int j = 0; j < NL; ++j) {
                acc[r][j] = fma(u, P.t.x[L::EPHI + (l * NQE + p) * NL + j], acc[r][j]);
              }
            }
          }
        }
      }
      if constexpr (TRIG) {
#pragma unroll 1
        for (int q = 0; q < NQV; ++q) {
          const double b0 = sq[(2 * q) * 32 + lane], b1 = sq[(2 * q + 1) * 32 + lane];
#pragma unroll
          for (int r = 0; r < RC; ++r) {
            const double f0 = b0 * P.t.x[L::PHI + q * NL + i0 + r];
            const double f1 = b1 * P.t.x[L::PHI + q * NL + i0 + r];
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
        for (int j = 0; j < NL; ++j) if (active) blk[(i0 + r) * NL + j] = acc[r][j];
      }
    }
    }  // register path
    if constexpr (!SM::kRowMode && !SM::kMma) {
      write_block<N2>(stw, st, active ? static_cast<long long>(rp + diag_slot) * N2 : -1LL,
                      o_val, lane, P.evict_first);
    }
  }

  // ---- neighbour blocks: K_ef = sum_p phi^l_p (x) b1_p + a2_p (x) phi^lf_(n-1-p) ---------------
#pragma unroll(NL <= 6 ? 3 : 1)  // small blocks: compile-time l (LDCU.128 immediates)
  for (int l = 0; l < 3; ++l) {
    const int meta = mk[l * 32 + lane];
    const bool has = (meta & 3) == DGB_EDGE_INTERIOR;
    if (!__any_sync(0xffffffffu, has)) continue;
    const int lf = (meta >> 2) & 3, slot = meta >> 4;
    if constexpr (SM::kMma) {
      if (DGB_ABLATE(4)) continue;
      // neighbour terms X, Y0, Y1, Z0, Z1 of edge l.  The B operand depends on the
      // neighbour's local edge lf, so the warp's elements are regrouped into 8-row m-tiles of
      // equal lf (rows are independent in D = C . B): ceil(n_lf / 8) tiles per lf value, each
      // an m8 x n(N2) x k8 product (5 terms) against that lf's operand.
      const bool store = active && has;
      const int g = lane >> 2, t = lane & 3;
      const unsigned lt = (1u << lane) - 1u;
      const unsigned m0 = __ballot_sync(0xffffffffu, has && lf == 0);
      const unsigned m1 = __ballot_sync(0xffffffffu, has && lf == 1);
      const unsigned m2 = __ballot_sync(0xffffffffu, has && lf == 2);
      const int t1 = (__popc(m0) + 7) >> 3, t2 = t1 + ((__popc(m1) + 7) >> 3);
      const int ntiles = t2 + ((__popc(m2) + 7) >> 3);
      int* pmap = mk + 96;  // sorted row -> lane (-1: padding row)
      pmap[lane] = -1;
      if (lane < 16) pmap[32 + lane] = -1;
      __syncwarp();
      if (has) {
        const unsigned mv = lf == 0 ? m0 : (lf == 1 ? m1 : m2);
        const int tv = lf == 0 ? 0 : (lf == 1 ? t1 : t2);
        pmap[8 * tv + __popc(mv & lt)] = lane;
      }
      __syncwarp();
      const long long my_base = store ? static_cast<long long>(rp + slot) * N2 : -1LL;
      const double* so = sk + (SM::kDRows + SM::kOffT * l) * SM::kCT;
      // class-major: each lf's operand is loaded once into registers, and the next tile's
      // row operands are fetched while the current tile's products run
      constexpr int KO = SM::kKO;
      auto tile_rows = [&](int r, double (&aa)[KO], long long& bm) {
        const int src = pmap[8 * r + g];
        const int sl = src < 0 ? 0 : src;
#pragma unroll
        for (int ks = 0; ks < KO; ++ks) {
          aa[ks] = (src < 0 || 4 * ks + t >= SM::kOffT) ? 0.0 : so[(4 * ks + t) * SM::kCT + sl];
        }
        bm = __shfl_sync(0xffffffffu, my_base, sl);
        if (src < 0) bm = -1;
      };
      if constexpr (kSplit) {
        // fused P-form batch: D_s = [X Y0 Y1] . Bxy + kappa_s [Z0 Z1] . Bz, one k-step each
        static_assert(KO == 2, "split form: neighbour terms X Y0 Y1 | Z0 Z1");
        auto rows_split = [&](int r, double (&aa)[2], long long& bm) {
          const int src = pmap[8 * r + g];
          const int sl = src < 0 ? 0 : src;
          aa[0] = (src < 0 || t >= 3) ? 0.0 : so[t * SM::kCT + sl];
          aa[1] = (src < 0 || t >= 2) ? 0.0 : so[(3 + t) * SM::kCT + sl];
          bm = __shfl_sync(0xffffffffu, my_base, sl);
          if (src < 0) bm = -1;
        };
        double aa[2];
        long long bm;
        if (ntiles > 0) rows_split(0, aa, bm);
#pragma unroll
        for (int v = 0; v < 3; ++v) {
          const int tb = v == 0 ? 0 : (v == 1 ? t1 : t2), te = v == 0 ? t1 : (v == 1 ? t2 : ntiles);
          if (tb == te) continue;
          const double* fr = o_bfrag + SM::kFragTile + 2 * SM::kNT * 32 +
                             (l * 3 + v) * SM::kOffTile + lane;
          double bv[2][SM::kNT];
#pragma unroll
          for (int nt = 0; nt < SM::kNT; ++nt) {
            bv[0][nt] = __ldg(fr + nt * 32);
            bv[1][nt] = __ldg(fr + (SM::kNT + nt) * 32);
          }
#pragma unroll 1
          for (int r = tb; r < te; ++r) {
            const double c0 = aa[0], c1 = aa[1];
            const long long cb = bm;
            if (r + 1 < ntiles) rows_split(r + 1, aa, bm);
#pragma unroll
            for (int nt = 0; nt < SM::kNT; ++nt) {
              double d0 = 0.0, d1 = 0.0, z0 = 0.0, z1 = 0.0;
              dmma_8x8x4(d0, d1, c0, bv[0][nt]);
              dmma_8x8x4(z0, z1, c1, bv[1][nt]);
              const int n0 = 8 * nt + 2 * t;
              if (cb >= 0 && !(DGB_ABLATE(1))) {
#pragma unroll
                for (int s = 0; s < kMaxBatch; ++s) {
                  if (s < n_sets) {
                    const double k = P.bt[mset + s].kappa;
                    store_entries<N2>(P.bt[mset + s].val + cb, n0, fma(k, z0, d0), fma(k, z1, d1), pol);
                  }
                }
              }
            }
          }
        }
      } else {
#pragma unroll 1
      for (int s = 0; s < n_sets; ++s) {
      const double* const o_bfrag = P.bt[mset + s].bfrag;
      double* const o_val = P.bt[mset + s].val;
      double aa[KO];
      long long bm;
      if (ntiles > 0) tile_rows(0, aa, bm);
      // small operands (P2, P3): the class's B fragments live in registers across its tiles
      constexpr bool kPreload = KO * SM::kNT <= 26;
#pragma unroll
      for (int v = 0; v < 3; ++v) {
        const int tb = v == 0 ? 0 : (v == 1 ? t1 : t2), te = v == 0 ? t1 : (v == 1 ? t2 : ntiles);
        if (tb == te) continue;
        const double* fr = o_bfrag + SM::kFragTile + (l * 3 + v) * SM::kOffTile + lane;
        double bv[kPreload ? KO : 1][kPreload ? SM::kNT : 1];
        if constexpr (kPreload) {
#pragma unroll
          for (int nt = 0; nt < SM::kNT; ++nt) {
#pragma unroll
            for (int ks = 0; ks < KO; ++ks) bv[ks][nt] = __ldg(fr + (ks * SM::kNT + nt) * 32);
          }
        }
        if constexpr (kPreload) {
#pragma unroll 1
          for (int r = tb; r < te; ++r) {
            double ca[KO];
#pragma unroll
            for (int ks = 0; ks < KO; ++ks) ca[ks] = aa[ks];
            const long long cb = bm;
            if (r + 1 < ntiles) tile_rows(r + 1, aa, bm);
#pragma unroll
            for (int nt = 0; nt < SM::kNT; ++nt) {
              double d0 = 0.0, d1 = 0.0;
#pragma unroll
              for (int ks = 0; ks < KO; ++ks) dmma_8x8x4(d0, d1, ca[ks], bv[ks][nt]);
              const int n0 = 8 * nt + 2 * t;
              if (cb >= 0 && !(DGB_ABLATE(1))) store_entries<N2>(o_val + cb, n0, d0, d1, pol);
            }
          }
        } else {
          // large operands (P4): n-tile outer -- each B fragment (streamed from L2 a few
          // n-tiles ahead) serves every tile of the class; the tiles' rows stay in registers
          constexpr int MT = 4;  // tiles per class: at most 32 rows
          double at[MT][KO];
          long long bt_[MT];
#pragma unroll
          for (int u = 0; u < MT; ++u) {
            bt_[u] = -1;
#pragma unroll
            for (int ks = 0; ks < KO; ++ks) at[u][ks] = 0.0;
            if (tb + u < te) tile_rows(tb + u, at[u], bt_[u]);
          }
          // a ring of PF register buffers, the n-tile loop fully unrolled so the ring needs no
          // moves: the L2 latency of a fragment is covered by PF n-tiles of products
          constexpr int PF = 8;
          double bq[PF][KO];
#pragma unroll
          for (int u = 0; u < PF; ++u) {
#pragma unroll
            for (int ks = 0; ks < KO; ++ks) bq[u][ks] = __ldg(fr + (ks * SM::kNT + u) * 32);
          }
#pragma unroll
          for (int nt = 0; nt < SM::kNT; ++nt) {
            double bk[KO];
#pragma unroll
            for (int ks = 0; ks < KO; ++ks) bk[ks] = bq[nt % PF][ks];
            if (nt + PF < SM::kNT) {
#pragma unroll
              for (int ks = 0; ks < KO; ++ks) bq[nt % PF][ks] = __ldg(fr + (ks * SM::kNT + nt + PF) * 32);
            }
            const int n0 = 8 * nt + 2 * t;
#pragma unroll
            for (int u = 0; u < MT; ++u) {
              if (tb + u < te) {
                double d0 = 0.0, d1 = 0.0;
#pragma unroll
                for (int ks = 0; ks < KO; ++ks) dmma_8x8x4(d0, d1, at[u][ks], bk[ks]);
                if (bt_[u] >= 0 && !(DGB_ABLATE(1))) store_entries<N2>(o_val + bt_[u], n0, d0, d1, pol);
              }
            }
          }
        }
      }
      }  // sets
      }  // !kSplit
      __syncwarp();  // the row map is rebuilt for the next l
      continue;
    }
    const double cY0 = K(F_Y0, l), cY1 = K(F_Y1, l), cZ0 = K(F_Z0, l), cZ1 = K(F_Z1, l);
    double cV[NQE];
#pragma unroll
    for (int p = 0; p < NQE; ++p) {
      if constexpr (BK == 0) {
        cV[p] = K(F_X, l) * P.t.x[L::EW + p];
      } else {
        cV[p] = K(F_U + NQE + p, l);
      }
    }
    const double* trm = tr + lf * (NQE * 3 * NL);
    if constexpr (!SM::kRowMode) bulk_wait_read();  // previous block copy has left the staging
    double* blk = block_at(slot);
    const bool store = active && has;
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
          b1[p][c] = fma(cV[p], f, fma(cY0, g0, cY1 * g1));  // g already w-scaled
        }
      }
#pragma unroll
      for (int i = 0; i < NL; ++i) {
        double acc[CJ];
#pragma unroll
        for (int c = 0; c < CJ; ++c) acc[c] = 0.0;
#pragma unroll
        for (int p = 0; p < NQE; ++p) {
          const double a2 = fma(cZ0, P.t.x[L::EDW + ((l * NQE + p) * 2) * NL + i],
                                cZ1 * P.t.x[L::EDW + ((l * NQE + p) * 2 + 1) * NL + i]);
          const double ph = P.t.x[L::EPHI + (l * NQE + p) * NL + i];
#pragma unroll
          for (int c = 0; c < CJ; ++c) acc[c] = fma(ph, b1[p][c], fma(a2, pm[p][c], acc[c]));
        }
#pragma unroll
        for (int c = 0; c < CJ; ++c) if (store) blk[i * NL + j0 + c] = acc[c];
      }
    }
    if constexpr (!SM::kRowMode) {
      write_block<N2>(stw, st, store ? static_cast<long long>(rp + slot) * N2 : -1LL, o_val, lane,
                      P.evict_first);
    }
  }
  if constexpr (SM::kRowMode) {
    // one bulk copy of the warp's whole row range; the unaligned head / tail doubles by hand
    fence_smem_to_async();  // every writer: its staged blocks -> the async (TMA) proxy
    __syncwarp();
    const int n = (rp_last - rp_first) * N2;
    double* dst = o_val + static_cast<long long>(rp_first) * N2;
    const int head = rp_first & 1;
    const int body = (n - head) & ~1;
    if (lane == 0 && body > 0) bulk_store(dst + head, srow + head, body * sizeof(double), P.evict_first);
    // (a warp past the last row has no range: n <= 0, nothing to write)
    if (lane == 1 && head && n > 0) dst[0] = srow[0];
    if (lane == 2 && n > 0 && head + body < n) dst[n - 1] = srow[n - 1];
  } else {
    bulk_wait_all();  // shared memory must outlive the copies
  }
  if (lane == 0) bulk_wait_all();
}

}  // namespace v2
}  // namespace dgb
