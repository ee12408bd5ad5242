// assemble_ws_t.cuh -- warp-specialised tensor-core kernel for the T-form (P4 with a
// trigonometric velocity: config 5), bound mesh.  Included by dg_assembly.cu after
// assemble_ws.cuh.
//
// The monolithic kernel (assemble_v2.cuh) runs each warp's 32-element chunk as the per-element
// pass (gathers, geometry, the trigonometric velocity at 19 volume and 15 edge points, the A
// rows of every block product) followed by the DMMA products and the fragment stores of the
// 4 x 225-entry blocks; at 240 registers and 66 KB of shared memory per two-warp CTA only 6 warps
// fit an SM, and the two halves of a chunk add up (tuning-build ablations: 0.33 ms of per-element
// pass and 1.26 ms of products and stores, profiles/NOTES.md).  Here one persistent CTA per SM
// holds NP producer warps and NC consumer warps around a ring of NS = NP + NC chunk slots:
//
//   producer: v2_chunk<.., kRoleProduce> -- the per-element pass into the slot (A rows, edge
//             metadata) plus the chunk's row_ptr, block columns and RHS, then rp / diagonal
//             slot / active for the consumer;
//   consumer: v2_consume -- the diagonal product and the neighbour products (mma_neighbours)
//             from the slot, stored from the fragments.
//
// Slots are handed over with mbarriers (full / empty per slot), as in the P2 kernel
// (assemble_ws.cuh).  The arithmetic is the monolithic kernel's, term for term.
#pragma once

namespace dgb {
namespace v2 {

template <int NL, int NQV, int NQE, int BK, int NPROD, int NCONS>
struct SmemWsT {
  using SM = Smem<NL, NQV, NQE, BK>;
  static constexpr int NP = NPROD, NC = NCONS, NS = NPROD + NCONS;
  static constexpr int kThreads = 32 * NS;
  // a slot is the monolithic kernel's per-warp region (stage | stash | meta | trig | rhs) plus
  // `xfer` (rp, diagonal slot, active: 96 ints)
  static constexpr int kSlot = SM::kWarp + 48;
  static constexpr int kBars = 2 * NS;
  static constexpr size_t kBytes = sizeof(double) * (size_t(kBars) + SM::kTr + size_t(NS) * kSlot);
};

// The consumer half of a chunk: the diagonal block D = C . B and the neighbour blocks, from a
// slot a producer filled.
template <int NL, int NQV, int NQE, int BK>
__device__ __forceinline__ void v2_consume(const Params2<NL, NQV, NQE, BK == 2, full_tensors(NL, BK)>& P,
                                           double* slot, int lane, int mset) {
  using SM = Smem<NL, NQV, NQE, BK>;
  constexpr int N2 = NL * NL;
  const double* sk = slot + SM::kStage;
  int* mk = reinterpret_cast<int*>(slot + SM::kStage + SM::kStash);
  const int* xfer = reinterpret_cast<const int*>(slot + SM::kWarp);
  const int rp = xfer[lane], diag_slot = xfer[32 + lane];
  const bool active = xfer[64 + lane] != 0;
  const unsigned long long pol = output_policy(P.evict_first);
  const int g = lane >> 2, t = lane & 3;
  if (!(DGB_ABLATE(8))) {
    mma_block_store<SM::kKS, SM::kNT, N2>(
        [&](int m, int ks) { return sk[(4 * ks + t) * SM::kCT + 8 * m + g]; }, P.bt[mset].bfrag,
        (active && !(DGB_ABLATE(1))) ? static_cast<long long>(rp + diag_slot) * N2 : -1LL,
        P.bt[mset].val, lane, pol);
  }
  mma_neighbours<NL, NQV, NQE, BK, false>(P, sk, mk, rp, active, lane, mset, 1, pol);
}

template <int NL, int NQV, int NQE, int BK, int NPROD, int NCONS>
__global__ void __launch_bounds__(SmemWsT<NL, NQV, NQE, BK, NPROD, NCONS>::kThreads, 1)
    assemble_ws_t_kernel(const __grid_constant__ Params2<NL, NQV, NQE, BK == 2, full_tensors(NL, BK)> P) {
  using W = SmemWsT<NL, NQV, NQE, BK, NPROD, NCONS>;
  using SM = Smem<NL, NQV, NQE, BK>;
  using L = Lay<NL, NQV, NQE, BK == 2, full_tensors(NL, BK)>;
  constexpr int NP = W::NP, NC = W::NC, NS = W::NS;
  extern __shared__ double smem[];
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem);  // [NS][full, empty]
  double* tr = smem + W::kBars;
  double* slots = tr + SM::kTr;
  if (P.tr_src) {
    for (int i = threadIdx.x; i < 3 * NQE * 3 * NL; i += blockDim.x) tr[i] = __ldg(P.tr_src + i);
  } else {
    for (int i = threadIdx.x; i < 3 * NQE * 3 * NL; i += blockDim.x) {  // as assemble_kernel
      const int j = i % NL, c = (i / NL) % 3, p = (i / (3 * NL)) % NQE, l = i / (3 * NL * NQE);
      const double g0 = P.t.x[L::EDW + ((l * NQE + p) * 2) * NL + j];
      const double g1 = P.t.x[L::EDW + ((l * NQE + p) * 2 + 1) * NL + j];
      tr[i] = c == 0 ? P.t.x[L::EPHI + (l * NQE + p) * NL + j]
              : l == 0 ? (c == 1 ? g0 : g1)
              : l == 1 ? (c == 1 ? g1 - g0 : -g0)
                       : (c == 1 ? -g1 : g0 - g1);
    }
  }
  if (threadIdx.x < W::kBars) mbar_init(bars + threadIdx.x, 32);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mset = blockIdx.y;
  const int n_rows = P.row_end - P.row_begin;
  const int n_chunks = (n_rows + 31) >> 5;
  const int n_local = n_chunks > static_cast<int>(blockIdx.x)
                          ? (n_chunks - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1
                          : 0;
  if (warp < NP) {
    for (int k = warp; k < n_local; k += NP) {
      const int s = k % NS, r = k / NS;
      double* slot = slots + s * W::kSlot;
      if (r > 0) mbar_wait(bars + 2 * s + 1, (r - 1) & 1);  // empty: round r - 1 consumed
      const int c = blockIdx.x + k * gridDim.x;
      v2_chunk<NL, NQV, NQE, BK, false, kRoleProduce>(P, tr, slot, c * 32, lane,
                                                       reinterpret_cast<int*>(slot + SM::kWarp));
      mbar_arrive(bars + 2 * s);
    }
  } else {
    for (int k = warp - NP; k < n_local; k += NC) {
      const int s = k % NS, r = k / NS;
      mbar_wait(bars + 2 * s, r & 1);  // full: round r produced
      v2_consume<NL, NQV, NQE, BK>(P, slots + s * W::kSlot, lane, mset);
      mbar_arrive(bars + 2 * s + 1);
    }
  }
}

}  // namespace v2
}  // namespace dgb
