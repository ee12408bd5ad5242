// Drop-in check: the reference library calls the B200 path through the INTEGRATION.md
// adapter (include/dgfem/gpu.hpp) and compares it with its own assemble_all + stiffness().
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "dgfem/assembly.hpp"
#include "dgfem/gpu.hpp"
#include "dgfem/mesh.hpp"
#include "dgfem/problems.hpp"
#include "dgfem/reference.hpp"

using namespace dgfem;

int main() {
  Mesh mesh = uniform_refine(uniform_refine(uniform_refine(unit_square_mesh())));
  int failures = 0;
  for (int k = 1; k <= 4; ++k) {
    ReferenceElement ref(k);
    for (DgMethod m : {DgMethod::SIPG, DgMethod::NIPG, DgMethod::IIPG}) {
      const DgParameters prm = set_parameters(m, k);
      // smooth-sine (problems.cpp:136-164) as a device descriptor
      dgb_problem p{};
      p.diffusion = {DGB_FIELD_CONSTANT, 0, 0, 0, 1.0};
      p.advection = {DGB_VEC_CONSTANT, 0, {1.0, 2.0}};
      p.linear_reaction = {DGB_FIELD_CONSTANT, 0, 0, 0, 1.0};
      p.source = {DGB_FIELD_FUNCTION, DGB_FN_SIN_SIN, DGB_MODE_SOURCE, 0, 0.0, {1.0},
                  {1.0, 1.0, 1.0, 2.0}};
      p.dirichlet = {DGB_FIELD_FUNCTION, DGB_FN_SIN_SIN, DGB_MODE_VALUE, 0, 0.0, {1.0}};
      p.neumann = {DGB_FIELD_FUNCTION, DGB_FN_SIN_SIN, DGB_MODE_FLUX_X, 0, 0.0, {1.0},
                   {0.0, 1.0}};
      const gpu::BsrSystem g = gpu::assemble_all(mesh, ref, p, prm);
      const DgSystem cpu = assemble_all(mesh, ref, registry_get("smooth-sine"), prm);
      const CsrMatrix K = cpu.stiffness();
      // expand BSR -> CSR and compare with a per-row scale
      const int nl = g.block_dim;
      double kerr = 0.0, ferr = 0.0;
      bool pattern = static_cast<std::size_t>(K.nnz()) == g.val.size();
      for (int e = 0; e < g.n_block_rows && pattern; ++e) {
        for (int i = 0; i < nl; ++i) {
          const int r = e * nl + i;
          double scale = 0.0;
          for (int t = K.row_offsets[r]; t < K.row_offsets[r + 1]; ++t)
            scale = std::max(scale, std::abs(K.values[t]));
          int t = K.row_offsets[r];
          for (int b = g.row_ptr[e]; b < g.row_ptr[e + 1]; ++b) {
            for (int j = 0; j < nl; ++j, ++t) {
              if (K.col_indices[t] != g.col[b] * nl + j) pattern = false;
              kerr = std::max(kerr, std::abs(K.values[t] - g.val[(b * nl + i) * nl + j]) / scale);
            }
          }
        }
        double fs = 0.0;
        for (int i = 0; i < nl; ++i) fs = std::max(fs, std::abs(cpu.F[e * nl + i]));
        for (int i = 0; i < nl; ++i)
          ferr = std::max(ferr, std::abs(cpu.F[e * nl + i] - g.F[e * nl + i]) / fs);
      }
      const bool ok = pattern && kerr <= 1e-12 && ferr <= 1e-12;
      failures += !ok;
      std::printf("[%s] k=%d %s: pattern %s, K err %.2e, F err %.2e\n", ok ? "PASS" : "FAIL", k,
                  to_string(m), pattern ? "bit-exact" : "DIFFERS", kerr, ferr);
    }
  }
  return failures;
}
