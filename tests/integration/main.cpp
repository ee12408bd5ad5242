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

// Compares the adapter's K and F with the reference's own assemble_all + stiffness() (per-row
// scaled K, per-element-block scaled F); returns 1 on failure.
static int compare(const char* what, int k, DgMethod m, const gpu::BsrSystem& g, const DgSystem& cpu) {
  const CsrMatrix K = cpu.stiffness();
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
  std::printf("[%s] %s k=%d %s: pattern %s, K err %.2e, F err %.2e\n", ok ? "PASS" : "FAIL", what, k,
              to_string(m), pattern ? "bit-exact" : "DIFFERS", kerr, ferr);
  return ok ? 0 : 1;
}

int main() {
  Mesh mesh = uniform_refine(uniform_refine(uniform_refine(unit_square_mesh())));
  int failures = 0;
  // the reference's own benchmark problem (bench/assembly_bench.cpp:31-48): paper-boundary-layer
  // with its own callbacks (problems.cpp:78-134, f += u^2) against the device descriptor
  for (int k = 1; k <= 2; ++k) {
    ReferenceElement ref(k);
    const DgParameters prm = set_parameters(DgMethod::SIPG, k);
    const double eps = 1e-6, b1 = 1.0 / std::sqrt(5.0), b2 = 2.0 / std::sqrt(5.0);
    dgb_problem p{};
    p.diffusion = {DGB_FIELD_CONSTANT, 0, 0, 0, eps};
    p.advection = {DGB_VEC_CONSTANT, 0, {b1, b2}};
    p.linear_reaction = {DGB_FIELD_CONSTANT, 0, 0, 0, 1.0};
    p.source = {DGB_FIELD_FUNCTION, DGB_FN_TANH_LAYER, DGB_MODE_SOURCE_SQUARE, 0, 0.0,
                {2.0, -1.0, -0.25, std::sqrt(5.0 * eps)}, {1.0, eps, b1, b2}};
    p.dirichlet = {DGB_FIELD_FUNCTION, DGB_FN_TANH_LAYER, DGB_MODE_VALUE, 0, 0.0,
                   {2.0, -1.0, -0.25, std::sqrt(5.0 * eps)}};
    p.neumann = {DGB_FIELD_CONSTANT, 0, 0, 0, 0.0};
    failures += compare("paper-boundary-layer", k, DgMethod::SIPG, gpu::assemble_all(mesh, ref, p, prm),
                        assemble_all(mesh, ref, registry_get("paper-boundary-layer"), prm));
  }
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
      failures += compare("smooth-sine", k, m, gpu::assemble_all(mesh, ref, p, prm),
                          assemble_all(mesh, ref, registry_get("smooth-sine"), prm));
    }
  }
  return failures;
}
