// capi_common.cpp -- status names, last-error storage, parameters (C-ABI).
#include <cstring>
#include <string>

#include "common.hpp"

namespace {
thread_local std::string g_message;
thread_local long long g_detail = -1;
}  // namespace

namespace dgb {

int record_error(int status, const std::string& message, long long detail) {
  g_message = message;
  g_detail = detail;
  return status;
}

void clear_error() {
  g_message.clear();
  g_detail = -1;
}

}  // namespace dgb

extern "C" {

// Names of dgfem::ErrorCode (errors.cpp:5-27), offset by one.
const char* dgb_status_name(int status) {
  switch (status) {
    case DGB_OK: return "Ok";
    case DGB_STATUS_INVALID_TOPOLOGY: return "InvalidTopology";
    case DGB_STATUS_INVALID_BOUNDARY_SPEC: return "InvalidBoundarySpec";
    case DGB_STATUS_NON_MANIFOLD: return "NonManifold";
    case DGB_STATUS_DEGENERATE_ELEMENT: return "DegenerateElement";
    case DGB_STATUS_UNSUPPORTED_DEGREE: return "UnsupportedDegree";
    case DGB_STATUS_INVALID_INDEX: return "InvalidIndex";
    case DGB_STATUS_DIMENSION_MISMATCH: return "DimensionMismatch";
    case DGB_STATUS_SINGULAR_MATRIX: return "SingularMatrix";
    case DGB_STATUS_SOLVE_ACCURACY: return "SolveAccuracy";
    case DGB_STATUS_INFLOW_ON_NEUMANN: return "InflowOnNeumann";
    case DGB_STATUS_NON_POSITIVE_DIFFUSION: return "NonPositiveDiffusion";
    case DGB_STATUS_INVALID_REACTION: return "InvalidReaction";
    case DGB_STATUS_NO_EXACT_SOLUTION: return "NoExactSolution";
    case DGB_STATUS_UNKNOWN_PROBLEM: return "UnknownProblem";
    case DGB_STATUS_UNKNOWN_METHOD: return "UnknownMethod";
    case DGB_STATUS_IO_FAILURE: return "IoFailure";
    case DGB_STATUS_INVALID_ARGUMENT: return "InvalidArgument";
    case DGB_STATUS_CUDA: return "CudaError";
    default: return "Unknown";
  }
}

const char* dgb_last_error_message(void) { return g_message.c_str(); }
long long dgb_last_error_detail(void) { return g_detail; }
const char* dgb_version(void) { return "dgfem_b200 0.1 (sm_100a)"; }

// dgfem::set_parameters (assembly.cpp:483-506).
int dgb_set_parameters(int32_t method, int32_t degree, dgb_params* out) {
  return dgb::guarded([&] {
    if (degree < 1) {
      throw dgb::Error(DGB_STATUS_INVALID_ARGUMENT, "polynomial degree must be at least 1",
                       degree);
    }
    dgb_params p;
    std::memset(&p, 0, sizeof p);
    p.method = method;
    p.degree = degree;
    switch (method) {
      case DGB_SIPG:
        p.kappa = -1.0;
        p.sigma_interior = 3.0 * degree * (degree + 1);
        break;
      case DGB_NIPG:
        p.kappa = 1.0;
        p.sigma_interior = 1.0;
        break;
      case DGB_IIPG:
        p.kappa = 0.0;
        p.sigma_interior = 3.0 * degree * (degree + 1);
        break;
      default:
        throw dgb::Error(DGB_STATUS_UNKNOWN_METHOD, "unknown method code", method);
    }
    p.sigma_boundary = 2.0 * p.sigma_interior;
    p.neumann_inflow = DGB_INFLOW_ERROR;
    *out = p;
  });
}

int64_t dgb_bsr_nnzb(int32_t n_elements, int32_t n_interior_edges) {
  return static_cast<int64_t>(n_elements) + 2 * static_cast<int64_t>(n_interior_edges);
}

}  // extern "C"
