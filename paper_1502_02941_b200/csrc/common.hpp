// common.hpp -- error plumbing shared by the host C++ and the CUDA translation units.
//
// Mirrors dgfem::Error (/root/reference/proj/include/dgfem/errors.hpp:35-48): a status code
// (1 + dgfem::ErrorCode), a message and an index `detail`.  C-ABI entry points catch it and
// publish message/detail through dgb_last_error_message()/dgb_last_error_detail().
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/dgfem_b200.h"

namespace dgb {

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& message, long long detail = -1)
      : std::runtime_error(std::string(dgb_status_name(status)) + ": " + message),
        status_(status),
        detail_(detail) {}
  int status() const noexcept { return status_; }
  long long detail() const noexcept { return detail_; }

 private:
  int status_;
  long long detail_;
};

// Records the error for dgb_last_error_*() and returns its status.
int record_error(int status, const std::string& message, long long detail);
// Clears the thread's last error (successful calls).
void clear_error();

#ifdef __CUDACC__
// y = K x over a BSR on `s` (spmv.cu): the one SpMV of the library (dgb_spmv and the solve).
void launch_bsr_spmv(const dgb_bsr* a, const double* x, double* y, cudaStream_t s);
#endif

// Runs fn, translating exceptions into status codes.
template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    clear_error();
    return DGB_OK;
  } catch (const Error& e) {
    return record_error(e.status(), e.what(), e.detail());
  } catch (const std::bad_alloc&) {
    return record_error(DGB_STATUS_INVALID_ARGUMENT, "host allocation failed", -1);
  } catch (const std::exception& e) {
    return record_error(DGB_STATUS_INVALID_ARGUMENT, e.what(), -1);
  }
}

}  // namespace dgb
