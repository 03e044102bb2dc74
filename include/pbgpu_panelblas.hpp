// C++ shim with the reference's own signatures (panelblas, /root/reference/proj/include/
// panelblas/blas.hpp and level3.hpp), implemented over the pbgpu C ABI (pbgpu.h).
//
// A caller of the reference switches by replacing `#include "panelblas/blas.hpp"` with
// `#include "pbgpu_panelblas.hpp"` and `panelblas::` with `pbgpu::`; argument lists,
// validation order, info conventions, BlasCallError reports and the abort_on_error
// (xerbla) mode are the same.  Pointers may be host or device memory (pbgpu.h).
// Fields with no GPU meaning (PackStats, GemmVariant) are not carried.
#pragma once

#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "pbgpu.h"

namespace pbgpu {

enum class TransOp { NoTrans, Trans };  // mat_view.hpp:18

// mat_view.hpp:60-68
class ArgError : public std::invalid_argument {
 public:
  ArgError(int index, const std::string& message) : std::invalid_argument(message), index_(index) {}
  int index() const noexcept { return index_; }

 private:
  int index_;
};

// mat_view.hpp:72-76
struct BlasCallError {
  std::string routine;
  int index = 0;
  std::string message;
};

// mat_view.hpp:82-90
struct Status {
  int info = 0;
  std::string message{};
  bool ok() const noexcept { return info == 0; }
};

// blas.hpp:21-25 (the engine tuning of the CPU library has no GPU counterpart)
struct EngineConfig {};
struct BlasConfig {
  EngineConfig engine{};
  bool abort_on_error = false;
};

// blas.hpp:32-40
struct BlasResult {
  int info = 0;
  std::optional<BlasCallError> error;
  long long flops = 0;
  bool ok() const { return info == 0; }
};

// level3.hpp:318-323
struct NdResult {
  Status status;
  long long flops = 0;
  bool ok() const { return status.ok(); }
};

// panel_mat.hpp:51-81 (byte-compatible with pb_dmat)
struct PanelRef {
  double* data = nullptr;
  int ps = 4;
  int m = 0, n = 0;
  int pm = 0, cn = 0;
  static PanelRef over(double* buf, int m, int n, int ps = 4) {
    return {buf, ps, m, n, (m + ps - 1) / ps * ps, (n + ps - 1) / ps * ps};
  }
};
struct ConstPanelRef {
  const double* data = nullptr;
  int ps = 4;
  int m = 0, n = 0;
  int pm = 0, cn = 0;
  ConstPanelRef() = default;
  ConstPanelRef(const PanelRef& r) : data(r.data), ps(r.ps), m(r.m), n(r.n), pm(r.pm), cn(r.cn) {}
  ConstPanelRef(const double* d, int ps_, int m_, int n_, int pm_, int cn_)
      : data(d), ps(ps_), m(m_), n(n_), pm(pm_), cn(cn_) {}
};

namespace detail {
inline pb_dmat dm(const ConstPanelRef& r) {
  return pb_dmat{const_cast<double*>(r.data), r.ps, r.m, r.n, r.pm, r.cn};
}
inline pb_dmat dm(const PanelRef& r) { return pb_dmat{r.data, r.ps, r.m, r.n, r.pm, r.cn}; }
inline BlasResult blas(const BlasConfig& cfg, const pb_result& r) {
  if (r.info == PB_INFO_CUDA_ERROR || r.info == PB_INFO_NO_DEVICE)
    throw std::runtime_error(std::string("pbgpu: ") + (r.message ? r.message : "CUDA failure"));
  BlasResult out;
  out.info = r.info;
  out.flops = r.flops;
  if (r.error_index) {
    out.error = BlasCallError{r.routine ? r.routine : "", r.error_index, r.message ? r.message : ""};
    if (cfg.abort_on_error) throw ArgError(r.error_index, out.error->routine + ": " + out.error->message);
  }
  return out;
}
inline NdResult nd(const pb_result& r) {
  if (r.info == PB_INFO_CUDA_ERROR || r.info == PB_INFO_NO_DEVICE)
    throw std::runtime_error(std::string("pbgpu: ") + (r.message ? r.message : "CUDA failure"));
  NdResult out;
  out.status.info = r.info;
  if (r.message) out.status.message = r.message;
  out.flops = r.flops;
  return out;
}
inline char tc(TransOp t) { return t == TransOp::NoTrans ? 'N' : 'T'; }
}  // namespace detail

// ---- netlib-shaped adapters (blas.hpp:73-215) ----
inline BlasResult dgemm(const BlasConfig& cfg, char transa, char transb, int m, int n, int k,
                        double alpha, const double* a, int lda, const double* b, int ldb, double beta,
                        double* c, int ldc) {
  pb_result r{};
  pb_dgemm(transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, &r);
  return detail::blas(cfg, r);
}
inline BlasResult dsyrk(const BlasConfig& cfg, char uplo, char trans, int n, int k, double alpha,
                        const double* a, int lda, double beta, double* c, int ldc) {
  pb_result r{};
  pb_dsyrk(uplo, trans, n, k, alpha, a, lda, beta, c, ldc, &r);
  return detail::blas(cfg, r);
}
inline BlasResult dtrsm(const BlasConfig& cfg, char side, char uplo, char transa, char diag, int m,
                        int n, double alpha, const double* a, int lda, double* b, int ldb) {
  pb_result r{};
  pb_dtrsm(side, uplo, transa, diag, m, n, alpha, a, lda, b, ldb, &r);
  return detail::blas(cfg, r);
}
inline BlasResult dpotrf(const BlasConfig& cfg, char uplo, int n, double* a, int lda) {
  pb_result r{};
  pb_dpotrf(uplo, n, a, lda, &r);
  return detail::blas(cfg, r);
}
inline BlasResult dgetrf(const BlasConfig& cfg, int m, int n, double* a, int lda, std::vector<int>& ipiv) {
  ipiv.assign(static_cast<size_t>(m > 0 && n > 0 ? (m < n ? m : n) : 0), 0);
  pb_result r{};
  pb_dgetrf(m, n, a, lda, ipiv.data(), &r);
  return detail::blas(cfg, r);
}

// ---- native panel-major routines (level3.hpp:360-575) ----
inline NdResult gemm_nd(const EngineConfig&, TransOp transa, TransOp transb, int m, int n, int k,
                        double alpha, ConstPanelRef a, ConstPanelRef b, double beta, ConstPanelRef c,
                        PanelRef d) {
  pb_result r{};
  pb_gemm_nd(detail::tc(transa), detail::tc(transb), m, n, k, alpha, detail::dm(a), detail::dm(b), beta,
             detail::dm(c), detail::dm(d), &r);
  return detail::nd(r);
}
inline NdResult syrk_nd(const EngineConfig&, int n, int k, double alpha, ConstPanelRef a, double beta,
                        ConstPanelRef c, PanelRef d) {
  pb_result r{};
  pb_syrk_nd(n, k, alpha, detail::dm(a), beta, detail::dm(c), detail::dm(d), &r);
  return detail::nd(r);
}
inline NdResult trsm_rltn_nd(const EngineConfig&, int m, int n, double alpha, ConstPanelRef a,
                             ConstPanelRef b, PanelRef d) {
  pb_result r{};
  pb_trsm_rltn_nd(m, n, alpha, detail::dm(a), detail::dm(b), detail::dm(d), &r);
  return detail::nd(r);
}
inline NdResult syrk_potrf_nd(const EngineConfig&, int n, int k, ConstPanelRef a, ConstPanelRef b,
                              ConstPanelRef c, PanelRef d) {
  pb_result r{};
  pb_syrk_potrf_nd(n, k, detail::dm(a), detail::dm(b), detail::dm(c), detail::dm(d), &r);
  return detail::nd(r);
}

}  // namespace pbgpu
