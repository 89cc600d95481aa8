// runtime.hpp — the process-wide B200 context behind the drop-in headers and
// the status -> exception mapping (include/lrgw_cuda.h <-> errors.hpp).
#pragma once

#include <memory>
#include <mutex>
#include <string>

#include "lrgw/errors.hpp"
#include "lrgw_cuda.h"

namespace lrgw {

namespace detail {

struct CtxHolder {
  lrgw_ctx ctx = nullptr;
  int device = 0;
  ~CtxHolder() {
    if (ctx) lrgw_ctx_destroy(ctx);
  }
};

inline CtxHolder& ctx_holder() {
  static CtxHolder h;
  return h;
}

inline std::mutex& ctx_mutex() {
  static std::mutex m;
  return m;
}

// Throw the reference exception type for a status code.
inline void check(int status, lrgw_ctx ctx, const char* what) {
  if (status == LRGW_OK) return;
  std::string msg = std::string(what);
  if (ctx) {
    const char* m = lrgw_ctx_last_error(ctx);
    if (m && *m) msg += std::string(": ") + m;
  }
  switch (status) {
    case LRGW_ERR_INVALID_INPUT:
    case LRGW_ERR_UNSUPPORTED: throw invalid_input(msg);
    case LRGW_ERR_GUARD_EXCEEDED: throw guard_exceeded(msg);
    case LRGW_ERR_SINGULAR: throw singular_matrix(msg, ctx ? lrgw_ctx_last_pivot(ctx) : -1);
    case LRGW_ERR_NUMERIC:
    case LRGW_ERR_CONTOUR_CONVERGENCE: throw numeric_error(msg);
    case LRGW_ERR_IO: throw io_error(msg);
    default: throw device_error(msg);
  }
}

}  // namespace detail

// The context every drop-in call runs on (created on first use).
inline lrgw_ctx context() {
  std::lock_guard<std::mutex> lock(detail::ctx_mutex());
  auto& h = detail::ctx_holder();
  if (!h.ctx) detail::check(lrgw_ctx_create(h.device, &h.ctx), nullptr, "lrgw_ctx_create");
  return h.ctx;
}

// Select the CUDA device for subsequent calls (before the first call).
inline void set_device(int device) {
  std::lock_guard<std::mutex> lock(detail::ctx_mutex());
  auto& h = detail::ctx_holder();
  if (h.ctx && h.device != device) {
    lrgw_ctx_destroy(h.ctx);
    h.ctx = nullptr;
  }
  h.device = device;
}

}  // namespace lrgw
