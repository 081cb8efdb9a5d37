// abi.hpp — shared plumbing of the C ABI translation units (engine.cu,
// model.cu): the context object, the error state behind mfadd_last_error*,
// and the exception -> status-code mapping (the reference's exception types,
// include/mfadd_b200.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/mfadd_b200.h"
#include "dev.cuh"
#include "layout.hpp"

#define MFB_API extern "C" __attribute__((visibility("default")))

struct mfadd_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::int64_t launches = 0;
  mfb::DevStatus* d_status = nullptr;
  double* h_pinned = nullptr;  // 16 doubles of pinned host scratch
};

namespace mfb_abi {

extern thread_local std::string g_err;
extern thread_local int g_err_dim;
extern thread_local std::int64_t g_err_span;

struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& w) : std::runtime_error(w), code(c) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw ApiError(MFADD_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return MFADD_OK;
  } catch (const ApiError& e) {
    g_err = e.what();
    return e.code;
  } catch (const mfb::SingularFit& e) {
    g_err = e.what();
    g_err_dim = e.dim;
    g_err_span = e.span;
    return MFADD_ESINGULAR;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return MFADD_EINVAL;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return MFADD_ERANGE;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return MFADD_ELOGIC;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return MFADD_ENOMEM;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return MFADD_ERUNTIME;
  } catch (...) {
    g_err = "unknown error";
    return MFADD_ERUNTIME;
  }
}

// Make the context's device current for the call.
struct ContextScope {
  int prev = -1;
  explicit ContextScope(const mfadd_context* c) {
    cudaGetDevice(&prev);
    if (prev != c->device) cuda_check(cudaSetDevice(c->device), "cudaSetDevice");
  }
  ~ContextScope() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

}  // namespace mfb_abi
