// hsdla_b200 internals shared by every translation unit of libhsdla_b200.so:
// error transport (C++ Fail -> C-ABI status code + hsdla_b200_last_error), CUDA /
// NCCL checks, small environment / tracing helpers.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <exception>
#include <new>
#include <string>

#include "../../include/hsdla_b200.h"

namespace hsdla_b200 {

extern thread_local std::string g_last_error;

// Every internal failure: a C-ABI status code (errors.hpp:9-26 taxonomy) and a message.
struct Fail {
  int code;
  std::string msg;
};

#define HS_CUDA(x)                                                                                 \
  do {                                                                                             \
    cudaError_t e_ = (x);                                                                          \
    if (e_ != cudaSuccess) {                                                                       \
      (void)cudaGetLastError();                                                                    \
      throw ::hsdla_b200::Fail{e_ == cudaErrorMemoryAllocation ? HSDLA_B200_SIZING_ERROR            \
                                                               : HSDLA_B200_CUDA_ERROR,            \
                               std::string(#x) + ": " + cudaGetErrorString(e_)};                   \
    }                                                                                              \
  } while (0)

#define HS_NCCL(x)                                                                                   \
  do {                                                                                               \
    ncclResult_t r_ = (x);                                                                           \
    if (r_ != ncclSuccess)                                                                           \
      throw ::hsdla_b200::Fail{HSDLA_B200_NCCL_ERROR, std::string(#x) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

// Run f, mapping any exception onto a status code (the C-ABI never throws).
template <class F>
int guarded(F&& f) {
  try {
    f();
    return HSDLA_B200_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return HSDLA_B200_SIZING_ERROR;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HSDLA_B200_CUDA_ERROR;
  }
}

// Development knobs for the streaming / banding heuristics (tools/stream_tune.py).
inline double env_double(const char* name, double dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atof(v) : dflt;
}

// HSDLA_B200_TRACE=1: host-side timelines of the drop-in (staging, download) on stderr (tuning).
inline bool trace_on() {
  static const bool on = [] {
    const char* v = std::getenv("HSDLA_B200_TRACE");
    return v && *v == '1';
  }();
  return on;
}
inline double host_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// column-major packed lower ('L'): column j starts at j (2n - j + 1) / 2
inline uint64_t packed_col(uint64_t n, uint64_t j) { return j * (2 * n - j + 1) / 2; }

}  // namespace hsdla_b200
