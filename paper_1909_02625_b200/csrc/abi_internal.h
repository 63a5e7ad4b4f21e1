// Internal helpers shared by the C-ABI translation units.
#pragma once
#include <cuda_runtime.h>
#include "../../include/dsp_b200.h"

#define DSP_ABI_VERSION 2

namespace dsp {
int set_error(int code, const char* fmt, ...);
int cuda_check(cudaError_t e, const char* what);
}  // namespace dsp

#define DSP_TRY(expr)              \
  do {                             \
    int _rc = (expr);              \
    if (_rc != DSP_OK) return _rc; \
  } while (0)

#define DSP_CUDA(expr) DSP_TRY(::dsp::cuda_check((expr), #expr))
