// Host-side helpers shared by the C-ABI translation units: error capture,
// TMA tensor-map encoding (driver entry point fetched through the runtime, so
// the library does not link libcuda directly), launch helpers.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../../include/samp_b200.h"

namespace samp {

struct SampError : std::runtime_error {
  int code;
  SampError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SAMP_CUDA(call)                                                                       \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      throw ::samp::SampError(SAMP_E_DEVICE, std::string(#call) + ": " + cudaGetErrorString(_e)); \
  } while (0)

#define SAMP_REQUIRE(cond, code, msg)                                \
  do {                                                               \
    if (!(cond)) throw ::samp::SampError((code), std::string(msg));  \
  } while (0)

// thread-local last error for calls that have no engine handle
void set_last_error(const std::string& msg);

CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dtype, int elt_bytes, uint64_t rows,
                         uint64_t cols, uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows,
                         CUtensorMapSwizzle swizzle);

inline CUtensorMap tmap_i8(const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                           uint32_t box_rows, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  return make_tmap_2d(base, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, rows, cols, ld, box_cols, box_rows, sw);
}
inline CUtensorMap tmap_f16(const void* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_cols,
                            uint32_t box_rows, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  return make_tmap_2d(base, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, rows, cols, ld * 2, box_cols, box_rows, sw);
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return SAMP_OK;
  } catch (const SampError& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return SAMP_E_INTERNAL;
  }
}

}  // namespace samp
