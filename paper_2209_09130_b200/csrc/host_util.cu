#include "host_util.h"

#include <cudaTypedefs.h>

#include <mutex>

namespace samp {

static thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  SAMP_REQUIRE(fn != nullptr, SAMP_E_DEVICE, "cuTensorMapEncodeTiled unavailable (driver too old?)");
  return fn;
}

CUtensorMap make_tmap_2d(const void* base, CUtensorMapDataType dtype, int elt_bytes, uint64_t rows,
                         uint64_t cols, uint64_t row_stride_bytes, uint32_t box_cols, uint32_t box_rows,
                         CUtensorMapSwizzle swizzle) {
  CUtensorMap map;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  (void)elt_bytes;
  CUresult r = encode_fn()(&map, dtype, 2, const_cast<void*>(base), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  SAMP_REQUIRE(r == CUDA_SUCCESS, SAMP_E_DEVICE,
               "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ") rows=" + std::to_string(rows) +
                   " cols=" + std::to_string(cols) + " stride=" + std::to_string(row_stride_bytes));
  return map;
}

}  // namespace samp

extern "C" const char* samp_last_error(void) { return samp::g_last_error.c_str(); }

extern "C" int samp_device_check(int device) {
  return samp::guarded([&] {
    int n = 0;
    SAMP_CUDA(cudaGetDeviceCount(&n));
    SAMP_REQUIRE(device >= 0 && device < n, SAMP_E_DEVICE, "no CUDA device " + std::to_string(device));
    cudaDeviceProp prop;
    SAMP_CUDA(cudaGetDeviceProperties(&prop, device));
    SAMP_REQUIRE(prop.major == 10 && prop.minor == 0, SAMP_E_DEVICE,
                 std::string("device is ") + prop.name + " (sm_" + std::to_string(prop.major) +
                     std::to_string(prop.minor) + "); this library is built for sm_100a (B200)");
  });
}
