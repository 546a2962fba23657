// Library identity and diagnostics entry points of the C ABI.
#include "capi_util.cuh"

extern "C" const char* paqif_version(void) { return "paqif_b200 0.1.0 (sm_100a, fp64)"; }

extern "C" const char* paqif_last_error(void) { return paqif::last_error_buf(); }

extern "C" int paqif_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}
