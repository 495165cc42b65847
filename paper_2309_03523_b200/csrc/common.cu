#include "common.cuh"

namespace dgc {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  (void)cudaGetLastError();  // a non-sticky error must not surface at the next launch check
  return DGC_ERR_CUDA;
}
}  // namespace dgc

extern "C" int dgc_version(void) { return 1; }
extern "C" const char* dgc_last_error(void) { return dgc::g_last_error.c_str(); }
