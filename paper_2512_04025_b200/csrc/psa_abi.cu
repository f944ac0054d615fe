// Error plumbing of the C ABI (include/psa.h): thread-local last-error string.
// Status codes mirror the reference error taxonomy (pkg/src/pyrattn/errors.py:9-18):
// PSA_EINVAL -> ValidationError, PSA_ENUMERIC -> NumericError, PSA_ECUDA -> RuntimeError.
#include <cstdarg>
#include <cstdio>

#include "psa_internal.h"

static thread_local char g_last_error[512] = "";

int psa_fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
  return code;
}

int psa_check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return psa_fail(PSA_ECUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
  return PSA_OK;
}

extern "C" const char* psa_last_error(void) { return g_last_error; }

extern "C" int psa_version(void) { return 100; }
