// Internal host-side helpers shared by the C-ABI translation units: thread-local error
// string, argument checks, launch checks, and small by-value parameter structs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>

#include "../../include/psa.h"

namespace psa {

constexpr int kMaxLevels = 8;
constexpr int kMaxCuts = 16;

struct SimTaus {
  double v[kMaxLevels];
};

struct LevelRule {  // thresholds (mode 0) or quantile rank counts (mode 1)
  double taus[kMaxCuts];
  int32_t counts[kMaxCuts];
  int n_cuts;
  int mode;
};

}  // namespace psa

int psa_fail(int code, const char* fmt, ...);
int psa_check_launch(const char* what);

#define PSA_CHECK_ARG(cond, msg)                           \
  do {                                                     \
    if (!(cond)) return psa_fail(PSA_EINVAL, "%s", (msg)); \
  } while (0)
