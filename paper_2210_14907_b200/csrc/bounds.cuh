// bounds.cuh -- the bounds-checked build (-DNBM_BOUNDS; scripts/r2/bounds_check.sh), the
// substitute for compute-sanitizer on this GPU pool: NBM_CHECK(cond) prints the failing site and
// traps (the launch then fails with cudaErrorLaunchFailure); it compiles to nothing otherwise.
#pragma once
#ifdef NBM_BOUNDS
#include <cstdio>
#endif

namespace nbm {
#ifdef NBM_BOUNDS
static __device__ __noinline__ void nbm_bounds_fail(const char* file, int line) {
  printf("NBM_BOUNDS violation %s:%d block %d thread %d\n", file, line, (int)blockIdx.x, (int)threadIdx.x);
  __trap();
}
#define NBM_CHECK(c)                                       \
  do {                                                     \
    if (!(c)) ::nbm::nbm_bounds_fail(__FILE__, __LINE__);  \
  } while (0)
#else
#define NBM_CHECK(c) \
  do {               \
  } while (0)
#endif
}  // namespace nbm
