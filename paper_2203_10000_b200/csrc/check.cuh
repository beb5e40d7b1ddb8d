// Device-side bounds checks for the checked build (NM_CHECKED; built by
// paper_2203_10000_b200/build.py into lib/checked/ and run under the GPU test
// suite by tests/test_gpu_checked.py). compute-sanitizer is closed on this GPU
// pool (profiles/r02/compute_sanitizer_refusal.log), so every global index the
// main kernels form is checked against its array's bound instead: a failure
// prints the site and traps (the launch fails, the test fails loudly). In the
// product build the checks compile to nothing.
#pragma once
#include <cstdio>

#ifdef NM_CHECKED
#define NM_DCHECK(cond, what)                                                                                 \
  do {                                                                                                        \
    if (!(cond)) {                                                                                            \
      printf("NM_DCHECK failed: %s (%s:%d) block (%d,%d) thread %d\n", what, __FILE__, __LINE__, blockIdx.x,  \
             blockIdx.y, threadIdx.x);                                                                        \
      __trap();                                                                                               \
    }                                                                                                         \
  } while (0)
#else
#define NM_DCHECK(cond, what) \
  do {                        \
  } while (0)
#endif
