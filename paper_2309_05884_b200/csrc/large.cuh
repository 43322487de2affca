// Batched-GEMM path for large symmetry blocks (d > 16).  (stub, filled in next)
#pragma once
#include <cuda_runtime.h>

namespace sqoc {

struct LargeBlock {
  int d = 0;
};

struct LargeArgs {
  const double* u;
  int batch;
  const double2* gen;
  const double2* x0;
  const double2* target;
  double weight;
  double2* tau_out;
  int tau_stride;
  double* grad_out;
};

inline const char* large_last_error() { return "large-block path not built yet"; }
inline int large_init(LargeBlock& lb, int d, int, int, bool, int) { lb.d = d; return 4; }
inline int large_eval(LargeBlock&, const LargeArgs&, cudaStream_t, int*) { return 4; }
inline void large_free(LargeBlock&) {}

}  // namespace sqoc
