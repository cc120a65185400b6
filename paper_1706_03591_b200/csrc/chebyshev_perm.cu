// Length-ordered sweep schedule (skewed degree distributions, BASELINE
// configs[3]): the PERM = true instantiations of sweep.cuh, in their own
// translation unit so they compile in parallel with chebyshev.cu.
#include "sweep.cuh"

namespace csc_sweep {

int run_order_perm_f64(const SweepPlan &op, const SweepArgs &A, int mode, double *partials,
                       int64_t &nparts, cudaStream_t st, void *seg_scratch) {
  return run_order<double, true>(op, A, mode, partials, nparts, st, seg_scratch);
}

int run_order_perm_f32(const SweepPlan &op, const SweepArgs &A, int mode, double *partials,
                       int64_t &nparts, cudaStream_t st, void *seg_scratch) {
  return run_order<float, true>(op, A, mode, partials, nparts, st, seg_scratch);
}

}  // namespace csc_sweep
