// Plane-layout fast path (placeholder until the plane-skewed kernels land).
#include "tilu_plan.cuh"

namespace tilu {
bool plane_supported(const tilu_plan *) { return false; }
int plane_sweep(const tilu_plan *, double *, const double *, int, int, double *, cudaStream_t, int *) { return TILU_EUNSUPPORTED; }
}  // namespace tilu
