// Fused 3-D level pass — placeholder until the plane/column kernels land:
// every level takes the general per-step path.
#include "fused3d.h"

namespace mgrx_b200 {

Fused3DPlan fused3d_plan(const LevelGeom&, int) { return Fused3DPlan{}; }

template <typename T>
cudaError_t fused3d_decompose_level(const T*, T*, T*, void*, const LevelGeom&, const Fused3DPlan&,
                                    const ThomasLevel&, const Exec&) {
  return cudaErrorNotSupported;
}
template <typename T>
cudaError_t fused3d_recompose_level(const T*, T*, T*, void*, const LevelGeom&, const Fused3DPlan&,
                                    const ThomasLevel&, const Exec&) {
  return cudaErrorNotSupported;
}

template cudaError_t fused3d_decompose_level<float>(const float*, float*, float*, void*, const LevelGeom&,
                                                    const Fused3DPlan&, const ThomasLevel&, const Exec&);
template cudaError_t fused3d_decompose_level<double>(const double*, double*, double*, void*, const LevelGeom&,
                                                     const Fused3DPlan&, const ThomasLevel&, const Exec&);
template cudaError_t fused3d_recompose_level<float>(const float*, float*, float*, void*, const LevelGeom&,
                                                    const Fused3DPlan&, const ThomasLevel&, const Exec&);
template cudaError_t fused3d_recompose_level<double>(const double*, double*, double*, void*, const LevelGeom&,
                                                     const Fused3DPlan&, const ThomasLevel&, const Exec&);

}  // namespace mgrx_b200
