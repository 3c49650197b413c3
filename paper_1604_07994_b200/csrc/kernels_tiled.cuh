// Tiled constant-stencil kernels (placeholder: filled in by the next milestone).
#pragma once
#include "stk_common.cuh"

namespace stk {
inline bool tiled_supported(int) { return false; }
inline bool assemble_stencils(int, double, double, int, cudaStream_t) { return true; }
inline bool launch_apply_tiled(int, DGrid, const double*, double*, unsigned, cudaStream_t) { return false; }
inline bool launch_residual_tiled(int, DGrid, const double*, const double*, double*, cudaStream_t) { return false; }
inline bool launch_vel_pass_tiled(int, DGrid, const double*, const double*, const double*, double*, int, int, cudaStream_t) { return false; }
inline bool launch_p_pass1_tiled(int, DGrid, const double*, const double*, double*, cudaStream_t) { return false; }
inline bool launch_p_pass2_tiled(DGrid, const double*, double*, double, cudaStream_t) { return false; }
}  // namespace stk
