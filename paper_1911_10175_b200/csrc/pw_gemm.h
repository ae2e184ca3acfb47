// pw_gemm.h -- 1x1 FWD/BWI as a register-blocked GEMM (internal).
#pragma once
#include "common.cuh"

namespace spc {
bool pw_gemm_supported(bool fwd, const DevShape& sh, int V);
// `finite` -> device int (1 = every filter element finite), see launch_finite_all.
cudaError_t launch_pw_gemm(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, const int* finite, cudaStream_t st,
                           const Epi& epi = Epi{});
}  // namespace spc
