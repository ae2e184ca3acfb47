// pw_conv.h -- 1x1 FWD/BWI kernels with zero-quad skipping (internal).
#pragma once
#include "common.cuh"

namespace spc {
bool pw_conv_supported(bool fwd, const DevShape& sh, int V);
// `finite` -> device int: 1 = every filter element finite (quad skipping is
// exact), 0 = per-element tests; written by launch_filter_finite.
cudaError_t launch_pw_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, cudaStream_t st, const int* finite,
                           const Epi& epi = Epi{}, const Gate& gate = Gate{});
void launch_filter_finite(const float* filt, size_t n, int* flag, cudaStream_t st);
}  // namespace spc
