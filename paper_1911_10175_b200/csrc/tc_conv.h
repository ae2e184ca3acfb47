// tc_conv.h -- 3xTF32 tcgen05 FWD/BWI (internal).
#pragma once
#include "common.cuh"

namespace spc {
bool tc_conv_supported(bool fwd, const DevShape& sh, int V);
cudaError_t launch_tc_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi);
bool tc_bww_supported(const DevShape& sh, int V);
cudaError_t launch_tc_bww(bool check_input, bool sparse, const DevShape& sh, const float* chk, const float* oth,
                          float* dst, unsigned long long* exec_ctr, cudaStream_t st);
}  // namespace spc
