// pw_bww.h -- 1x1 BWW (check = input) as a register-blocked GEMM (internal).
#pragma once
#include "common.cuh"

namespace spc {
bool pw_bww_supported(bool check_input, const DevShape& sh, int V);
// `finite` -> device int written by launch_finite_all over dY (1 = all finite).
cudaError_t launch_pw_bww(bool sparse, const DevShape& sh, const float* dchw, const float* dy, float* dst,
                          unsigned long long* exec_ctr, const int* finite, cudaStream_t st);
// tma_pw_bww.cu: the finite-dY case (runs when *finite == 1)
bool tma_pw_bww_supported(const DevShape& sh);
cudaError_t launch_tma_pw_bww(bool sparse, const DevShape& sh, const float* dchw, const float* dy, float* dst,
                              unsigned long long* exec_ctr, const int* finite, cudaStream_t st);
void launch_finite_all(const float* t, size_t n, int* flag, cudaStream_t st);
void launch_set_flag(int* flag, cudaStream_t st);  // *flag = 1
void launch_finite_also(const float* t, size_t n, int* flag, cudaStream_t st);
}  // namespace spc
