// tile_bww.h -- tuned V=16 BWW tile kernels (internal).
#pragma once
#include "common.cuh"
#include "tile_conv.h"

namespace spc {
bool tile_bww_supported(bool check_input, const DevShape& sh, int V);
cudaError_t launch_tile_bww(bool check_input, bool sparse, const DevShape& sh, const float* chk, const float* oth,
                            float* dst, unsigned long long* exec_ctr, cudaStream_t st);
#ifdef SPC_DEV
cudaError_t launch_tile_bww_variant(int variant, bool check_input, bool sparse, const DevShape& sh, const float* chk,
                                    const float* oth, float* dst, unsigned long long* exec_ctr, cudaStream_t st);
#endif
// both_finite_gated: *sel == want implies BOTH operands are finite (allows the counted-dense
// configurations, which execute every FMA)
cudaError_t launch_tile_bww_when(bool check_input, bool sparse, const DevShape& sh, const float* chk,
                                 const float* oth, float* dst, unsigned long long* exec_ctr, cudaStream_t st,
                                 const int* sel, int want, bool both_finite_gated = false);
// true when launch_tile_bww_when runs this shape counted dense (every FMA executes): the gate word
// must then cover the finiteness of BOTH operands
bool tile_bww_counted_dense(bool check_input, const DevShape& sh);
// row_bww.cu: check = input, 3x3 stride 1 pad 1 (row-streaming window kernel)
bool row_bww_supported(bool check_input, const DevShape& sh, int V);
// runs when *sel == 1 (the checked tensor is finite), exits otherwise
cudaError_t launch_row_bww_when(bool sparse, const DevShape& sh, const float* chk, const float* oth, float* dst,
                                unsigned long long* exec_ctr, const int* sel, cudaStream_t st);

// tma_bww.cu: check = input, 3x3 stride 1 pad 1, K % 128 == 0 (TMA-staged tile kernel)
bool tma_bww_supported(bool check_input, const DevShape& sh, int V);
// runs when *sel == want (sel == nullptr: always).  scan_flag (normally == sel, want == 1): the kernel's
// pre-pass over the checked tensor also is its finiteness scan -- it presets the flag to 1 and clears it
// on Inf / NaN, replacing a separate launch_finite_all
cudaError_t launch_tma_bww_when(bool sparse, const DevShape& sh, const float* chk, const float* oth, float* dst,
                                unsigned long long* exec_ctr, const int* sel, int want, cudaStream_t st,
                                int* scan_flag = nullptr);

}  // namespace spc
