// dispatch.h -- kernel selection behind the C ABI (internal).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace spc {

int math_mode();
void set_math_mode(int m);

// FWD (fwd=true) or BWI: picks the tuned V=16 tile kernel when the geometry
// has one, else the shape-general kernel.
cudaError_t launch_conv(bool fwd, bool sparse, const DevShape& sh, int V, const float* src, const float* filt,
                        float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi = Epi{},
                        const Gate& gate = Gate{});
// True when launch_conv runs a kernel that honours a Gate (tile / 1x1 paths).
bool conv_supports_gate(bool fwd, const DevShape& sh, int V);

// Standalone epilogue over n output elements (the generic kernels' path).
cudaError_t launch_epilogue(const Epi& epi, float* out, size_t n, cudaStream_t st);

// BWW: partial sums + fixed-order reduction into FilterKCRSblk (K, C).
cudaError_t launch_bww(bool check_input, bool sparse, const DevShape& sh, int V, const float* chk,
                       const float* oth, float* dst, unsigned long long* exec_ctr, cudaStream_t st);

// generic.cu
cudaError_t launch_conv_generic(bool fwd, bool sparse, const DevShape& sh, int V, const float* src,
                                const float* filt, float* dst, unsigned long long* exec_ctr, cudaStream_t st);
int bww_generic_splits(const DevShape& sh);
cudaError_t launch_bww_generic(bool check_input, bool sparse, const DevShape& sh, int V, const float* chk,
                               const float* oth, float* partial, int splits, float* dst,
                               unsigned long long* exec_ctr, cudaStream_t st, const int* sel = nullptr,
                               int want = 0);

}  // namespace spc
