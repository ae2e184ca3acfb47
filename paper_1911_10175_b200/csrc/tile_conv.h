// tile_conv.h -- tuned V=16 FWD/BWI tile kernels (internal).
#pragma once
#include "common.cuh"

namespace spc {
bool tile_conv_supported(bool fwd, const DevShape& sh, int V);
cudaError_t launch_tile_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                             float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi = Epi{},
                             const int* sel = nullptr, int want = 0, const Gate& gate = Gate{});
cudaError_t launch_tile_conv_variant(int variant, bool fwd, bool sparse, const DevShape& sh, const float* src,
                                     const float* filt, float* dst, unsigned long long* exec_ctr, cudaStream_t st);
cudaError_t launch_tile_conv_when(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                                  float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi,
                                  const int* sel, int want);
// Device-side selector for the jump-table kernels: sel = density <= pct%.
void launch_density_probe(const float* t, size_t n, int pct, int* sel, cudaStream_t st, const Gate& gate = Gate{});
}  // namespace spc
