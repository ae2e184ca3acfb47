// common.cuh -- shared device-side definitions for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spconv_b200.h"

namespace spc {

// conv_shape plus derived output extents, passed by value to kernels.
struct DevShape {
    int N, C, K, H, W, R, S, O, P, padW, padH;
    int Hp, Wp;  // out_h(), out_w()  (P/include/spconv/tensor.hpp:44-45)
};

inline DevShape make_dev_shape(const spc_shape& s) {
    DevShape d;
    d.N = s.N; d.C = s.C; d.K = s.K; d.H = s.H; d.W = s.W; d.R = s.R; d.S = s.S;
    d.O = s.O; d.P = s.P; d.padW = s.padW; d.padH = s.padH;
    d.Wp = (s.W + 2 * s.padW - s.R) / s.O + 1;
    d.Hp = (s.H + 2 * s.padH - s.S) / s.P + 1;
    return d;
}

// Blocked layout address maps (P/include/spconv/tensor.hpp:98-119).
// ActNCHWc: element (i, ch, y, x) of a tensor with `chans` channels.
__host__ __device__ __forceinline__ size_t act_index(int chans, int rows, int cols, int V, int i, int ch,
                                                     int y, int x) {
    return ((((size_t)i * (chans / V) + ch / V) * rows + y) * cols + x) * V + ch % V;
}
// ActCHWNn: element (i, ch, y, x).
__host__ __device__ __forceinline__ size_t chwnn_index(int chans, int rows, int cols, int V, int i, int ch,
                                                       int y, int x) {
    return ((((size_t)(i / V) * chans + ch) * rows + y) * cols + x) * V + i % V;
}
// FilterKCRSblk with `cdim` input channels: element (k, c, u, v).
__host__ __device__ __forceinline__ size_t filter_index(int cdim, int S, int R, int V, int k, int c, int u,
                                                        int v) {
    return (((((size_t)(k / V) * (cdim / V) + c / V) * S + v) * R + u) * V + c % V) * V + k % V;
}

// Warp-aggregated u64 counter add from the lanes that hold a count.
__device__ __forceinline__ void warp_count_add(unsigned long long* ctr, unsigned v) {
    if (!ctr) return;
    const unsigned total = __reduce_add_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && total) atomicAdd(ctr, (unsigned long long)total);
}

}  // namespace spc

// Host-side launch bookkeeping shared by every translation unit.
namespace spc {
void note_launch(unsigned n = 1);
}
