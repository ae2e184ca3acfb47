// common.cuh -- shared device-side definitions for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/spconv_b200.h"

namespace spc {

// conv_shape plus derived output extents, passed by value to kernels.
struct DevShape {
    int N, C, K, H, W, R, S, O, P, padW, padH;
    int Hp, Wp;  // out_h(), out_w()  (P/include/spconv/tensor.hpp:44-45)
};

// Fused output epilogue of FWD/BWI: out = acc*alpha (+ add)
// (+ beta, a scalar bias: Fixup's), then ReLU (v > 0 ? v : 0,
// P/src/sparsity.cpp:13), then the ReLU-gradient mask (mask > 0 ? v : 0,
// P/src/sparsity.cpp:26).  `add` and `mask` have the output's ActNCHWc
// layout.  The identity epilogue leaves acc untouched.
struct Epi {
    float alpha = 1.0f;
    const float* add = nullptr;
    const float* mask = nullptr;
    int relu = 0;
    float beta = 0.0f;
    __host__ __device__ bool active() const { return alpha != 1.0f || add || mask || relu || beta != 0.0f; }
    __device__ __forceinline__ float apply(float v, size_t i) const {
        v = add ? fmaf(v, alpha, add[i]) : v * alpha;
        if (beta != 0.0f) v += beta;
        if (relu) v = v > 0.0f ? v : 0.0f;
        if (mask) v = mask[i] > 0.0f ? v : 0.0f;
        return v;
    }
};

// Copy/compute overlap inside ONE launch (the host-buffer path): the CTAs of
// image i wait for the ready word of i's input chunk, which the copy-in
// stream raises (stream memory op) right after that chunk's H2D; the last CTA
// to finish a chunk raises its out_ready word, on which the copy-out stream
// waits before that chunk's D2H.  Disabled when in_ready == nullptr.  Waits
// are bounded (a stuck copy sets *err instead of hanging the GPU).
struct Gate {
    const unsigned* in_ready = nullptr;
    unsigned* done = nullptr;       // finished CTAs per chunk
    unsigned* out_ready = nullptr;  // 1 once all of a chunk's outputs are written
    unsigned* err = nullptr;
    int ipc = 1;                    // images per chunk
    int nimg = 0;                   // images in the launch

    __device__ __forceinline__ void wait_input(int image) const {
        if (in_ready == nullptr) return;
        if (threadIdx.x == 0) {
            const unsigned* w = in_ready + image / ipc;
            for (unsigned n = 0;; ++n) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(w) : "memory");
                if (v) break;
                if ((n & 1023u) == 0 && *(volatile const unsigned*)err) break;  // another CTA gave up
                if (n > (1u << 24)) {  // ~seconds: give up, report
                    atomicExch(err, 1u);
                    break;
                }
                __nanosleep(200);
            }
        }
        __syncthreads();
    }
    __device__ __forceinline__ void finish(int image) const {
        if (done == nullptr) return;
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            const int c = image / ipc;
            const int in_chunk = (nimg - c * ipc) < ipc ? (nimg - c * ipc) : ipc;
            const unsigned expected = gridDim.x * (unsigned)in_chunk;
            if (atomicAdd(done + c, 1u) + 1u == expected) {
                __threadfence_system();  // out_ready is mapped host memory the host thread polls
                asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(out_ready + c), "r"(1u) : "memory");
            }
        }
    }
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

// acc[j] += d * g[j] for the lane's KK channels.  Packed FFMA2 (two fp32
// FMAs per instruction, each rounded exactly like fmaf) halves the issue
// slots of the FMA stream; the kernels are issue-bound, so the checks and
// staging instructions fill the freed slots.
//
// `ntap` is the number of fma_lane calls the caller's pixel block makes (a
// compile-time constant after unrolling).  ptxas if-converts blocks of <= ~7
// instructions into predicated straight-line code, which issues a ZERO
// pixel's FMAs too; so a pixel block uses FFMA2 only when it stays >= 8
// instructions that way, otherwise scalar FFMAs (the pre-FFMA2 code, where
// only the 1-tap corner blocks were predicated).  KK=2 lanes stay scalar:
// measured 15-19% slower with FFMA2 on the C=64 VGG layers.
#ifndef SPC_FFMA2
#define SPC_FFMA2 1
#endif
#ifndef SPC_FFMA2_MIN
#define SPC_FFMA2_MIN 16  // minimum FMAs per lane in a pixel block for the packed form
#endif
template <int KK, int MIN = SPC_FFMA2_MIN>
__device__ __forceinline__ void fma_lane(float (&a)[KK], float d, const float (&g)[KK], int ntap) {
    if (SPC_FFMA2 && KK >= 4 && ntap * KK >= MIN) {
        const float2 dd = make_float2(d, d);
#pragma unroll
        for (int j = 0; j < KK; j += 2) {
            const float2 r = __ffma2_rn(dd, make_float2(g[j], g[j + 1]), make_float2(a[j], a[j + 1]));
            a[j] = r.x;
            a[j + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < KK; ++j) a[j] = fmaf(d, g[j], a[j]);
    }
}

}  // namespace spc

// Host-side launch bookkeeping shared by every translation unit.
namespace spc {
void note_launch(unsigned n = 1);

// Per-(device, stream) block of device ints for the small selector / finite
// flags the dispatchers pass between kernels on one stream (allocated once,
// reused by every call on that stream: stream order makes the reuse safe).
// Slots: see FLAG_* below.  nullptr if the allocation failed.
int* stream_flags(cudaStream_t st);
enum : int { FLAG_FINITE = 0, FLAG_CONV_SEL = 1, FLAG_BWW_SEL = 2, FLAG_TC_SEL2 = 3 /* 2 ints */,
             FLAG_CONV_FINITE = 5, FLAG_COUNT = 64 };

// Kernel attributes (cudaFuncSetAttribute) live in the device context, so a
// "set once" guard must be per device: a process driving several GPUs sets
// them on each.  Usage: `static PerDeviceOnce g; int d; if (g.needed(d)) {
// ...set...; g.done(d); }`.
struct PerDeviceOnce {
    std::atomic<unsigned long long> mask{0};
    bool needed(int& dev) {
        if (cudaGetDevice(&dev) != cudaSuccess) dev = 0;
        return ((mask.load(std::memory_order_acquire) >> (dev & 63)) & 1ull) == 0;
    }
    void done(int dev) { mask.fetch_or(1ull << (dev & 63), std::memory_order_release); }
};
}
