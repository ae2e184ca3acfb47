// pw_conv.cu -- 1x1 (pointwise) FWD / BWI, stride 1 or 2, V = 16.
//
// A 1x1 conv is a GEMM over (pixels x input channels x output channels):
// Y[i, co, o] = sum_ci W[co, ci] * X[i, ci, s(o)] with s(o) the source pixel
// of output pixel o (FWD: o*STR; BWI: o/STR when o is on the stride grid, else
// none -- the stride gaps stay exactly 0, P/tests/test_kernels.cpp:354-385).
//
// Zero skipping does not pay at this granularity on B200, so this kernel
// executes every FMA and counts the reference's executed_vector_fmas exactly
// (per-element nonzero tests of the staged source, P/src/oracle.cpp:168-280).
// A 1x1 source element feeds ONE output pixel: a per-(pixel, channel) check
// guards KK/2 FFMA2, a per-(pixel, 4-channel quad) check 2*KK -- both measured
// SLOWER than no check at every grid sparsity (VGG/ResNet 1x1 layers, s = 0.6
// and 0.9: the warp-uniform branch per pixel costs more than the FMAs it
// skips, and a quad is all-zero only with probability s^4).  Skipped and
// executed zero products give identical results (x*0 = +-0, acc + +-0 = acc)
// as long as the filter is finite; a filter holding Inf/NaN (0*Inf = NaN where
// the reference skips) runs the per-element-skip 1x1 tile kernel instead
// (device-side flag, both launched, one exits), so the reference's semantics
// hold for every input.
//
// Layout: the CTA's 32 output pixels x 16 source channels are staged
// pixel-major (the global ActNCHWc order, cp.async 16 B, no transpose) with a
// 20-float pixel stride, so the per-lane LDS.128 of the zero test is
// conflict-free.  Each warp owns 32*KK output channels (lanes own KK each, the
// filter vector of the current channel quad in registers, the next quad's in
// flight); NWK warps of a CTA share the staged pixels.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "pw_conv.h"

namespace spc {
namespace {

constexpr int PW_P = 32;     // output pixels per CTA (one per ballot bit)
constexpr int PW_PS = 20;    // padded pixel stride in floats (conflict-free LDS.128)
constexpr int PW_NST = 4;    // staging pipeline depth (16-channel blocks in flight)

__device__ __forceinline__ uint32_t pw_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int KK>
struct PwVec {
    float v[KK];
    __device__ __forceinline__ void load(const float* p) {
        if constexpr (KK == 4) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(p));
            v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        } else {
            static_assert(KK == 2, "KK in {2, 4}");
            const float2 t = __ldg(reinterpret_cast<const float2*>(p));
            v[0] = t.x; v[1] = t.y;
        }
    }
};

// acc[j] += d * g[j]; packed FFMA2 for KK >= 4 (common.cuh fma_lane rationale)
template <int KK>
__device__ __forceinline__ void pw_fma(float (&a)[KK], float d, const PwVec<KK>& g) {
    if constexpr (KK >= 4) {
        const float2 dd = make_float2(d, d);
#pragma unroll
        for (int j = 0; j < KK; j += 2) {
            const float2 r = __ffma2_rn(dd, make_float2(g.v[j], g.v[j + 1]), make_float2(a[j], a[j + 1]));
            a[j] = r.x;
            a[j + 1] = r.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < KK; ++j) a[j] = fmaf(d, g.v[j], a[j]);
    }
}

// One CTA = 32 output pixels x NWK*32*KK output channels of one image.
template <bool FWD, int KK, int NWK, int STR, bool COUNT>
__global__ void __launch_bounds__(NWK * 32) pw_conv_kernel(DevShape sh, const float* __restrict__ src,
                                                           const float* __restrict__ filt, float* __restrict__ dst,
                                                           unsigned long long* __restrict__ exec_ctr,
                                                           const int* __restrict__ finite, Epi epi, Gate gate) {
    // a filter with Inf/NaN runs the per-element-skip tile kernel instead
    // (launched alongside with the same flag, want = 0)
    if (finite != nullptr && __ldg(finite) == 0) return;
    gate.wait_input(blockIdx.y);
    constexpr int NT = NWK * 32;
    __shared__ __align__(16) float Xs[PW_NST][PW_P * PW_PS];

    const int Co = FWD ? sh.K : sh.C, Ci = FWD ? sh.C : sh.K;
    const int Hs = FWD ? sh.H : sh.Hp, Ws = FWD ? sh.W : sh.Wp;
    const int Ho = FWD ? sh.Hp : sh.H, Wo = FWD ? sh.Wp : sh.W;
    const int CiB = Ci / 16, CoB = Co / 16;
    const int HWo = Ho * Wo;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntile = (HWo + PW_P - 1) / PW_P;
    const int tile = blockIdx.x % ntile;
    const int kg = (blockIdx.x / ntile) * NWK + warp;  // this warp's group of 32*KK output channels
    const int i = blockIdx.y;
    const int o0 = tile * PW_P;
    const int k0 = kg * 32 * KK + lane * KK;

    // source pixel of output pixel o (or -1: stride gap / past the image)
    auto source = [&](int o) -> int {
        if (o >= HWo) return -1;
        const int oy = o / Wo, ox = o - oy * Wo;
        if (FWD) return (oy * STR) * Ws + ox * STR;
        if (STR > 1 && (oy % STR || ox % STR)) return -1;
        const int sy = oy / STR, sx = ox / STR;
        return (sy < Hs && sx < Ws) ? sy * Ws + sx : -1;
    };

    // staging tasks: 32 pixels x 4 chunks of 16 B; per thread a fixed list
    constexpr int NTASK = PW_P * 4 / NT;
    int t_src[NTASK];
    uint32_t t_dst[NTASK];
#pragma unroll
    for (int t = 0; t < NTASK; ++t) {
        const int task = threadIdx.x + t * NT;
        const int p = task >> 2, ch4 = task & 3;
        const int sidx = source(o0 + p);
        t_src[t] = sidx < 0 ? -1 : sidx * 16 + ch4 * 4;
        t_dst[t] = (uint32_t)(p * PW_PS + ch4 * 4) * 4u;
    }
    const size_t plane = (size_t)Hs * Ws * 16;  // one 16-channel block of the source image
    const float* sbase = src + (size_t)i * CiB * plane;
    auto stage = [&](int cb, int buf) {
        const float* sp = sbase + (size_t)cb * plane;
        const uint32_t d0 = pw_smem_u32(&Xs[buf][0]);
#pragma unroll
        for (int t = 0; t < NTASK; ++t) {
            const bool ok = t_src[t] >= 0;
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d0 + t_dst[t]),
                         "l"(ok ? sp + t_src[t] : sp), "r"(ok ? 16 : 0));
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };

    float acc[PW_P][KK];
#pragma unroll
    for (int p = 0; p < PW_P; ++p)
#pragma unroll
        for (int j = 0; j < KK; ++j) acc[p][j] = 0.0f;

    // filter element (co, ci) at ((co/16 * CiB + ci/16) * 256) + (ci%16)*16 + co%16
    const float* fbase = filt + (size_t)(k0 / 16) * CiB * 256 + (k0 % 16);
    uint32_t nzcount = 0;  // nonzero source elements of this lane's pixel (exact counter)

#pragma unroll
    for (int d = 0; d < PW_NST - 1; ++d) {
        if (d < CiB) stage(d, d);
        else asm volatile("cp.async.commit_group;\n" ::);
    }
    PwVec<KK> g[4], gn[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) g[c].load(fbase + c * 16);

    for (int cb = 0; cb < CiB; ++cb) {
        if (cb + PW_NST - 1 < CiB) stage(cb + PW_NST - 1, (cb + PW_NST - 1) % PW_NST);
        else asm volatile("cp.async.commit_group;\n" ::);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PW_NST - 1));
        __syncthreads();
        const float* X = &Xs[cb % PW_NST][0];
        const float* fcb = fbase + (size_t)cb * 256;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // next quad's filter vectors in flight while this quad computes
            const float* nf = q < 3 ? fcb + (q + 1) * 64 : fcb + 256;
            if (q < 3 || cb + 1 < CiB) {
#pragma unroll
                for (int c = 0; c < 4; ++c) gn[c].load(nf + c * 16);
            }
            if (COUNT) {
                const float4 mine = *reinterpret_cast<const float4*>(X + lane * PW_PS + q * 4);
                nzcount += (uint32_t)(mine.x != 0.0f) + (uint32_t)(mine.y != 0.0f) + (uint32_t)(mine.z != 0.0f) +
                           (uint32_t)(mine.w != 0.0f);
            }
#pragma unroll
            for (int p = 0; p < PW_P; ++p) {
                const float4 d = *reinterpret_cast<const float4*>(X + p * PW_PS + q * 4);
                pw_fma(acc[p], d.x, g[0]);
                pw_fma(acc[p], d.y, g[1]);
                pw_fma(acc[p], d.z, g[2]);
                pw_fma(acc[p], d.w, g[3]);
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) g[c] = gn[c];
        }
        __syncthreads();  // the buffer is restaged PW_NST-1 blocks later
    }

    // epilogue: every output pixel of the tile written once (gaps -> acc = 0)
#pragma unroll
    for (int p = 0; p < PW_P; ++p) {
        const int o = o0 + p;
        if (o < HWo) {
            const size_t off = (((size_t)i * CoB + k0 / 16) * HWo + o) * 16 + (k0 % 16);
            float v[KK];
#pragma unroll
            for (int j = 0; j < KK; ++j) v[j] = epi.active() ? epi.apply(acc[p][j], off + j) : acc[p][j];
            if constexpr (KK == 4)
                *reinterpret_cast<float4*>(dst + off) = make_float4(v[0], v[1], v[2], v[3]);
            else
                *reinterpret_cast<float2*>(dst + off) = make_float2(v[0], v[1]);
        }
    }
    if (COUNT && exec_ctr) {
        // each staged source element is delivered to this warp once; a nonzero
        // feeds its one output pixel x the warp's 32*KK channels = 2*KK vector FMAs
        const uint32_t total = __reduce_add_sync(0xffffffffu, nzcount);
        if (lane == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (2 * KK));
    }
    gate.finish(blockIdx.y);
}

// flag = 1 when every filter element is finite (zero-quad skipping is then
// exact), else 0 (per-element tests).
__global__ void __launch_bounds__(256) filter_finite_kernel(const float* __restrict__ f, size_t n, int* flag) {
    __shared__ int bad;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    int b = 0;
    for (size_t e = threadIdx.x; e < n; e += blockDim.x) b |= !isfinite(f[e]);
    if (b) bad = 1;
    __syncthreads();
    if (threadIdx.x == 0) *flag = bad ? 0 : 1;
}

template <bool FWD, int KK, int NWK, int STR>
cudaError_t pw_launch(bool sparse, const DevShape& sh, const float* src, const float* filt, float* dst,
                      unsigned long long* exec_ctr, cudaStream_t st, const int* finite, const Epi& epi, const Gate& gate) {
    const int Co = FWD ? sh.K : sh.C;
    const int Ho = FWD ? sh.Hp : sh.H, Wo = FWD ? sh.Wp : sh.W;
    const int ntile = (Ho * Wo + PW_P - 1) / PW_P;
    dim3 grid(ntile * (Co / (32 * KK * NWK)), sh.N, 1);
    if (sparse)
        pw_conv_kernel<FWD, KK, NWK, STR, true><<<grid, NWK * 32, 0, st>>>(sh, src, filt, dst, exec_ctr, finite, epi, gate);
    else
        pw_conv_kernel<FWD, KK, NWK, STR, false><<<grid, NWK * 32, 0, st>>>(sh, src, filt, dst, exec_ctr, finite, epi, gate);
    note_launch();
    return cudaGetLastError();
}

template <bool FWD, int STR>
cudaError_t pw_pick(bool sparse, const DevShape& sh, const float* src, const float* filt, float* dst,
                    unsigned long long* exec_ctr, cudaStream_t st, const int* finite, const Epi& epi, const Gate& gate) {
    const int Co = FWD ? sh.K : sh.C;
    if (Co % 512 == 0) return pw_launch<FWD, 4, 4, STR>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
    if (Co % 256 == 0) return pw_launch<FWD, 4, 2, STR>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
    if (Co % 128 == 0) return pw_launch<FWD, 4, 1, STR>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
    return pw_launch<FWD, 2, 1, STR>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
}

}  // namespace

bool pw_conv_supported(bool fwd, const DevShape& sh, int V) {
    (void)fwd;
    if (V != 16 || sh.R != 1 || sh.S != 1 || sh.O != sh.P || sh.padW != 0 || sh.padH != 0) return false;
    if (sh.O != 1 && sh.O != 2) return false;
    return sh.C % 64 == 0 && sh.K % 64 == 0;
}

cudaError_t launch_pw_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, cudaStream_t st, const int* finite,
                           const Epi& epi, const Gate& gate) {
    if (fwd) return sh.O == 1 ? pw_pick<true, 1>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate)
                              : pw_pick<true, 2>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
    return sh.O == 1 ? pw_pick<false, 1>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate)
                     : pw_pick<false, 2>(sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
}

void launch_filter_finite(const float* filt, size_t n, int* flag, cudaStream_t st) {
    filter_finite_kernel<<<1, 256, 0, st>>>(filt, n, flag);
    note_launch();
}

}  // namespace spc
