// pw_gemm.cu -- 1x1 FWD / BWI (stride 1 or 2, V = 16) as a register-blocked GEMM.
//
// Y[i, co, o] = sum_ci W[co, ci] * X[i, ci, s(o)]: M = output channels, N = the
// flattened (image, output pixel) index, reduction = input channels.  Same
// policy as pw_conv.cu / pw_bww.cu (measured: per-element or per-quad zero
// branches never beat dense FMAs for 1x1 on B200): every FMA executes, zero
// products are exact for finite filters, and a filter with Inf/NaN runs the
// EXACT instantiation, which applies an FMA only where X != 0 (the reference's
// skip, P/include/spconv/vec.hpp:120-128).  executed_vector_fmas counts the
// nonzero staged X elements x Co/16 -- the reference's count.
//
// Tiles: CTA = BK output channels x 128 (image, pixel) rows; per 16-channel
// reduction step it stages
//   Xs[p][c]  the 128 rows' 16 channels, pixel-major exactly as ActNCHWc
//             stores them (16-byte cp.async, 20-float rows: the strided-p
//             LDS.128 of a thread hit 8 distinct bank groups per phase);
//   Ws[c][k]  16 input channels x BK output channels from FilterKCRSblk
//             ([Co/16][Ci/16][16 ci][16 co], 64 contiguous bytes per (ci, co-block)).
// Each thread owns 4 output-channel pairs x 8 rows (FFMA2 over the pair, X
// broadcast), 4-stage cp.async pipeline.  The fused epilogue (Epi) applies at
// the store.  Stride 2: FWD reads source pixel 2o; BWI rows are the SOURCE
// pixels (an output-pixel row space would spend 3/4 of its FMAs on the stride
// gaps: measured 1145 us against 330 us of useful work on ResNet-50's stage-2
// projection), and each row also writes its 2x2 cell's gap pixels, which
// accumulate nothing (exactly 0, epilogue applied).
#include <cstdint>

#include "common.cuh"
#include "pw_gemm.h"

namespace spc {
namespace {

constexpr int PG_BP = 128;  // rows (image, output pixel) per CTA
constexpr int PG_NST = 4;
constexpr int PG_XS = 20;   // padded Xs row (floats)

__device__ __forceinline__ uint32_t pg_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <bool FWD, int BK, int STR, bool COUNT, bool EXACT>
__global__ void __launch_bounds__((BK / 8) * 16, 2) pw_gemm_kernel(DevShape sh, const float* __restrict__ src,
                                                               const float* __restrict__ filt,
                                                               float* __restrict__ dst,
                                                               unsigned long long* __restrict__ exec_ctr,
                                                               const int* __restrict__ finite, Epi epi) {
    if ((__ldg(finite) != 0) == EXACT) return;  // EXACT runs only for a filter with Inf/NaN
    constexpr int NT = (BK / 8) * 16;
    constexpr int WS = BK + 4;  // padded Ws row
    extern __shared__ __align__(16) float smem[];
    float* Xs = smem;                            // [NST][BP][PG_XS]
    float* Ws = smem + PG_NST * PG_BP * PG_XS;   // [NST][16][WS]

    const int Co = FWD ? sh.K : sh.C, Ci = FWD ? sh.C : sh.K;
    const int Hs = FWD ? sh.H : sh.Hp, Wsrc = FWD ? sh.W : sh.Wp;
    const int Ho = FWD ? sh.Hp : sh.H, Wo = FWD ? sh.Wp : sh.W;
    const int CiB = Ci / 16, CoB = Co / 16;
    const int HWo = Ho * Wo;
    constexpr bool SRCROWS = !FWD && STR > 1;  // BWI stride 2: one row per source pixel
    const int HWr = SRCROWS ? Hs * Wsrc : HWo;
    const long rows = (long)sh.N * HWr;
    const int ktile = blockIdx.y;
    const long row0 = (long)blockIdx.x * PG_BP;
    const int k_base = ktile * BK;
    const int tid = threadIdx.x;
    const int tx = tid & 15, ty = tid >> 4;

    // per-thread staging tasks: rows x 4 chunks of 16 B; source offsets fixed per CTA
    constexpr int XT = PG_BP * 4 / NT;
    long x_src[XT];
    uint32_t x_dst[XT];
#pragma unroll
    for (int t = 0; t < XT; ++t) {
        const int task = tid + t * NT;
        const int p = task >> 2, q = task & 3;
        const long row = row0 + p;
        long off = -1;
        if (row < rows) {
            const int i = (int)(row / HWr), o = (int)(row % HWr);
            int sidx = -1;
            if (FWD) {
                const int oy = o / Wo, ox = o - oy * Wo;
                sidx = (oy * STR) * Wsrc + ox * STR;
            } else {
                sidx = o;  // stride 1: output pixel = source pixel; stride 2: the row IS the source pixel
            }
            if (sidx >= 0) off = ((long)i * CiB * Hs * Wsrc + sidx) * 16 + q * 4;  // + cb * Hs*Wsrc*16
        }
        x_src[t] = off;
        x_dst[t] = (uint32_t)(p * PG_XS + q * 4) * 4u;
    }
    const long plane = (long)Hs * Wsrc * 16;
    auto stage = [&](int cb, int buf) {
        if (cb < CiB) {
            const uint32_t xb = pg_smem_u32(Xs + (size_t)buf * PG_BP * PG_XS);
#pragma unroll
            for (int t = 0; t < XT; ++t) {
                const bool ok = x_src[t] >= 0;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(xb + x_dst[t]),
                             "l"(ok ? src + x_src[t] + (long)cb * plane : src), "r"(ok ? 16 : 0));
            }
            // Ws[c][k]: 16 c x BK k; element (co, ci) at ((co/16 * CiB + ci/16) * 256) + (ci%16)*16 + co%16
            const uint32_t wb = pg_smem_u32(Ws + (size_t)buf * 16 * WS);
            for (int t = tid; t < 16 * BK / 4; t += NT) {
                const int c = t / (BK / 4), k4 = t % (BK / 4);
                const int k = k4 * 4;
                const float* g = filt + ((size_t)((k_base + k) / 16) * CiB + cb) * 256 + c * 16 + (k_base + k) % 16;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(wb + (uint32_t)(c * WS + k) * 4u),
                             "l"(g));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };

    // thread tile: k pairs {ty*2, ty*2+1} and {BK/4 + ty*2, +1}; rows p = tx + 16*j
    float2 acc[4][8];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[a][j] = make_float2(0.0f, 0.0f);
    const int k0 = ty * 4, k1 = BK / 2 + ty * 4;  // element offsets of the two 4-k groups
    uint32_t nz = 0;

#pragma unroll
    for (int d = 0; d < PG_NST - 1; ++d) stage(d, d);
    for (int cb = 0; cb < CiB; ++cb) {
        stage(cb + PG_NST - 1, (cb + PG_NST - 1) % PG_NST);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PG_NST - 1));
        __syncthreads();
        const float* X = Xs + (size_t)(cb % PG_NST) * PG_BP * PG_XS;
        const float* W = Ws + (size_t)(cb % PG_NST) * 16 * WS;
        if (COUNT && ktile == 0) {
            for (int t = tid; t < PG_BP * 16; t += NT) nz += X[(t >> 4) * PG_XS + (t & 15)] != 0.0f;
        }
#pragma unroll
        for (int c4 = 0; c4 < 16; c4 += 4) {
            float4 b[8];  // rows p_j, channels c4..c4+3
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const float4*>(X + (tx + 16 * j) * PG_XS + c4);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const float4 w0 = *reinterpret_cast<const float4*>(W + (c4 + cc) * WS + k0);
                const float4 w1 = *reinterpret_cast<const float4*>(W + (c4 + cc) * WS + k1);
                const float2 pr[4] = {make_float2(w0.x, w0.y), make_float2(w0.z, w0.w), make_float2(w1.x, w1.y),
                                      make_float2(w1.z, w1.w)};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float v = cc == 0 ? b[j].x : cc == 1 ? b[j].y : cc == 2 ? b[j].z : b[j].w;
                    if constexpr (EXACT) {
                        if (v != 0.0f) {
#pragma unroll
                            for (int a = 0; a < 4; ++a) acc[a][j] = __ffma2_rn(pr[a], make_float2(v, v), acc[a][j]);
                        }
                    } else {
#pragma unroll
                        for (int a = 0; a < 4; ++a) acc[a][j] = __ffma2_rn(pr[a], make_float2(v, v), acc[a][j]);
                    }
                }
            }
        }
        __syncthreads();
    }

    // store: row (i, o), channels k_base + {k0..k0+3, k1..k1+3}
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const long row = row0 + tx + 16 * j;
        if (row < rows) {
            const int i = (int)(row / HWr);
            int o = (int)(row % HWr);
            int oy = 0, ox = 0;
            if constexpr (SRCROWS) {
                oy = (o / Wsrc) * STR;
                ox = (o % Wsrc) * STR;
                o = oy * Wo + ox;
            }
#pragma unroll
            for (int g = 0; g < 2; ++g) {
                const int k = k_base + (g ? k1 : k0);
                const size_t off = (((size_t)i * CoB + k / 16) * HWo + o) * 16 + (k % 16);
                float v[4] = {acc[2 * g][j].x, acc[2 * g][j].y, acc[2 * g + 1][j].x, acc[2 * g + 1][j].y};
                if (epi.active()) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[e] = epi.apply(v[e], off + e);
                }
                *reinterpret_cast<float4*>(dst + off) = make_float4(v[0], v[1], v[2], v[3]);
                if constexpr (SRCROWS) {  // the cell's gap pixels
#pragma unroll
                    for (int dy = 0; dy < STR; ++dy)
#pragma unroll
                        for (int dx = 0; dx < STR; ++dx) {
                            if ((dy == 0 && dx == 0) || oy + dy >= Ho || ox + dx >= Wo) continue;
                            const size_t goff = off + (size_t)(dy * Wo + dx) * 16;
                            float z[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                            if (epi.active()) {
#pragma unroll
                                for (int e = 0; e < 4; ++e) z[e] = epi.apply(0.0f, goff + e);
                            }
                            *reinterpret_cast<float4*>(dst + goff) = make_float4(z[0], z[1], z[2], z[3]);
                        }
                }
            }
        }
    }
    if (COUNT && ktile == 0 && exec_ctr) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, nz);
        if ((tid & 31) == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * CoB);
    }
}

template <bool FWD, int BK, int STR>
cudaError_t pg_launch(bool sparse, const DevShape& sh, const float* src, const float* filt, float* dst,
                      unsigned long long* exec_ctr, const int* finite, cudaStream_t st, const Epi& epi) {
    constexpr int NT = (BK / 8) * 16;
    const int Co = FWD ? sh.K : sh.C;
    const int Ho = FWD ? sh.Hp : sh.H, Wo = FWD ? sh.Wp : sh.W;
    const long rows = (!FWD && STR > 1) ? (long)sh.N * sh.Hp * sh.Wp : (long)sh.N * Ho * Wo;
    const size_t smem = (size_t)PG_NST * (PG_BP * PG_XS + 16 * (BK + 4)) * sizeof(float);
    auto k0 = sparse ? pw_gemm_kernel<FWD, BK, STR, true, false> : pw_gemm_kernel<FWD, BK, STR, false, false>;
    auto k1 = sparse ? pw_gemm_kernel<FWD, BK, STR, true, true> : pw_gemm_kernel<FWD, BK, STR, false, true>;
    cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid((unsigned)((rows + PG_BP - 1) / PG_BP), Co / BK, 1);
    k0<<<grid, NT, smem, st>>>(sh, src, filt, dst, exec_ctr, finite, epi);
    k1<<<grid, NT, smem, st>>>(sh, src, filt, dst, exec_ctr, finite, epi);
    note_launch(2);
    return cudaGetLastError();
}

template <bool FWD>
cudaError_t pg_pick(bool sparse, const DevShape& sh, const float* src, const float* filt, float* dst,
                    unsigned long long* exec_ctr, const int* finite, cudaStream_t st, const Epi& epi) {
    const int Co = FWD ? sh.K : sh.C;
    if (Co % 128 == 0)
        return sh.O == 1 ? pg_launch<FWD, 128, 1>(sparse, sh, src, filt, dst, exec_ctr, finite, st, epi)
                         : pg_launch<FWD, 128, 2>(sparse, sh, src, filt, dst, exec_ctr, finite, st, epi);
    return sh.O == 1 ? pg_launch<FWD, 64, 1>(sparse, sh, src, filt, dst, exec_ctr, finite, st, epi)
                     : pg_launch<FWD, 64, 2>(sparse, sh, src, filt, dst, exec_ctr, finite, st, epi);
}

}  // namespace

bool pw_gemm_supported(bool fwd, const DevShape& sh, int V) {
    (void)fwd;
    if (V != 16 || sh.R != 1 || sh.S != 1 || sh.O != sh.P || sh.padW != 0 || sh.padH != 0) return false;
    if (sh.O != 1 && sh.O != 2) return false;
    return sh.C % 64 == 0 && sh.K % 64 == 0;
}

cudaError_t launch_pw_gemm(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, const int* finite, cudaStream_t st,
                           const Epi& epi) {
    return fwd ? pg_pick<true>(sparse, sh, src, filt, dst, exec_ctr, finite, st, epi)
               : pg_pick<false>(sparse, sh, src, filt, dst, exec_ctr, finite, st, epi);
}

}  // namespace spc
