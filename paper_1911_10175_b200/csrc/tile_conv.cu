// tile_conv.cu -- tuned sm_100a FWD / BWI kernels for V = 16 blocked layouts.
//
// The GPU restatement of the paper's K-vectorised sparse row sweep
// (P/src/kernel_impl.hpp:51-202, Alg. 2-3):
//
//   * lanes own OUTPUT channels (KK consecutive channels per lane, 32*KK per
//     warp) -- the paper's "vectorise along K" -- so every lane consumes the
//     same checked element d and the zero test is warp-uniform: one
//     __ballot_sync per 32 region pixels per channel replaces the per-vector
//     compare (vec.hpp:120-128), and a uniform branch skips all R*S*KK FMAs
//     a zero would have fed (`d != 0.0f`: -0 is zero, NaN is not);
//   * each warp keeps a TH x TW output tile x KK channels in registers for the
//     whole reduction (the ring of kernel_impl.hpp:110-157 becomes a static
//     register tile: outputs are written exactly once, never re-read);
//   * the swept tensor's region for one 16-channel block is staged in shared
//     memory with cp.async (double-buffered across channel blocks, 128-bit
//     transfers, zero-filled virtual padding), filters stream through L1 with
//     128/64-bit loads, prefetched one channel ahead;
//   * BWI runs the same body with channel roles swapped, the transposed filter
//     (pack_filter swap_kc) and the inverse spatial map (kernel_impl.hpp:85-89).
//
// Exact skip accounting (kernel_counters::executed_vector_fmas): every lane
// adds popcount(its pixel's 16-channel nonzero mask) x (valid output taps of
// that pixel) per channel block; the warp total x (2*KK vectors) is the
// reference's count (P/src/kernel_impl.hpp:188-189) independent of tiling.
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

// Minimum FMAs per lane in a pixel block for the packed form in the in-line
// (branch) loop.  16 keeps 1-3-tap blocks (image-border region pixels) as a
// branch + scalar FFMAs; 4 (every KK=4 block FFMA2, 2-6 instructions that ptxas
// if-converts) measured 7-12% SLOWER on VGG16 conv2_2-conv5_2 at s = 0.4 / 0.6
// (round 2, A/B on one box): predicated-off FFMA2s still occupy the FMA pipe.
#ifndef SPC_CONV_FFMA2_MIN
#define SPC_CONV_FFMA2_MIN 16
#endif
#include "jt_blocks.cuh"
#include "pw_bww.h"
#include "tile_conv.h"

namespace spc {

__host__ __device__ constexpr int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int KK>
struct FVec;
template <>
struct FVec<2> {
    float v[2];
    __device__ __forceinline__ void load(const float* p) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = t.x; v[1] = t.y;
    }
    __device__ __forceinline__ void store(float* p) const { *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]); }
};
template <>
struct FVec<4> {
    float v[4];
    __device__ __forceinline__ void load(const float* p) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    __device__ __forceinline__ void store(float* p) const {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};

template <>
struct FVec<8> {
    float v[8];
    __device__ __forceinline__ void load(const float* p) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        const float4 u = __ldg(reinterpret_cast<const float4*>(p) + 1);
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
        v[4] = u.x; v[5] = u.y; v[6] = u.z; v[7] = u.w;
    }
    __device__ __forceinline__ void store(float* p) const {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        *(reinterpret_cast<float4*>(p) + 1) = make_float4(v[4], v[5], v[6], v[7]);
    }
};

template <>
struct FVec<16> {
    float v[16];
    __device__ __forceinline__ void load(const float* p) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float4 t = __ldg(reinterpret_cast<const float4*>(p) + h);
            v[4 * h] = t.x; v[4 * h + 1] = t.y; v[4 * h + 2] = t.z; v[4 * h + 3] = t.w;
        }
    }
    __device__ __forceinline__ void store(float* p) const {
#pragma unroll
        for (int h = 0; h < 4; ++h)
            *(reinterpret_cast<float4*>(p) + h) = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
    }
};

// KK fp32 channels as KK/2 64-bit lanes (two channels each): the operand form
// of the packed f32x2 jump-table blocks (JtBlocks2).
template <int KK>
struct FVecP {
    unsigned long long p[KK / 2];
    __device__ __forceinline__ void load(const float* q) {
        static_assert(KK == 4, "FVecP: KK == 4 only");
        asm volatile("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(p[0]), "=l"(p[1]) : "l"(q));
    }
};
__device__ __forceinline__ float2 unpack_f32x2(unsigned long long x) {
    float2 r;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(x));
    return r;
}



// Static geometry of one warp tile.  Target = output of the pass (Y for FWD,
// dD for BWI); source = the swept tensor (D for FWD, dY for BWI).
template <bool FWD, int T, int F, int STR>  // T = tile extent, F = filter extent
struct Axis {
    static constexpr int PAD = (F - 1) / 2;
    // first source coordinate of the region relative to (tile origin mapped)
    static constexpr int R0 = FWD ? 0 : fdiv(PAD - (F - 1), STR);
    static constexpr int EXT = FWD ? (T - 1) * STR + F : fdiv(T - 1 + PAD, STR) - R0 + 1;
    // target index fed by region coordinate r through filter tap f, or -1
    __host__ __device__ static constexpr int target(int r, int f) {
        if (FWD) {
            const int num = r - f;
            if (num < 0 || num % STR) return -1;
            return num / STR < T ? num / STR : -1;
        } else {
            const int t = (R0 + r) * STR + f - PAD;
            return (t >= 0 && t < T) ? t : -1;
        }
    }
};

// One CTA = NWY x NWX warps; each warp owns a TH x TW output tile x 32*KK
// output channels (the CTA's channel group).  All warps share the staged
// source region and read the same filter lines (L1 hits after the first).
template <bool FWD, int KK, int TH, int TW, int NWY, int NWX, int R, int S, int STR>
struct ConvGeom {
    using AY = Axis<FWD, TH, S, STR>;
    using AX = Axis<FWD, TW, R, STR>;
    static constexpr int RH = AY::EXT, RWW = AX::EXT;         // one warp's region
    static constexpr int YSTEP = FWD ? TH * STR : TH / STR;   // source offset between warp tiles
    static constexpr int XSTEP = FWD ? TW * STR : TW / STR;
    static constexpr int NQ = (RWW + 3) / 4;                  // float4 chunks per warp region row
    static constexpr int RWWP = 4 * NQ;                        // padded row of a warp region
    static constexpr int NW = NWY * NWX;
    // SHARED: the warps' regions overlap inside one CTA region (halo staged
    // once) -- possible when every warp's x offset keeps rows 16B-aligned.
    // Otherwise each warp keeps its own padded copy (halos duplicated).
    static constexpr bool SHARED = NWX == 1 || XSTEP % 4 == 0;
    static constexpr int CRH = (NWY - 1) * YSTEP + RH;
    static constexpr int CRW = (NWX - 1) * XSTEP + RWW;
    static constexpr int CRWP = ((NWX - 1) * XSTEP + RWWP + 3) / 4 * 4;
    static constexpr int ROW = SHARED ? CRWP : RWWP;           // row stride inside a plane
    static constexpr int WPLANE = RH * RWWP;                   // per-warp copy, one channel
    static constexpr int PLANE = SHARED ? CRH * CRWP : NW * WPLANE;  // one channel
    static constexpr int RHW = RH * RWW;
    static constexpr int NWORD = (RHW + 31) / 32;
    static constexpr int NT = NW * 32;
    static constexpr int NST = 3;  // staging pipeline depth (channel blocks in flight)
    static constexpr int SMEM = NST * 16 * PLANE * 4;
};

// Static loop over the 32-pixel mask words of the jump-table path.
template <int W, int NW, class JB, class Acc, class Gv>
__device__ __forceinline__ void jt_words(Acc& acc, const Gv& g, const float* vv, const uint32_t* m) {
    if constexpr (W < NW) {
        if (m[W]) JB::template Word<W>::run(acc, g, vv[W], m[W]);
        jt_words<W + 1, NW, JB>(acc, g, vv, m);
    }
}

// GPF selects how the next channel's filter taps are fetched: 0 = L1
// prefetch + just-in-time loads (fewer registers), 1 = register double
// buffer (latency fully hidden, +R*S*KK registers).
// JT selects the sparse inner loop: 0 = one uniform branch per region pixel;
// 100 = jump-table dispatch over the nonzero pixels only (jt_blocks.cuh,
// generated); 1..99 = a CTA-collective choice per 16-channel block: the jump
// table when the previous block's measured density (nonzeros / region
// pixels, summed over the CTA's warps) is at most JT%, else per-pixel
// branches.  All variants accumulate in the same order (bitwise identical).

// Register caps for sparse 3x3 s1 kernels of launch_tile_conv, applied
// through tile_conv_kernel_capped.  KK=4 7x4 branches (244) and KK=4 4x8 jump
// table (228): no occupancy change (2 warps per SM sub-partition either way:
// 16K registers each), only ptxas's allocation and schedule.  KK=2 4x8 jump
// table (128, from 166): 4 warps per sub-partition instead of 3.  Measured on
// the VGG16 b32 sweep.  0 = no cap.
#ifndef SPC_TILE_MAXREG
#define SPC_TILE_MAXREG 244
#endif
#ifndef SPC_TILE_MAXREG_JT
#define SPC_TILE_MAXREG_JT 228
#endif
#ifndef SPC_TILE_MAXREG_JT2
#define SPC_TILE_MAXREG_JT2 128
#endif
constexpr int tile_maxreg(int nt, int kk, int th, int tw, int r, int str, int jt) {
    return (r != 3 || str != 1)                            ? 0
           : (kk == 2 && th * tw == 32 && jt == 100)        ? SPC_TILE_MAXREG_JT2
           : (kk != 4)                                     ? 0
           : (nt == 32 && th * tw == 28 && jt == 0)         ? SPC_TILE_MAXREG
           : (th * tw == 32 && jt == 100)                  ? SPC_TILE_MAXREG_JT
                                                           : 0;
}

template <bool FWD, int KK, int TH, int TW, int NWY, int NWX, int R, int S, int STR, int GPF, int JT, bool SPARSE,
          bool EPI>
__device__ __forceinline__ void tile_conv_body(DevShape sh, const float* __restrict__ src,
                                               const float* __restrict__ filt, float* __restrict__ dst,
                                               unsigned long long* __restrict__ exec_ctr,
                                               const int* __restrict__ sel, int want, int group_fastest, Epi epi,
                                               Gate gate) {
    using Gm = ConvGeom<FWD, KK, TH, TW, NWY, NWX, R, S, STR>;
    // device-side kernel choice (see launch_tile_conv): the variant whose
    // selector value does not match exits before touching memory
    if (sel != nullptr && __ldg(sel) != want) return;
    gate.wait_input(blockIdx.y);
    using AY = typename Gm::AY;
    using AX = typename Gm::AX;
    constexpr int RH = Gm::RH, RWW = Gm::RWW, NQ = Gm::NQ, ROW = Gm::ROW;
    constexpr int PLANE = Gm::PLANE, WPLANE = Gm::WPLANE, RHW = Gm::RHW, NWORD = Gm::NWORD, NT = Gm::NT;
    constexpr int TAPS = R * S;

    // channel-major staging of the swept tensor: [buf][16 channels][CRH][CRWP]
    extern __shared__ __align__(16) float Ds[];
    __shared__ int wnnz[NWY * NWX];  // per-warp nonzero count of the last channel block

    const int Co = FWD ? sh.K : sh.C, Ci = FWD ? sh.C : sh.K;
    const int Hs = FWD ? sh.H : sh.Hp, Ws = FWD ? sh.W : sh.Wp;
    const int Ho = FWD ? sh.Hp : sh.H, Wo = FWD ? sh.Wp : sh.W;
    const int CiB = Ci / 16, CoB = Co / 16;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wy = warp / NWX, wx = warp % NWX;
    const int tiles_x = (Wo + TW * NWX - 1) / (TW * NWX);
    // block order: group_fastest -> blockIdx.x = tile * groups + group, so the
    // CTAs that share a source region run back to back (its second read hits
    // L2; used when the source tensor is larger than L2 wants); otherwise
    // tile-fastest, so co-resident CTAs share a channel group's filter lines
    // in L1 (used when the source fits in L2 anyway)
    const int ngroups = Co / (32 * KK);
    const int ntile = gridDim.x / ngroups;
    const int kg = group_fastest ? blockIdx.x % ngroups : blockIdx.x / ntile;
    const int tile = group_fastest ? blockIdx.x / ngroups : blockIdx.x % ntile;
    const int ty_idx = tile / tiles_x, tx_idx = tile % tiles_x;
    const int yc0 = ty_idx * TH * NWY, xc0 = tx_idx * TW * NWX;  // target origin of the CTA
    const int y0 = yc0 + wy * TH, x0 = xc0 + wx * TW;              // target origin of this warp
    const int i = blockIdx.y;
    const int k0 = kg * 32 * KK + lane * KK;  // this lane's channels k0 .. k0+KK-1

    // source origin of the CTA region
    const int sy0 = FWD ? yc0 * STR - AY::PAD : yc0 / STR + AY::R0;
    const int sx0 = FWD ? xc0 * STR - AX::PAD : xc0 / STR + AX::R0;

    // filter element (k0, c = 16*cb + cl, u, v) at
    // (((k/16*CiB + cb)*S + v)*R + u)*256 + cl*16 + k%16
    const float* fbase = filt + (size_t)(k0 / 16) * CiB * TAPS * 256 + (k0 % 16);
    const float* sbase = src + (size_t)i * CiB * Hs * Ws * 16;

    // 4-byte cp.async transposes pixel-major global vectors into per-warp
    // channel planes (zero-filled outside the image = virtual padding):
    // element (warp w, ry, rx, ch) -> Ds[buf][ch][w][ry][rx]
    auto stage = [&](int cb, int buf) {
        const float* sp = sbase + (size_t)cb * Hs * Ws * 16;
        const uint32_t d0 = smem_u32(Ds + buf * 16 * PLANE);
        if constexpr (Gm::SHARED) {
            for (int idx = threadIdx.x; idx < Gm::CRH * Gm::CRW * 16; idx += NT) {
                const int ch = idx & 15, p = idx >> 4;
                const int ry = p / Gm::CRW, rx = p - ry * Gm::CRW;
                const int gy = sy0 + ry, gx = sx0 + rx;
                const bool ok = gy >= 0 && gy < Hs && gx >= 0 && gx < Ws;
                const float* g = ok ? sp + ((size_t)gy * Ws + gx) * 16 + ch : sp;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(
                                 d0 + (uint32_t)(ch * PLANE + ry * ROW + rx) * 4u),
                             "l"(g), "r"(ok ? 4 : 0));
            }
        } else {
            for (int idx = threadIdx.x; idx < Gm::NW * RH * RWW * 16; idx += NT) {
                const int ch = idx & 15;
                int p = idx >> 4;
                const int rx = p % RWW;
                p /= RWW;
                const int ry = p % RH;
                const int w = p / RH;
                const int gy = sy0 + (w / NWX) * Gm::YSTEP + ry, gx = sx0 + (w % NWX) * Gm::XSTEP + rx;
                const bool ok = gy >= 0 && gy < Hs && gx >= 0 && gx < Ws;
                const float* g = ok ? sp + ((size_t)gy * Ws + gx) * 16 + ch : sp;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(
                                 d0 + (uint32_t)(ch * PLANE + w * WPLANE + ry * ROW + rx) * 4u),
                             "l"(g), "r"(ok ? 4 : 0));
            }
        }
        cp_async_commit();
    };

    // this warp's region origin inside a channel plane
    const int woff = Gm::SHARED ? wy * Gm::YSTEP * ROW + wx * Gm::XSTEP : warp * WPLANE;

    // per-lane region pixels q = lane + 32w: plane offset and valid-tap
    // weight (number of (target, tap) pairs whose target is in the image)
    int qoff[NWORD];
    uint32_t wt[NWORD], nzc[NWORD];
#pragma unroll
    for (int w = 0; w < NWORD; ++w) {
        const int q = lane + 32 * w;
        int ny = 0, nx = 0;
        qoff[w] = woff;
        if (q < RHW) {
            const int ry = q / RWW, rx = q % RWW;
            qoff[w] = woff + ry * ROW + rx;
#pragma unroll
            for (int v = 0; v < S; ++v) {
                const int t = AY::target(ry, v);
                if (t >= 0 && y0 + t < Ho) ++ny;
            }
#pragma unroll
            for (int u = 0; u < R; ++u) {
                const int t = AX::target(rx, u);
                if (t >= 0 && x0 + t < Wo) ++nx;
            }
        }
        wt[w] = (uint32_t)(ny * nx);
        nzc[w] = 0;
    }

    // JTP: jump-table kernel with packed f32x2 blocks -- accumulators and taps
    // live as 64-bit channel pairs for the whole pass (no in-line path)
    using JB2 = JtBlocks2<FWD, KK, TH, TW, R, S, STR>;
    // JT == 200: "counted dense" -- every region pixel's FMAs execute (no
    // per-pixel branch) while the zero test still runs for the exact counter;
    // for geometries whose per-pixel blocks are too small for a branch to pay
    // (3x3 stride-2 FWD: ~2.25 taps per source pixel).  Finite filters only
    // (dispatch guards: 0*Inf would be NaN where the reference skips).
    constexpr bool FORCE = JT == 200;
    constexpr bool JTP = SPARSE && JT >= 100 && !FORCE && SPC_FFMA2 && JB2::available;
    constexpr int KA = JTP ? KK / 2 : KK;
    using AccT = std::conditional_t<JTP, unsigned long long, float>;
    using GV = std::conditional_t<JTP, FVecP<KK>, FVec<KK>>;
    AccT acc[TH * TW][KA];
#pragma unroll
    for (int t = 0; t < TH * TW; ++t)
#pragma unroll
        for (int j = 0; j < KA; ++j) acc[t][j] = AccT(0);

    constexpr int NST = Gm::NST;
#ifndef SPC_CONV_CUNROLL
#define SPC_CONV_CUNROLL 1
#endif
    // channel-loop unroll factor.  Measured with 2 (VGG16 b32): dense mode +4%, the sparse
    // branch kernel -3%, the jump-table kernel 3-4x slower (instruction-cache misses)
    constexpr int CUNROLL = SPC_CONV_CUNROLL;
    bool use_jt = JT >= 100 && !FORCE;  // JT in 1..99: decided per block below, starting with branches
#pragma unroll
    for (int d = 0; d < NST - 1; ++d) {
        if (d < CiB) stage(d, d);
        else cp_async_commit();
    }
    for (int cb = 0; cb < CiB; ++cb) {
        if (cb + NST - 1 < CiB) stage(cb + NST - 1, (cb + NST - 1) % NST);
        else cp_async_commit();  // keep one group per iteration
        cp_async_wait<NST - 1>();
        __syncthreads();
        const float* fcb = fbase + (size_t)cb * TAPS * 256;
        int blk_nnz = 0;  // this warp's region nonzeros over the block (uniform)
        GV g[TAPS];
        if constexpr (GPF == 1) {
#pragma unroll
            for (int f = 0; f < TAPS; ++f) g[f].load(fcb + f * 256);
        }

#pragma unroll CUNROLL
        for (int c = 0; c < 16; ++c) {
            const float* P = Ds + (cb % NST) * 16 * PLANE + c * PLANE;
            GV gn[GPF == 1 ? TAPS : 1];
            if constexpr (GPF == 0) {
                // this channel's taps: L1 hits (prefetched one channel ahead,
                // shared by the CTA's warps), issued before the mask ballots so
                // the two latencies overlap
#pragma unroll
                for (int f = 0; f < TAPS; ++f) g[f].load(fcb + f * 256 + c * 16);
                const float* nf = c + 1 < 16 ? fcb + (c + 1) * 16 : fcb + TAPS * 256;
                if (cb + 1 < CiB || c + 1 < 16) {
#pragma unroll
                    for (int f = 0; f < TAPS; ++f) asm volatile("prefetch.global.L1 [%0];" ::"l"(nf + f * 256));
                }
            } else if (c + 1 < 16) {
                // next channel's taps in flight while this channel computes
#pragma unroll
                for (int f = 0; f < TAPS; ++f) gn[f].load(fcb + f * 256 + (c + 1) * 16);
            }
            uint32_t m[NWORD];
            float vv[NWORD];
            if (SPARSE) {
#pragma unroll
                for (int w = 0; w < NWORD; ++w) {
                    vv[w] = (lane + 32 * w < RHW) ? P[qoff[w]] : 0.0f;
                    const bool nz = vv[w] != 0.0f;
                    nzc[w] += nz ? 1u : 0u;
                    m[w] = __ballot_sync(0xffffffffu, nz);
                }
            }
            using JB = JtBlocks<FWD, KK, TH, TW, R, S, STR>;
            if constexpr (SPARSE && JT > 0 && JT < 100) {
#pragma unroll
                for (int w = 0; w < NWORD; ++w) blk_nnz += __popc(m[w]);
            }
            if constexpr (JTP) {
                jt_words<0, NWORD, JB2>(acc, g, vv, m);
            } else {
            if (use_jt) {
                if constexpr (SPARSE && JT > 0 && !FORCE && JB::available) jt_words<0, NWORD, JB>(acc, g, vv, m);
            } else {
            const float* Pw = P + woff;
            float4 cur[NQ], nxt[NQ];
#pragma unroll
            for (int h = 0; h < NQ; ++h) cur[h] = *reinterpret_cast<const float4*>(Pw + 4 * h);
#pragma unroll
            for (int ry = 0; ry < RH; ++ry) {
                if (ry + 1 < RH) {
#pragma unroll
                    for (int h = 0; h < NQ; ++h)
                        nxt[h] = *reinterpret_cast<const float4*>(Pw + (ry + 1) * ROW + 4 * h);
                }
#pragma unroll
                for (int rx = 0; rx < RWW; ++rx) {
                    const int p = ry * RWW + rx;
                    if (!SPARSE || FORCE || ((m[p >> 5] >> (p & 31)) & 1u)) {
                        const float4 q4 = cur[rx >> 2];
                        const float d = (rx & 3) == 0 ? q4.x : (rx & 3) == 1 ? q4.y : (rx & 3) == 2 ? q4.z : q4.w;
                        int ntap = 0;  // folds to a constant per unrolled pixel
#pragma unroll
                        for (int v = 0; v < S; ++v)
#pragma unroll
                            for (int u = 0; u < R; ++u) ntap += AY::target(ry, v) >= 0 && AX::target(rx, u) >= 0;
#pragma unroll
                        for (int v = 0; v < S; ++v) {
                            const int ty = AY::target(ry, v);
                            if (ty < 0) continue;
#pragma unroll
                            for (int u = 0; u < R; ++u) {
                                const int tx = AX::target(rx, u);
                                if (tx < 0) continue;
                                fma_lane<KK, SPC_CONV_FFMA2_MIN>(acc[ty * TW + tx], d, g[v * R + u].v, ntap);
                            }
                        }
                    }
                }
                if (ry + 1 < RH) {
#pragma unroll
                    for (int h = 0; h < NQ; ++h) cur[h] = nxt[h];
                }
            }
            }  // in-line path
            }  // !JTP
            if constexpr (GPF == 1) {
                if (c + 1 < 16) {
#pragma unroll
                    for (int f = 0; f < TAPS; ++f) g[f] = gn[f];
                }
            }
        }
        if constexpr (SPARSE && JT > 0 && JT < 100) {
            if (lane == 0) wnnz[warp] = blk_nnz;
        }
        __syncthreads();
        if constexpr (SPARSE && JT > 0 && JT < 100) {
            int tot = 0;
#pragma unroll
            for (int w = 0; w < NWY * NWX; ++w) tot += wnnz[w];
            use_jt = (long)tot * 100 <= (long)JT * 16 * NWY * NWX * RHW;
        }
    }

    // epilogue: every valid output written exactly once
#pragma unroll
    for (int ty = 0; ty < TH; ++ty) {
        const int y = y0 + ty;
        if (y >= Ho) break;
#pragma unroll
        for (int tx = 0; tx < TW; ++tx) {
            const int x = x0 + tx;
            if (x >= Wo) break;
            FVec<KK> o;
#pragma unroll
            for (int j = 0; j < KK; ++j) {
                if constexpr (JTP) {
                    const float2 q = unpack_f32x2(acc[ty * TW + tx][j / 2]);
                    o.v[j] = j & 1 ? q.y : q.x;
                }
                else o.v[j] = acc[ty * TW + tx][j];
            }
            const size_t off = ((((size_t)i * CoB + k0 / 16) * Ho + y) * Wo + x) * 16 + (k0 % 16);
            if constexpr (EPI) {  // a separate instantiation: the unrolled epilogue costs registers and I-cache
#pragma unroll
                for (int j = 0; j < KK; ++j) o.v[j] = epi.apply(o.v[j], off + j);
            }
            o.store(dst + off);
        }
    }
    if (SPARSE && exec_ctr) {
        uint32_t cnt = 0;
#pragma unroll
        for (int w = 0; w < NWORD; ++w) cnt += nzc[w] * wt[w];
        const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (2 * KK));
    }
    gate.finish(blockIdx.y);
}

#define SPC_TC_TPARAMS                                                                                          \
    bool FWD, int KK, int TH, int TW, int NWY, int NWX, int R, int S, int STR, int GPF, int JT, bool SPARSE, bool EPI
#define SPC_TC_TARGS FWD, KK, TH, TW, NWY, NWX, R, S, STR, GPF, JT, SPARSE, EPI
#define SPC_TC_ARGS                                                                                             \
    DevShape sh, const float* __restrict__ src, const float* __restrict__ filt, float* __restrict__ dst,         \
        unsigned long long* __restrict__ exec_ctr, const int* __restrict__ sel, int want, int group_fastest, Epi epi, \
        Gate gate
template <SPC_TC_TPARAMS>
__global__ void __launch_bounds__(NWY * NWX * 32) tile_conv_kernel(SPC_TC_ARGS) {
    tile_conv_body<SPC_TC_TARGS>(sh, src, filt, dst, exec_ctr, sel, want, group_fastest, epi, gate);
}
// the same kernel under a register cap (tile_maxreg); separate so the
// uncapped instantiations keep ptxas's own allocation
template <SPC_TC_TPARAMS>
__global__ void __launch_bounds__(NWY * NWX * 32) __maxnreg__(tile_maxreg(NWY * NWX * 32, KK, TH, TW, R, STR, JT) > 0 ? tile_maxreg(NWY * NWX * 32, KK, TH, TW, R, STR, JT) : 255)
    tile_conv_kernel_capped(SPC_TC_ARGS) {
    tile_conv_body<SPC_TC_TARGS>(sh, src, filt, dst, exec_ctr, sel, want, group_fastest, epi, gate);
}
template <SPC_TC_TPARAMS>
constexpr auto tile_conv_entry() {
    if constexpr (SPARSE && tile_maxreg(NWY * NWX * 32, KK, TH, TW, R, STR, JT) > 0)
        return tile_conv_kernel_capped<SPC_TC_TARGS>;
    else
        return tile_conv_kernel<SPC_TC_TARGS>;
}
#undef SPC_TC_TPARAMS
#undef SPC_TC_TARGS
#undef SPC_TC_ARGS

// ---------------------------------------------------------------- dispatch
template <bool FWD, int KK, int TH, int TW, int NWY, int NWX, int R, int S, int STR, int GPF = 1, int JT = 0,
          bool WITH_EPI = false>
static cudaError_t launch_cfg(bool sparse, const DevShape& sh, const float* src, const float* filt, float* dst,
                              unsigned long long* exec_ctr, cudaStream_t st, const int* sel = nullptr,
                              int want = 0, const Epi& epi = Epi{}, const Gate& gate = Gate{}) {
    using Gm = ConvGeom<FWD, KK, TH, TW, NWY, NWX, R, S, STR>;
    const int Co = FWD ? sh.K : sh.C;
    const int Ho = FWD ? sh.Hp : sh.H, Wo = FWD ? sh.Wp : sh.W;
    const int tiles_x = (Wo + TW * NWX - 1) / (TW * NWX);
    const int tiles_y = (Ho + TH * NWY - 1) / (TH * NWY);
    dim3 grid(tiles_x * tiles_y * (Co / (32 * KK)), sh.N, 1);
    using KFn = void (*)(DevShape, const float*, const float*, float*, unsigned long long*, const int*, int, int, Epi,
                         Gate);
    KFn kern;
    const bool with_epi = epi.active();
    if (with_epi) {
        if constexpr (WITH_EPI)
            kern = sparse ? tile_conv_entry<FWD, KK, TH, TW, NWY, NWX, R, S, STR, GPF, JT, true, true>()
                          : tile_conv_entry<FWD, KK, TH, TW, NWY, NWX, R, S, STR, GPF, 0, false, true>();
        else
            return cudaErrorInvalidValue;
    } else {
        kern = sparse ? tile_conv_entry<FWD, KK, TH, TW, NWY, NWX, R, S, STR, GPF, JT, true, false>()
                      : tile_conv_entry<FWD, KK, TH, TW, NWY, NWX, R, S, STR, GPF, 0, false, false>();
    }
    static PerDeviceOnce attr_set[2][2];  // per instantiation: [epi][sparse], per device
    int attr_dev = 0;
    if (attr_set[with_epi][sparse].needed(attr_dev)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Gm::SMEM);
        attr_set[with_epi][sparse].done(attr_dev);
    }
    const int Ci = FWD ? sh.C : sh.K;
    const int Hs = FWD ? sh.H : sh.Hp, Ws = FWD ? sh.W : sh.Wp;
    const size_t src_bytes = (size_t)sh.N * Ci * Hs * Ws * sizeof(float);
    // SPC_GROUP_FASTEST=0/1 forces the block order (A/B testing only)
    static const int gf_env = std::getenv("SPC_GROUP_FASTEST") ? std::atoi(std::getenv("SPC_GROUP_FASTEST")) : -1;
    const int group_fastest = gf_env >= 0 ? gf_env : (src_bytes > ((size_t)48 << 20) ? 1 : 0);
    kern<<<grid, Gm::NT, Gm::SMEM, st>>>(sh, src, filt, dst, exec_ctr, sel, want, group_fastest, epi, gate);
    note_launch();
    return cudaGetLastError();
}

// Development entry (include/spconv_b200_dev.h): run one tile configuration
// of the 3x3 s1 kernel directly.  The product build keeps the branch /
// jump-table configurations the tests compare bit for bit (2, 6, 14, 17, 41,
// 42); the whole tuning table (tools/tune.py) needs `make DEV=1`.  Returns
// cudaErrorInvalidValue for an unknown or inapplicable variant.
cudaError_t launch_tile_conv_variant(int variant, bool fwd, bool sparse, const DevShape& sh, const float* src,
                                     const float* filt, float* dst, unsigned long long* exec_ctr, cudaStream_t st) {
    const int Co = fwd ? sh.K : sh.C;
#ifdef SPC_DEV
    if (variant >= 50) {  // 1x1 stride 1 variants
        if (sh.R != 1 || sh.O != 1) return cudaErrorInvalidValue;
#define SPC_V1(ID, KK, TH, TW, NWY, NWX)                                                                        \
    case ID:                                                                                                    \
        if (Co % (32 * KK)) return cudaErrorInvalidValue;                                                       \
        return fwd ? launch_cfg<true, KK, TH, TW, NWY, NWX, 1, 1, 1, 1, 0>(sparse, sh, src, filt, dst, exec_ctr, st) \
                   : launch_cfg<false, KK, TH, TW, NWY, NWX, 1, 1, 1, 1, 0>(sparse, sh, src, filt, dst, exec_ctr, st);
        switch (variant) {
            SPC_V1(50, 4, 4, 8, 2, 1)
            SPC_V1(51, 2, 4, 8, 2, 1)
            SPC_V1(52, 8, 4, 4, 2, 1)
            SPC_V1(53, 8, 2, 8, 2, 1)
            SPC_V1(54, 8, 2, 4, 2, 2)
            SPC_V1(55, 4, 7, 4, 1, 1)
            SPC_V1(56, 8, 7, 2, 1, 1)
            SPC_V1(57, 8, 4, 4, 1, 1)
            SPC_V1(58, 4, 4, 8, 1, 1)
            SPC_V1(59, 8, 7, 2, 2, 1)
            SPC_V1(60, 16, 2, 4, 1, 1)
            SPC_V1(61, 16, 1, 8, 1, 1)
            SPC_V1(62, 16, 2, 4, 2, 1)
            SPC_V1(63, 16, 2, 4, 4, 1)
            SPC_V1(64, 16, 1, 8, 4, 1)
            SPC_V1(65, 8, 2, 8, 1, 1)
            SPC_V1(66, 8, 4, 4, 4, 1)
            SPC_V1(67, 16, 1, 7, 2, 1)
            default: return cudaErrorInvalidValue;
        }
#undef SPC_V1
    }
#endif
    if (sh.R != 3 || sh.O != 1) return cudaErrorInvalidValue;
#define SPC_V(ID, KK, TH, TW, NWY, NWX, GPF) SPC_VJ(ID, KK, TH, TW, NWY, NWX, GPF, 0)
#define SPC_VJ(ID, KK, TH, TW, NWY, NWX, GPF, JT)                                                               \
    case ID:                                                                                                    \
        if (Co % (32 * KK)) return cudaErrorInvalidValue;                                                       \
        return fwd ? launch_cfg<true, KK, TH, TW, NWY, NWX, 3, 3, 1, GPF, JT>(sparse, sh, src, filt, dst, exec_ctr, st) \
                   : launch_cfg<false, KK, TH, TW, NWY, NWX, 3, 3, 1, GPF, JT>(sparse, sh, src, filt, dst, exec_ctr, st);
    switch (variant) {
        SPC_V(2, 4, 4, 8, 2, 1, 1)
        SPC_V(6, 2, 4, 8, 2, 2, 1)
        SPC_VJ(14, 2, 4, 8, 2, 2, 1, 100)
        SPC_VJ(17, 4, 4, 8, 2, 1, 1, 100)
        SPC_VJ(41, 4, 4, 8, 1, 1, 1, 100)
        SPC_V(42, 4, 7, 4, 1, 1, 1)
#ifdef SPC_DEV
        SPC_V(0, 4, 4, 4, 2, 2, 1)
        SPC_V(1, 4, 4, 4, 2, 2, 0)
        SPC_V(3, 4, 4, 8, 2, 1, 0)
        SPC_V(4, 4, 8, 4, 2, 1, 0)
        SPC_V(5, 2, 8, 8, 2, 1, 0)
        SPC_V(7, 8, 4, 4, 2, 1, 0)
        SPC_V(8, 8, 2, 4, 2, 2, 0)
        SPC_V(9, 8, 2, 4, 2, 2, 1)
        SPC_V(10, 4, 4, 4, 4, 1, 1)
        SPC_V(11, 4, 4, 4, 1, 4, 1)
        SPC_V(12, 2, 4, 8, 4, 1, 1)
        SPC_V(13, 4, 2, 8, 4, 1, 1)
        SPC_VJ(15, 2, 4, 8, 4, 1, 1, 100)
        SPC_VJ(16, 4, 4, 4, 2, 2, 1, 100)
        SPC_VJ(18, 4, 4, 8, 2, 1, 0, 100)
        SPC_VJ(19, 2, 4, 8, 2, 2, 0, 100)
        SPC_VJ(20, 2, 4, 8, 2, 2, 1, 15)
        SPC_VJ(21, 4, 4, 4, 2, 2, 1, 15)
        SPC_VJ(22, 4, 4, 8, 2, 1, 1, 15)
        SPC_VJ(23, 4, 4, 4, 2, 2, 1, 30)
        SPC_VJ(24, 4, 4, 8, 2, 1, 1, 30)
        SPC_VJ(25, 2, 4, 8, 2, 2, 1, 30)
        SPC_V(26, 2, 4, 7, 2, 2, 1)
        SPC_V(27, 2, 7, 4, 2, 2, 1)
        SPC_V(28, 2, 7, 7, 2, 1, 1)
        SPC_V(29, 4, 4, 7, 2, 1, 1)
        SPC_V(30, 4, 7, 4, 2, 1, 1)
        SPC_V(31, 2, 4, 7, 4, 1, 1)
        SPC_V(32, 4, 2, 7, 2, 2, 1)
        SPC_V(33, 2, 7, 7, 2, 2, 1)
        SPC_V(34, 4, 4, 7, 2, 2, 1)
        SPC_V(35, 4, 2, 7, 4, 1, 1)
        SPC_VJ(36, 4, 7, 4, 2, 1, 1, 100)
        SPC_VJ(37, 4, 4, 7, 2, 1, 1, 100)
        SPC_V(38, 4, 7, 4, 2, 1, 0)
        SPC_V(39, 4, 4, 7, 2, 1, 0)
        SPC_VJ(40, 4, 4, 8, 2, 2, 0, 100)
        SPC_V(43, 4, 7, 4, 4, 1, 0)
#endif
        default: return cudaErrorInvalidValue;
    }
#undef SPC_V
#undef SPC_VJ
}

// Nonzero density of the swept tensor from a strided sample (i.i.d. or
// spatially correlated data alike: 148*256 threads x 16 float4 spread over
// the whole tensor).  sel = 1 when density <= pct% (the jump-table kernel
// wins), else 0.
__global__ void __launch_bounds__(256) density_probe_kernel(const float* __restrict__ t, size_t n, int pct,
                                                            int* __restrict__ sel, Gate gate) {
    gate.wait_input(0);  // gated launches sample the first input chunk once it has landed
    __shared__ unsigned long long cnt[2];
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    __syncthreads();
    const size_t n4 = n / 4;
    const size_t nthreads = (size_t)gridDim.x * blockDim.x;
    const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    const size_t stride = n4 / (nthreads * 16) > 0 ? n4 / (nthreads * 16) : 1;
    unsigned nz = 0, tot = 0;
    // all 16 loads in flight at once (one DRAM round trip, not 16)
    float4 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        const size_t e = (tid + (size_t)i * nthreads) * stride;
        v[i] = e < n4 ? __ldg(reinterpret_cast<const float4*>(t) + e) : make_float4(0.f, 0.f, 0.f, 0.f);
        tot += e < n4 ? 4u : 0u;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) nz += (v[i].x != 0.0f) + (v[i].y != 0.0f) + (v[i].z != 0.0f) + (v[i].w != 0.0f);
    nz = __reduce_add_sync(0xffffffffu, nz);
    tot = __reduce_add_sync(0xffffffffu, tot);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&cnt[0], (unsigned long long)nz);
        atomicAdd(&cnt[1], (unsigned long long)tot);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // one CTA's sample decides for the whole launch when gridDim.x == 1
        sel[blockIdx.x] = cnt[0] * 100 <= (unsigned long long)pct * cnt[1] ? 1 : 0;
    }
}

void launch_density_probe(const float* t, size_t n, int pct, int* sel, cudaStream_t st, const Gate& gate) {
    // SPC_JT_PCT overrides the jump-table density threshold (0 = never, 100 = always)
    static const int override_pct = std::getenv("SPC_JT_PCT") ? std::atoi(std::getenv("SPC_JT_PCT")) : -1;
    if (override_pct >= 0) pct = override_pct;
    Gate g = gate;
    g.done = nullptr;  // the probe only waits; it never completes a chunk
    density_probe_kernel<<<1, 256, 0, st>>>(t, n, pct, sel, g);
    note_launch();
}

bool tile_conv_supported(bool fwd, const DevShape& sh, int V) {
    if (V != 16) return false;
    const int Co = fwd ? sh.K : sh.C;
    if (Co % 64) return false;
    if (sh.R != sh.S || sh.O != sh.P) return false;
    if (sh.padW != (sh.R - 1) / 2 || sh.padH != (sh.S - 1) / 2) return false;
    if (sh.R == 3 && (sh.O == 1 || sh.O == 2)) return true;
    if (sh.R == 1 && (sh.O == 1 || sh.O == 2)) return true;
    return false;
}

#ifndef SPC_CONV_CFG
#define SPC_CONV_CFG 0
#endif

cudaError_t launch_tile_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                             float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi,
                             const int* xsel, int xwant, const Gate& gate) {
    const int Co = fwd ? sh.K : sh.C;
    const bool kk4 = Co % 128 == 0;
#define SPC_L(F, KK, TH, TW, NWY, NWX, R, STR) \
    return launch_cfg<F, KK, TH, TW, NWY, NWX, R, R, STR, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, xsel, xwant, epi, gate)
    if (sh.R == 3 && sh.O == 1) {
        // tile choices from tools/tune.py sweeps over the VGG16 layers
        // (profiles/r01_tune.md): 7-wide tiles divide every VGG/ResNet
        // resolution; KK=4 branches for sparse, the KK=4 4x8 one-warp jump table for
        // density <= 28% (measured crossover near s = 0.7 for the capped one-warp
        // jump table: s = 0.75 3-9% ahead, s = 0.7 even), KK=2 7x7 for dense mode.
        if (sparse && kk4 && xsel == nullptr) {
            const int Ci = fwd ? sh.C : sh.K;
            const int Hs = fwd ? sh.H : sh.Hp, Ws = fwd ? sh.W : sh.Wp;
            int* sel = stream_flags(st) ? stream_flags(st) + FLAG_CONV_SEL : nullptr;
            cudaError_t e = sel ? cudaSuccess : cudaErrorMemoryAllocation;
            if (e != cudaSuccess) return e;
            // gated (host-buffer) launches sample only the first input chunk
            const size_t per_img = (size_t)Ci * Hs * Ws;
            launch_density_probe(src, per_img * (gate.in_ready ? (size_t)gate.ipc : (size_t)sh.N), 28, sel, st, gate);
            e = fwd ? launch_cfg<true, 4, 7, 4, 1, 1, 3, 3, 1, 1, 0, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 0, epi, gate)
                    : launch_cfg<false, 4, 7, 4, 1, 1, 3, 3, 1, 1, 0, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 0, epi, gate);
            if (e == cudaSuccess)
                e = fwd ? launch_cfg<true, 4, 4, 8, 1, 1, 3, 3, 1, 1, 100, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 1, epi, gate)
                        : launch_cfg<false, 4, 4, 8, 1, 1, 3, 3, 1, 1, 100, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 1, epi, gate);
            return e;
        }
        if (sparse && xsel == nullptr) {
            // 64-channel multiples: the KK=2 branch kernel, or below 21% density
            // its jump-table twin on the same 8x16 CTA tile (capped at 128
            // registers: 4 CTAs per SM; conv1_2 s=0.9 87 vs 64 TF/s, s=0.8 64 vs
            // 62.5, s=0.6 44 vs 59)
            const int Ci = fwd ? sh.C : sh.K;
            const int Hs = fwd ? sh.H : sh.Hp, Ws = fwd ? sh.W : sh.Wp;
            int* sel = stream_flags(st) ? stream_flags(st) + FLAG_CONV_SEL : nullptr;
            cudaError_t e = sel ? cudaSuccess : cudaErrorMemoryAllocation;
            if (e != cudaSuccess) return e;
            const size_t per_img = (size_t)Ci * Hs * Ws;
            launch_density_probe(src, per_img * (gate.in_ready ? (size_t)gate.ipc : (size_t)sh.N), 21, sel, st, gate);
            e = fwd ? launch_cfg<true, 2, 4, 8, 2, 2, 3, 3, 1, 1, 0, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 0, epi, gate)
                    : launch_cfg<false, 2, 4, 8, 2, 2, 3, 3, 1, 1, 0, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 0, epi, gate);
            if (e == cudaSuccess)
                e = fwd ? launch_cfg<true, 2, 4, 8, 2, 2, 3, 3, 1, 1, 100, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 1, epi, gate)
                        : launch_cfg<false, 2, 4, 8, 2, 2, 3, 3, 1, 1, 100, true>(true, sh, src, filt, dst, exec_ctr, st, sel, 1, epi, gate);
            return e;
        }
        if (sparse) {
            if (fwd) SPC_L(true, 2, 4, 8, 2, 2, 3, 1);
            SPC_L(false, 2, 4, 8, 2, 2, 3, 1);
        }
        if (fwd) SPC_L(true, 2, 7, 7, 2, 1, 3, 1);
        SPC_L(false, 2, 7, 7, 2, 1, 3, 1);
    }
    if (sh.R == 3) {  // stride 2
        if (fwd) {
            if (sparse && xsel == nullptr) {
                // a stride-2 source pixel feeds ~2.25 taps: per-pixel branches cost more
                // than the FMAs they skip, so finite filters run the counted-dense
                // kernel (JT = 200); a filter with Inf/NaN keeps the per-pixel skip
                int* finite = stream_flags(st) ? stream_flags(st) + FLAG_CONV_FINITE : nullptr;
                cudaError_t e = finite ? cudaSuccess : cudaErrorMemoryAllocation;
                if (e != cudaSuccess) return e;
                launch_finite_all(filt, (size_t)sh.K * sh.C * 9, finite, st);
                // SPC_FORCE_SKIP=1 runs the per-pixel-skip kernel for finite filters
                // too (A/B evidence for the counted-dense choice, tools/skip_evidence.py)
                static const bool force_skip = std::getenv("SPC_FORCE_SKIP") && std::atoi(std::getenv("SPC_FORCE_SKIP")) == 1;
                if (force_skip) cudaMemsetAsync(finite, 0, sizeof(int), st);
                if (kk4) {
                    e = launch_cfg<true, 4, 4, 4, 2, 1, 3, 3, 2, 1, 200, true>(true, sh, src, filt, dst, exec_ctr, st,
                                                                              finite, 1, epi, gate);
                    if (e == cudaSuccess)
                        e = launch_cfg<true, 4, 4, 4, 2, 1, 3, 3, 2, 1, 0, true>(true, sh, src, filt, dst, exec_ctr,
                                                                                st, finite, 0, epi, gate);
                } else {
                    e = launch_cfg<true, 2, 4, 4, 2, 1, 3, 3, 2, 1, 200, true>(true, sh, src, filt, dst, exec_ctr, st,
                                                                              finite, 1, epi, gate);
                    if (e == cudaSuccess)
                        e = launch_cfg<true, 2, 4, 4, 2, 1, 3, 3, 2, 1, 0, true>(true, sh, src, filt, dst, exec_ctr,
                                                                                st, finite, 0, epi, gate);
                }
                return e;
            }
            if (kk4) SPC_L(true, 4, 4, 4, 2, 1, 3, 2);
            SPC_L(true, 2, 4, 4, 2, 1, 3, 2);
        }
        if (kk4) SPC_L(false, 4, 4, 8, 2, 1, 3, 2);
        SPC_L(false, 2, 4, 8, 2, 1, 3, 2);
    }
    if (sh.O == 1) {  // 1x1
        if (fwd) {
            if (kk4) SPC_L(true, 4, 4, 8, 2, 1, 1, 1);
            SPC_L(true, 2, 4, 8, 2, 1, 1, 1);
        }
        if (kk4) SPC_L(false, 4, 4, 8, 2, 1, 1, 1);
        SPC_L(false, 2, 4, 8, 2, 1, 1, 1);
    }
    // 1x1 stride 2
    if (fwd) {
        if (kk4) SPC_L(true, 4, 4, 8, 2, 1, 1, 2);
        SPC_L(true, 2, 4, 8, 2, 1, 1, 2);
    }
    if (kk4) SPC_L(false, 4, 4, 8, 2, 1, 1, 2);
    SPC_L(false, 2, 4, 8, 2, 1, 1, 2);
#undef SPC_L
}

// FFMA tile kernel gated on a device word (*sel == want), used behind the
// tensor-core variant for sources / filters with Inf or NaN (tc_conv.cu).
cudaError_t launch_tile_conv_when(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                                  float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi,
                                  const int* sel, int want) {
    const bool kk4 = (fwd ? sh.K : sh.C) % 128 == 0;
    if (sh.O == 2) {  // the stride-2 tile configurations of launch_tile_conv
        if (sh.R == 3) {
            if (fwd)
                return kk4 ? launch_cfg<true, 4, 4, 4, 2, 1, 3, 3, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr,
                                                                                 st, sel, want, epi, Gate{})
                           : launch_cfg<true, 2, 4, 4, 2, 1, 3, 3, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr,
                                                                                 st, sel, want, epi, Gate{});
            return kk4 ? launch_cfg<false, 4, 4, 8, 2, 1, 3, 3, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                              sel, want, epi, Gate{})
                       : launch_cfg<false, 2, 4, 8, 2, 1, 3, 3, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                              sel, want, epi, Gate{});
        }
        if (fwd)
            return kk4 ? launch_cfg<true, 4, 4, 8, 2, 1, 1, 1, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                             sel, want, epi, Gate{})
                       : launch_cfg<true, 2, 4, 8, 2, 1, 1, 1, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                             sel, want, epi, Gate{});
        return kk4 ? launch_cfg<false, 4, 4, 8, 2, 1, 1, 1, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, sel,
                                                                          want, epi, Gate{})
                   : launch_cfg<false, 2, 4, 8, 2, 1, 1, 1, 2, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, sel,
                                                                          want, epi, Gate{});
    }
    if (sh.R == 3) {
        if (kk4)
            return fwd ? launch_cfg<true, 4, 7, 4, 1, 1, 3, 3, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                              sel, want, epi, Gate{})
                       : launch_cfg<false, 4, 7, 4, 1, 1, 3, 3, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr,
                                                                               st, sel, want, epi, Gate{});
        return fwd ? launch_cfg<true, 2, 4, 8, 2, 2, 3, 3, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, sel,
                                                                          want, epi, Gate{})
                   : launch_cfg<false, 2, 4, 8, 2, 2, 3, 3, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                           sel, want, epi, Gate{});
    }
    if (kk4)
        return fwd ? launch_cfg<true, 4, 4, 8, 2, 1, 1, 1, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, sel,
                                                                          want, epi, Gate{})
                   : launch_cfg<false, 4, 4, 8, 2, 1, 1, 1, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st,
                                                                           sel, want, epi, Gate{});
    return fwd ? launch_cfg<true, 2, 4, 8, 2, 1, 1, 1, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, sel,
                                                                      want, epi, Gate{})
               : launch_cfg<false, 2, 4, 8, 2, 1, 1, 1, 1, 1, 0, true>(sparse, sh, src, filt, dst, exec_ctr, st, sel,
                                                                       want, epi, Gate{});
}

}  // namespace spc
