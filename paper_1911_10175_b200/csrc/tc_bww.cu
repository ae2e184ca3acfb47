// tc_bww.cu -- BWW on the 5th-generation tensor cores (tcgen05, TMEM, TMA),
// 3xTF32 split arithmetic (the same split as tc_conv.cu, whose header states
// the error bound and the non-finite fallback): the optional tensor-core
// variant of SURVEY.md 8(f)4, selected with spc_set_math(SPC_MATH_TF32X3).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_conv.h"
#include "dispatch.h"
#include "pw_bww.h"
#include "tile_bww.h"

namespace spc {
namespace {
using namespace tc;

// ================================================================ BWW
// dG[k, c, v, u] = sum_{i, y', x'} dY[i, k, y', x'] * D[i, c, y'+v-padH, x'+u-padW]
// (P/src/kernel_impl.hpp:209-336, P/src/kernels.cpp:238-302), as one GEMM per
// tap: M = 128 output-gradient channels k, N = BN input channels c, reduction
// over (image, output pixel).  The prep kernels rewrite both operands (hi =
// raw, lo = split remainder) pixel-major, [N/16][H][W][C][16 images] -- the
// reference's ActCHWNn with the channel loop moved inside the pixel, so one
// pixel of one 16-image block is C x 64 contiguous bytes: a stage = one
// pixel, the A tile {16 images, 128 k} / B tile {16 images, BN c} are single
// contiguous TMA boxes that land in shared memory as K-major SWIZZLE_64B
// operands exactly like the FWD tiles.  Pixels outside the image are TMA
// zero-fill (the padding); ragged image lanes are zeros.
// A CTA owns (tap, k tile, c tile, reduction split); partial tiles go to
// scratch and a fixed-order reduction writes FilterKCRSblk (deterministic).
struct TcBwwGeo {
    int Hp, Wp;      // output (dY) extent
    int R, S, padW, padH;
    int K, C;
    int ktiles, ctiles, splits;
    int cw, tpc, tgroups;  // channels per tap in a c tile, taps stacked along N (BN = tpc * cw), tap groups
    long stages;     // ceil(N / 16) * Hp * Wp
    int str;         // stride (source pixel = str * output pixel + tap - pad)
    int seg;
};

// PX = output pixels per stage (2 for small N tiles: 1x1, one tap, stride 1 --
// twice the MMAs per barrier round trip, the small-N MMAs being issue-bound;
// the 2 pixels are consecutive along x, one TMA box of {16, channels, 2}).
template <int BN, int PX>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_bww_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                  const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                  TcBwwGeo g, float* __restrict__ partial, const int* __restrict__ nonfinite,
                  const unsigned long long* __restrict__ cnt_tmp, unsigned long long* __restrict__ exec_ctr) {
    if (__ldg(nonfinite) != 0) return;
    constexpr uint32_t A_BYTES = PX * TC_BM * 64;  // PX pixels x 128 k-rows x 64 B (16 images)
    constexpr uint32_t B_BYTES = PX * BN * 64;     // PX pixels x BN c-rows x 64 B
    constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
    constexpr int ST = PX == 1 ? TC_ST : (int)((200 * 1024) / STAGE);
    constexpr int HALF = BN / 2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // blockIdx.x = ((tap * ktiles + kt) * ctiles + ct), blockIdx.y = split
    int b = blockIdx.x;
    const int ct = b % g.ctiles;
    b /= g.ctiles;
    const int kt = b % g.ktiles;
    const int tg = b / g.ktiles;  // taps tg*tpc .. +tpc-1 stacked along N
    const int split = blockIdx.y;
    const long t0 = g.stages * split / g.splits, t1 = g.stages * (split + 1) / g.splits;
    const int niter = (int)(t1 - t0);
    const int D = g.seg;
    const int nseg = (niter + D - 1) / D;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (ST + s); };
    auto tfull_bar = [&](int bb) { return bar0 + 8u * (2 * ST + bb); };
    auto tempty_bar = [&](int bb) { return bar0 + 8u * (2 * ST + 2 + bb); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int bb = 0; bb < 2; ++bb) {
            mbar_init(tfull_bar(bb), 1);
            mbar_init(tempty_bar(bb), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (blockIdx.x == 0 && blockIdx.y == 0 && cnt_tmp && exec_ctr) atomicAdd(exec_ctr, *cnt_tmp);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(tmem_cols(2 * BN))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0 && niter > 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
            long t = t0;
            const long per_ib = (long)g.Hp * ((g.Wp + PX - 1) / PX);
            int ib = (int)(t / per_ib);
            int rem = (int)(t - (long)ib * per_ib);
            const int xw = (g.Wp + PX - 1) / PX;  // stages per output row
            int yp = rem / xw, xp = (rem - yp * xw) * PX;
            for (int it = 0; it < niter; ++it) {
                const int s = it % ST;
                if (it >= ST) mbar_wait(empty_bar(s), ((it / ST) - 1) & 1);
                const uint32_t st = sbase + s * STAGE;
                mbar_expect_tx(full_bar(s), STAGE);
                tma_load_5d(st, &map_ahi, full_bar(s), 0, kt * TC_BM, xp, yp, ib);
                tma_load_5d(st + A_BYTES, &map_alo, full_bar(s), 0, kt * TC_BM, xp, yp, ib);
                for (int j = 0; j < g.tpc; ++j) {
                    const int tap = tg * g.tpc + j;
                    const int v = tap / g.R, u = tap - v * g.R;
                    // a missing tap of the last group loads an all-out-of-bounds box (zeros)
                    const int sx = tap < g.R * g.S ? g.str * xp + u - g.padW : -(1 << 20);
                    const int sy = g.str * yp + v - g.padH;
                    const uint32_t boff = (uint32_t)(j * g.cw * 64);
                    tma_load_5d(st + 2 * A_BYTES + boff, &map_bhi, full_bar(s), 0, ct * g.cw, sx, sy, ib);
                    tma_load_5d(st + 2 * A_BYTES + B_BYTES + boff, &map_blo, full_bar(s), 0, ct * g.cw, sx, sy, ib);
                }
                if ((xp += PX) >= g.Wp) {
                    xp = 0;
                    if (++yp == g.Hp) {
                        yp = 0;
                        ++ib;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tf32_idesc<BN>();
            for (int it = 0; it < niter; ++it) {
                const int seg = it / D, buf = seg & 1;
                const bool first = it - seg * D == 0;
                if (first && seg >= 2) mbar_wait(tempty_bar(buf), ((seg >> 1) - 1) & 1);
                const int s = it % ST;
                mbar_wait(full_bar(s), (it / ST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = sbase + s * STAGE;
                const uint32_t tm = tmem + buf * BN;
#pragma unroll
                for (int k = 0; k < 2 * PX; ++k) {  // per pixel: images 0-7, 8-15 (32 bytes each)
                    const uint32_t ao = (k >> 1) * (TC_BM * 64) + 32 * (k & 1);
                    const uint32_t bo = (k >> 1) * (BN * 64) + 32 * (k & 1);
                    const uint64_t ahi = sw64_desc(st + ao);
                    const uint64_t alo = sw64_desc(st + A_BYTES + ao);
                    const uint64_t bhi = sw64_desc(st + 2 * A_BYTES + bo);
                    const uint64_t blo = sw64_desc(st + 2 * A_BYTES + B_BYTES + bo);
                    umma_tf32(tm, alo, bhi, idesc, (first && k == 0) ? 0u : 1u);
                    umma_tf32(tm, ahi, blo, idesc, 1u);
                    umma_tf32(tm, ahi, bhi, idesc, 1u);
                }
                umma_commit(empty_bar(s));
                if (it - seg * D == D - 1 || it == niter - 1) umma_commit(tfull_bar(buf));
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int krow = kt * TC_BM + q * 32 + lane;
        float acc[HALF];
#pragma unroll
        for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        for (int seg = 0; seg < nseg; ++seg) {
            const int buf = seg & 1;
            mbar_wait_sleep(tfull_bar(buf), (seg >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int j = 0; j < HALF / 16; ++j) {
                float vv[16];
                tmem_ld16(tmem + lane_off + buf * BN + h * HALF + 16 * j, vv);
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[16 * j + e] += vv[e];
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(tempty_bar(buf));
        }
        // partial[split][tap][k][c] (k < K, c < C, existing taps only); column
        // n of the tile = (tap tg*tpc + n / cw, channel ct*cw + n % cw)
        if (krow < g.K) {
#pragma unroll
            for (int j = 0; j < HALF; j += 4) {
                const int n = h * HALF + j;
                const int tj = n / g.cw, c = ct * g.cw + (n - tj * g.cw);
                const int tap = tg * g.tpc + tj;
                if (tap < g.R * g.S && c < g.C) {
                    float* o = partial + (((size_t)split * g.R * g.S + tap) * g.K + krow) * g.C + c;
                    *reinterpret_cast<float4*>(o) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * BN)) : "memory");
    }
}

// tc_bww_pair_kernel: the BWW GEMM on a CTA pair (cluster of 2, M = 256 = two
// k tiles): each CTA loads its own dY k tile and HALF of the 256 D channel rows
// of the stage; the leader issues one cta_group::2 MMA (the FWD pair kernel's
// protocol).  Single tap per CTA (tpc = 1), BN = 256, K a multiple of 256.
// blockIdx.x = ((tap group * ctiles + ct) * ktiles + kt): a cluster = kt, kt+1.
template <int ST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_bww_pair_kernel(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
                       const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                       TcBwwGeo g, float* __restrict__ partial, const int* __restrict__ nonfinite,
                       const unsigned long long* __restrict__ cnt_tmp, unsigned long long* __restrict__ exec_ctr) {
    if (__ldg(nonfinite) != 0) return;
    constexpr int BN = 256;
    constexpr uint32_t A_BYTES = TC_BM * 64;
    constexpr uint32_t BH_BYTES = (BN / 2) * 64;
    constexpr uint32_t STAGE = 2 * A_BYTES + 2 * BH_BYTES;
    constexpr int HALF = BN / 2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 4);
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int b = blockIdx.x;
    const int kt = b % g.ktiles;
    b /= g.ktiles;
    const int ct = b % g.ctiles;
    const int tap = b / g.ctiles;
    const int v = tap / g.R, u = tap - v * g.R;
    const int split = blockIdx.y;
    const long t0 = g.stages * split / g.splits, t1 = g.stages * (split + 1) / g.splits;
    const int niter = (int)(t1 - t0);
    const int D = g.seg;
    const int nseg = (niter + D - 1) / D;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (ST + s); };
    auto tfull_bar = [&](int bb) { return bar0 + 8u * (2 * ST + bb); };
    auto tempty_bar = [&](int bb) { return bar0 + 8u * (2 * ST + 2 + bb); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int bb = 0; bb < 2; ++bb) {
            mbar_init(tfull_bar(bb), 1);
            mbar_init(tempty_bar(bb), 16);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (blockIdx.x == 0 && blockIdx.y == 0 && cnt_tmp && exec_ctr) atomicAdd(exec_ctr, *cnt_tmp);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(tmem_cols(2 * BN))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0 && niter > 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
            long t = t0;
            const long per_ib = (long)g.Hp * g.Wp;
            int ib = (int)(t / per_ib);
            int rem = (int)(t - (long)ib * per_ib);
            int yp = rem / g.Wp, xp = rem - yp * g.Wp;
            for (int it = 0; it < niter; ++it) {
                const int s = it % ST;
                if (it >= ST) mbar_wait(empty_bar(s), ((it / ST) - 1) & 1);
                const uint32_t st = sbase + s * STAGE;
                if (rank == 0) mbar_expect_tx(full_bar(s), 2 * STAGE);
                tma_load_5d_pair(st, &map_ahi, full_bar(s), 0, kt * TC_BM, xp, yp, ib);
                tma_load_5d_pair(st + A_BYTES, &map_alo, full_bar(s), 0, kt * TC_BM, xp, yp, ib);
                const int sx = g.str * xp + u - g.padW, sy = g.str * yp + v - g.padH;
                const int c0 = ct * BN + (int)rank * HALF;
                tma_load_5d_pair(st + 2 * A_BYTES, &map_bhi, full_bar(s), 0, c0, sx, sy, ib);
                tma_load_5d_pair(st + 2 * A_BYTES + BH_BYTES, &map_blo, full_bar(s), 0, c0, sx, sy, ib);
                if (++xp == g.Wp) {
                    xp = 0;
                    if (++yp == g.Hp) {
                        yp = 0;
                        ++ib;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)(256 >> 4) << 24);
            for (int it = 0; it < niter; ++it) {
                const int seg = it / D, buf = seg & 1;
                const bool first = it - seg * D == 0;
                if (first && seg >= 2) mbar_wait(tempty_bar(buf), ((seg >> 1) - 1) & 1);
                const int s = it % ST;
                mbar_wait(full_bar(s), (it / ST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = sbase + s * STAGE;
                const uint32_t tm = tmem + buf * BN;
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const uint64_t ahi = sw64_desc(st + 32 * k);
                    const uint64_t alo = sw64_desc(st + A_BYTES + 32 * k);
                    const uint64_t bhi = sw64_desc(st + 2 * A_BYTES + 32 * k);
                    const uint64_t blo = sw64_desc(st + 2 * A_BYTES + BH_BYTES + 32 * k);
                    umma_tf32_pair(tm, alo, bhi, idesc, (first && k == 0) ? 0u : 1u);
                    umma_tf32_pair(tm, ahi, blo, idesc, 1u);
                    umma_tf32_pair(tm, ahi, bhi, idesc, 1u);
                }
                umma_commit_pair(empty_bar(s));
                if (it - seg * D == D - 1 || it == niter - 1) umma_commit_pair(tfull_bar(buf));
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int krow = kt * TC_BM + q * 32 + lane;
        float acc[HALF];
#pragma unroll
        for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        for (int seg = 0; seg < nseg; ++seg) {
            const int buf = seg & 1;
            mbar_wait_sleep(tfull_bar(buf), (seg >> 1) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
            for (int j = 0; j < HALF / 16; ++j) {
                float vv[16];
                tmem_ld16(tmem + lane_off + buf * BN + h * HALF + 16 * j, vv);
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[16 * j + e] += vv[e];
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 map_to_rank0(tempty_bar(buf)))
                             : "memory");
        }
        if (krow < g.K) {
#pragma unroll
            for (int j = 0; j < HALF; j += 4) {
                const int c = ct * BN + h * HALF + j;
                if (c < g.C) {
                    float* o = partial + (((size_t)split * g.R * g.S + tap) * g.K + krow) * g.C + c;
                    *reinterpret_cast<float4*>(o) = make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * BN))
                     : "memory");
    }
}

// Fixed-order sum over splits -> FilterKCRSblk (K, C) (P/include/spconv/tensor.hpp:112-119).
__global__ void tc_bww_reduce_kernel(const float* __restrict__ partial, float* __restrict__ dst, int splits, int K,
                                     int C, int R, int S, const int* __restrict__ nonfinite) {
    if (__ldg(nonfinite) != 0) return;
    const size_t n = (size_t)R * S * K * C;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int p = 0; p < splits; ++p) s += partial[(size_t)p * n + e];
        const int c = (int)(e % C);
        const int k = (int)((e / C) % K);
        const int tap = (int)(e / ((size_t)C * K));
        const int v = tap / R, u = tap - v * R;
        dst[filter_index(C, S, R, 16, k, c, u, v)] = s;
    }
}

// ActNCHWc [N][C/16][H][W][16] (FROM_CHWNN = false) or ActCHWNn
// [N/16][C][H][W][16 images] (true) -> pixel-major [N/16][H][W][C][16 images]
// hi (raw) + lo copies, ragged image lanes zero (the lane rule of
// pack_act_chwnn, P/src/tensor.cpp:94-108).  A CTA moves one (16-image block,
// 16-channel block, 16-pixel run) through a shared 16 x 16 x 16 tile: 1 KB
// contiguous reads (16 px x 16 ch of one image, or 16 px x 16 images of one
// channel) and 1 KB contiguous writes (16 ch x 16 images of one pixel).
// Fallback selector of the non-finite path: 0 = the tensor-core result
// stands, 1 = FFMA tile kernel (checked tensor finite), 2 = generic kernel.
__global__ void tc_select_kernel(const int* __restrict__ nonfinite, const int* __restrict__ chk_finite,
                                 int* __restrict__ sel) {
    *sel = *nonfinite == 0 ? 0 : (*chk_finite ? 1 : 2);
}

// Flags non-finite values.
template <bool FROM_CHWNN>
__global__ void __launch_bounds__(256) tc_to_hwcn_split_kernel(const float* __restrict__ in, float* __restrict__ hi,
                                                               float* __restrict__ lo, int N, int C, int HW,
                                                               int* __restrict__ nonfinite) {
    __shared__ float t[16 * 16 * 17];  // [pixel][channel][image], rows padded to 17
    const int pblocks = (HW + 15) / 16;
    const int pb = blockIdx.x % pblocks;
    const int cb = (blockIdx.x / pblocks) % (C / 16);
    const int ib = blockIdx.x / (pblocks * (C / 16));
    const int tid = threadIdx.x;
    const int p0 = pb * 16;
    int bad = 0;
    // reads: 1024 float4 = 16 runs of 1 KB (one per channel, or per image)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int q = tid + 256 * k;
        const int j = q >> 6, px = (q & 63) >> 2, l4 = (q & 3) * 4;
        float4 x = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (p0 + px < HW) {
            if (FROM_CHWNN) {  // j = channel, l4 = first of 4 image lanes
                x = __ldg(reinterpret_cast<const float4*>(in + (((size_t)ib * C + cb * 16 + j) * HW + p0 + px) * 16 + l4));
            } else if (ib * 16 + j < N) {  // j = image lane, l4 = first of 4 channels
                x = __ldg(reinterpret_cast<const float4*>(
                    in + (((size_t)(ib * 16 + j) * (C / 16) + cb) * HW + p0 + px) * 16 + l4));
            }
        }
        bad |= !isfinite(x.x) | !isfinite(x.y) | !isfinite(x.z) | !isfinite(x.w);
        const float v[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            if (FROM_CHWNN) t[(px * 16 + j) * 17 + l4 + e] = v[e];
            else t[(px * 16 + l4 + e) * 17 + j] = v[e];
        }
    }
    __syncthreads();
    // writes: pixel p0 + p = channels cb*16 .. +15 x 16 images (1 KB contiguous), float4 stores
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int q = tid + 256 * k;
        const int p = q >> 6, c = (q & 63) >> 2, i4 = (q & 3) * 4;
        if (p0 + p < HW) {
            const float* r = t + (p * 16 + c) * 17 + i4;
            const float4 x = make_float4(r[0], r[1], r[2], r[3]);
            float4 l;
            l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
            l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
            l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
            l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
            const size_t o = (((size_t)ib * HW + p0 + p) * C + cb * 16 + c) * 16 + i4;
            *reinterpret_cast<float4*>(hi + o) = x;
            *reinterpret_cast<float4*>(lo + o) = l;
        }
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(nonfinite, 1);
}

template <int BN, int PX>
cudaError_t launch_bww_bn(const CUtensorMap& ahi, const CUtensorMap& alo, const CUtensorMap& bhi,
                          const CUtensorMap& blo, const TcBwwGeo& g, float* partial, const int* nonfinite,
                          const unsigned long long* cnt, unsigned long long* exec_ctr, cudaStream_t st) {
    constexpr size_t STAGE = (size_t)PX * (2 * TC_BM * 64 + 2 * BN * 64);
    constexpr int ST = PX == 1 ? TC_ST : (int)((200 * 1024) / STAGE);
    const size_t smem = ST * STAGE + 1024 + 256;
    static PerDeviceOnce attr;
    int attr_dev = 0;
    if (attr.needed(attr_dev)) {
        cudaError_t e = cudaFuncSetAttribute(tc_bww_kernel<BN, PX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr.done(attr_dev);
    }
    dim3 grid((unsigned)(g.tgroups * g.ktiles * g.ctiles), (unsigned)g.splits);
    tc_bww_kernel<BN, PX><<<grid, TC_THREADS, smem, st>>>(ahi, alo, bhi, blo, g, partial, nonfinite, cnt, exec_ctr);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool tc_bww_supported(const DevShape& sh, int V) {
    if (V != 16) return false;
    if (sh.O != sh.P || (sh.O != 1 && sh.O != 2)) return false;
    if (!((sh.R == 3 && sh.S == 3) || (sh.R == 1 && sh.S == 1))) return false;
    if (sh.padW != (sh.R - 1) / 2 || sh.padH != (sh.S - 1) / 2) return false;
    if (sh.C % 16 || sh.K % 16) return false;
    if ((sh.K % 64) || (sh.C % 64)) return false;  // the exact fallback (tile BWW) needs 64-channel multiples
    // K = 64 wastes half of the M = 128 MMA rows but still beats the FFMA BWW
    // since the one-wave split fix (VGG conv1_2 62 vs ~50 TF/s; ResNet-50 3x3
    // 64-channel 55 vs 41)
    return tc::encode_fn() != nullptr;
}

// check_input: chk = D (ActCHWNn), oth = dY (ActNCHWc); else chk = dY (ActCHWNn), oth = D (ActNCHWc).
cudaError_t launch_tc_bww(bool check_input, bool sparse, const DevShape& sh, const float* chk, const float* oth,
                          float* dst, unsigned long long* exec_ctr, cudaStream_t st) {
    const int HW = sh.H * sh.W, HWp = sh.Hp * sh.Wp;
    const int NB = (sh.N + 15) / 16;
    const size_t nD = (size_t)NB * 16 * sh.C * HW, nY = (size_t)NB * 16 * sh.K * HWp;  // CHWNn sizes
    const int taps = sh.R * sh.S;
    // N tile = tpc taps x cw channels: stacking taps keeps the MMA N (and the
    // work per pipeline stage) large for 64/128-channel layers
    const int cw = sh.C >= 256 ? 256 : sh.C;
    const int tpc = taps == 1 ? 1 : (cw == 64 ? 3 : (cw == 128 ? 2 : 1));
    const int BN = cw * tpc;
    TcBwwGeo g;
    g.cw = cw;
    g.tpc = tpc;
    g.tgroups = (taps + tpc - 1) / tpc;
    g.Hp = sh.Hp;
    g.Wp = sh.Wp;
    g.R = sh.R;
    g.S = sh.S;
    g.padW = sh.padW;
    g.padH = sh.padH;
    g.K = sh.K;
    g.C = sh.C;
    g.ktiles = (sh.K + TC_BM - 1) / TC_BM;
    g.ctiles = (sh.C + cw - 1) / cw;
    g.str = sh.O;
    // two output pixels per stage for a small single-tap N tile (stride 1)
    const int px = (tpc == 1 && BN <= 128 && sh.O == 1) ? 2 : 1;
    g.stages = (long)NB * sh.Hp * ((sh.Wp + px - 1) / px);
    const long tiles = (long)g.tgroups * g.ktiles * g.ctiles;
    // at most one wave of CTAs (one per SM): rounding up would leave a second
    // wave of a few CTAs as long as the first (VGG conv3_2: 162 CTAs -> 144)
    long splits = 148 / tiles > 0 ? 148 / tiles : 1;
    const long min_stages = 64;               // keep each split's pipeline long
    if (splits > g.stages / min_stages) splits = g.stages / min_stages > 0 ? g.stages / min_stages : 1;
    g.splits = (int)splits;
    static const int seg_env = std::getenv("SPC_TC_SEG") ? std::atoi(std::getenv("SPC_TC_SEG")) : 0;
    g.seg = seg_env > 0 ? seg_env : 8;
    // scratch: [flag][counter] | D hi, D lo, dY hi, dY lo (pixel-major) | partials
    const size_t nP = (size_t)g.splits * taps * sh.K * sh.C;
    const size_t bytes = 256 + (2 * nD + 2 * nY) * 4 + nP * 4;
    uint8_t* scratch = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&scratch, bytes, st);
    if (e != cudaSuccess) return e;
    int* nonfinite = reinterpret_cast<int*>(scratch);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(scratch + 128);
    float* d_hi = reinterpret_cast<float*>(scratch + 256);
    float* d_lo = d_hi + nD;
    float* y_hi = d_lo + nD;
    float* y_lo = y_hi + nY;
    float* part = y_lo + nY;
    tc_zero_kernel<<<1, 1, 0, st>>>(nonfinite, cnt);
    unsigned long long* cp = (sparse && exec_ctr) ? cnt : nullptr;
    // exact executed_vector_fmas from the checked (ActCHWNn) operand -- its
    // ragged lanes are zeros; then both operands -> pixel-major hi + lo
    const unsigned tb_d = (unsigned)(NB * (sh.C / 16) * ((HW + 15) / 16));
    const unsigned tb_y = (unsigned)(NB * (sh.K / 16) * ((HWp + 15) / 16));
    if (check_input) {
        if (cp)
            tc_split_src_kernel<<<148 * 8, 256, 0, st>>>(chk, nullptr, nD / 4, sh.H, sh.W, sh.Hp, sh.Wp, sh.R, sh.S,
                                                         sh.padW, sh.padH, 0, (unsigned)(sh.K / 16), cp, nonfinite,
                                                         sh.O);
        tc_to_hwcn_split_kernel<true><<<tb_d, 256, 0, st>>>(chk, d_hi, d_lo, sh.N, sh.C, HW, nonfinite);
        tc_to_hwcn_split_kernel<false><<<tb_y, 256, 0, st>>>(oth, y_hi, y_lo, sh.N, sh.K, HWp, nonfinite);
    } else {
        if (cp)
            tc_split_src_kernel<<<148 * 8, 256, 0, st>>>(chk, nullptr, nY / 4, sh.Hp, sh.Wp, sh.H, sh.W, sh.R, sh.S,
                                                         sh.padW, sh.padH, 1, (unsigned)(sh.C / 16), cp, nonfinite,
                                                         sh.O);
        tc_to_hwcn_split_kernel<true><<<tb_y, 256, 0, st>>>(chk, y_hi, y_lo, sh.N, sh.K, HWp, nonfinite);
        tc_to_hwcn_split_kernel<false><<<tb_d, 256, 0, st>>>(oth, d_hi, d_lo, sh.N, sh.C, HW, nonfinite);
    }
    note_launch(cp ? 3 : 2);
    CUtensorMap ahi, alo, bhi, blo;
    // pixel-major [NB][H][W][C][16] = 5-D (16, C, W, H, NB); boxes = one pixel's channel tile
    const int dY5[5] = {16, sh.K, sh.Wp, sh.Hp, NB}, dD5[5] = {16, sh.C, sh.W, sh.H, NB};
    const int bA[5] = {16, TC_BM, px, 1, 1}, bB[5] = {16, cw, px, 1, 1};
    if (!make_map5(&ahi, y_hi, dY5, bA) || !make_map5(&alo, y_lo, dY5, bA) || !make_map5(&bhi, d_hi, dD5, bB) ||
        !make_map5(&blo, d_lo, dD5, bB)) {
        cudaFreeAsync(scratch, st);
        return cudaErrorInvalidValue;
    }
    unsigned long long* ex = (sparse && exec_ctr) ? exec_ctr : nullptr;
    // CTA pairs (two k tiles, half the D rows each) for single-tap 256-wide c tiles
    static const int bpair_env = std::getenv("SPC_TC_PAIR") ? std::atoi(std::getenv("SPC_TC_PAIR")) : 1;
    if (bpair_env && BN == 256 && tpc == 1 && g.ktiles % 2 == 0 && px == 1) {
        CUtensorMap bhi2, blo2;
        const int bB2[5] = {16, 128, 1, 1, 1};
        if (!make_map5(&bhi2, d_hi, dD5, bB2) || !make_map5(&blo2, d_lo, dD5, bB2)) {
            cudaFreeAsync(scratch, st);
            return cudaErrorInvalidValue;
        }
        constexpr size_t STAGE = 2 * TC_BM * 64 + 2 * 128 * 64;
        constexpr int PST = 6;
        const size_t smem = PST * STAGE + 1024 + 256;
        static PerDeviceOnce attr;
    int attr_dev = 0;
        if (attr.needed(attr_dev)) {
            e = cudaFuncSetAttribute(tc_bww_pair_kernel<PST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess) {
                cudaFreeAsync(scratch, st);
                return e;
            }
            attr.done(attr_dev);
        }
        dim3 grid((unsigned)(g.tgroups * g.ktiles * g.ctiles), (unsigned)g.splits);
        tc_bww_pair_kernel<PST><<<grid, TC_THREADS, smem, st>>>(ahi, alo, bhi2, blo2, g, part, nonfinite, cnt, ex);
        note_launch();
        e = cudaGetLastError();
    } else if (BN == 256)
        e = launch_bww_bn<256, 1>(ahi, alo, bhi, blo, g, part, nonfinite, cnt, ex, st);
    else if (BN == 192)
        e = launch_bww_bn<192, 1>(ahi, alo, bhi, blo, g, part, nonfinite, cnt, ex, st);
    else if (BN == 128)
        e = px == 2 ? launch_bww_bn<128, 2>(ahi, alo, bhi, blo, g, part, nonfinite, cnt, ex, st)
                    : launch_bww_bn<128, 1>(ahi, alo, bhi, blo, g, part, nonfinite, cnt, ex, st);
    else
        e = px == 2 ? launch_bww_bn<64, 2>(ahi, alo, bhi, blo, g, part, nonfinite, cnt, ex, st)
                    : launch_bww_bn<64, 1>(ahi, alo, bhi, blo, g, part, nonfinite, cnt, ex, st);
    if (e == cudaSuccess) {
        tc_bww_reduce_kernel<<<148 * 4, 256, 0, st>>>(part, dst, g.splits, sh.K, sh.C, sh.R, sh.S, nonfinite);
        note_launch();
        e = cudaGetLastError();
    }
    // non-finite operands: the FP32 dispatch with the reference's exact skip
    // semantics -- the FFMA tile kernel when the checked tensor is finite, the
    // shape-general kernel otherwise (dispatch.cu launch_bww); sel2 = 0 (TC
    // ran), 1 (tile), 2 (generic)
    if (e == cudaSuccess) {
        int* sel2 = stream_flags(st) ? stream_flags(st) + FLAG_TC_SEL2 : nullptr;
        e = sel2 ? cudaSuccess : cudaErrorMemoryAllocation;
        if (e == cudaSuccess) {
            const size_t chk_n = (size_t)((sh.N + 15) / 16) * 16 *
                                 (check_input ? (size_t)sh.C * sh.H * sh.W : (size_t)sh.K * sh.Hp * sh.Wp);
            launch_finite_all(chk, chk_n, sel2 + 1, st);
            tc_select_kernel<<<1, 1, 0, st>>>(nonfinite, sel2 + 1, sel2);
            note_launch();
            e = launch_tile_bww_when(check_input, sparse, sh, chk, oth, dst, exec_ctr, st, sel2, 1);
            if (e == cudaSuccess) {
                const int gs = bww_generic_splits(sh);
                const size_t E = (size_t)sh.K * sh.C * sh.S * sh.R;
                float* gpart = nullptr;
                e = cudaMallocAsync((void**)&gpart, (size_t)gs * E * sizeof(float), st);
                if (e == cudaSuccess) {
                    e = launch_bww_generic(check_input, sparse, sh, 16, chk, oth, gpart, gs, dst, exec_ctr, st, sel2, 2);
                    cudaFreeAsync(gpart, st);
                }
            }
        }
    }
    cudaFreeAsync(scratch, st);
    return e;
}

}  // namespace spc
