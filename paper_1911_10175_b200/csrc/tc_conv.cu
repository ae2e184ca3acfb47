// tc_conv.cu -- FWD / BWI on the 5th-generation tensor cores (tcgen05, TMEM,
// TMA), 3xTF32 split arithmetic: the optional tensor-core variant of
// SURVEY.md 8(f)4, selected with spc_set_math(SPC_MATH_TF32X3).
//
// Same semantics as the FFMA kernels (P/src/kernel_impl.hpp:51-202 for FWD,
// the BWI role swap at :61-66 and inverse row map at :85-89), different
// arithmetic: every fp32 operand x is split into hi = x with the low 13
// mantissa bits dropped (what the tensor core reads from an fp32 word in
// kind::tf32) and lo = x - hi (exact in fp32), and each product is formed as
// hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM.  The dropped lo*lo
// term and lo's own tf32 truncation leave ~2^-21 relative error per product,
// far inside the north-star gate (max|d|/max|ref| <= 1e-5); the measured
// errors are in DESIGN.md 4.7.  Zero source elements contribute exact zeros
// (0 * w = 0), so skipping them would not change the sum; the tensor-core
// variant therefore executes them (an all-zero tile is skipped).
//
// Inf/NaN: the split cannot reproduce IEEE products with Inf (Inf - Inf = NaN
// in lo), and the reference SKIPS zero sources, so a zero times an Inf filter
// tap contributes nothing there but NaN here.  A device-side scan sets a flag
// when the source or the filter holds a non-finite value; the tensor-core
// kernel then exits at entry and the FFMA tile kernel (gated on the same flag)
// computes the pass with the reference's exact skip semantics.
//
// GEMM view (one tile = one 128-pixel output box x BN output channels; CTAs
// are persistent and walk tiles n-tile-slowest):
//   M = 128 output pixels: a BW x BH box of one image (or of one output parity
//       class for BWI stride 2), BW*BH = 128
//   N = BN output channels (64 / 128 / 256)
//   reduction = (KB 16-channel blocks, tap): per stage the A tile is the
//   source box shifted by the tap (TMA 5-D tiled load from ActNCHWc
//   [N][C/16][H][W][16]: 64-byte rows, SWIZZLE_64B, traversal stride 2 for FWD
//   stride 2, out-of-image pixels zero-filled by TMA = the virtual padding),
//   the B tile is the tap's [BN][16] filter slice from a K-major copy the prep
//   kernel writes.
// Warp roles (384 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// MMA issuer (one thread), warps 2-9 = accumulator drain + epilogue, warps
// 10-11 = A hi/lo splitters (1x1 only).  The MMAs accumulate a segment of
// `seg` pipeline stages into one of two TMEM buffers (2 x BN columns) while the
// epilogue warps add the other buffer's partial sums into fp32 registers; the
// last segment's drain is followed by the store (TMEM -> registers ->
// ActNCHWc, fused Epi), which overlaps the next tile's MMAs.  All-zero tiles
// (sparse mode) are skipped.  BWW is in tc_bww.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tc_common.cuh"
#include "tc_conv.h"
#include "tile_conv.h"

namespace spc {
namespace {
using namespace tc;

// Geometry of one FWD/BWI launch, by value.  The output is covered by up to
// four parity classes (four only for BWI with stride 2, whose output pixel
// (2m + cy, 2n + cx) takes the taps v with (cy + pad - v) even from dY pixel
// m + (cy + pad - v) / 2 -- the reference's inverse row map, kernel_impl.hpp:
// 85-89); each class is a stride-1 (or, FWD stride 2, strided-source) conv
// over its own grid, listed as a tap table.
struct TcClass {
    int oy, ox;              // first output row / column; position = (oy + os*m, ox + os*n)
    int Hc, Wc;              // class grid extent
    int tiles_x, tiles_y;    // 128-pixel boxes over the class grid
    int tile0;               // first tile of the class within one (N tile, image)
    int ntap;
    int tap[9], dy[9], dx[9];  // filter tap v*R+u; source = (sstr*m + dy, sstr*n + dx)
};
struct TcGeo {
    int Ho, Wo;        // output spatial extent
    int bw, bh;        // output box (bw * bh = 128)
    int os, sstr;      // output position stride of the class grids; source traversal stride
    int ncls;
    TcClass cls[4];
    int tiles_img;     // tiles per (N tile, image)
    int Co;            // output channels
    int RB;            // reduction blocks (input channels / 16)
    int seg;           // pipeline stages per TMEM accumulation segment
    int N, ntiles;     // images; tiles = N * tiles_img * (Co / BN)
    size_t out_img;    // floats per output image
};

// INK: A's lo half computed in shared memory by two converter warps (1x1
// convs: each A element is used by one stage, and the split pass's lo copy --
// a full write + read of the source -- would dominate a 1x1 layer's traffic);
// otherwise (3x3: A elements recur in up to 9 tap stages) A_lo is a TMA load
// of the lo copy the split pass writes.
template <int BN, int ST, int KB, bool INK>
__global__ void __launch_bounds__(TC_CONV_THREADS, BN == 64 ? 2 : 1)  // BN = 64: two CTAs per SM (<= 80 registers)
    tc_conv_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                   const __grid_constant__ CUtensorMap map_bhi,
                   const __grid_constant__ CUtensorMap map_blo, TcGeo g, float* __restrict__ dst,
                   const int* __restrict__ nonfinite, const unsigned long long* __restrict__ cnt_tmp,
                   unsigned long long* __restrict__ exec_ctr, Epi epi, const uint8_t* __restrict__ zflag) {
    if (__ldg(nonfinite) != 0) return;  // the exact FFMA kernel runs instead
    // a stage = KB 16-channel blocks of one tap: A = KB sub-tiles of 128 rows x
    // 64 B (hi, then lo), B = KB sub-tiles of BN rows x 64 B (hi, then lo)
    constexpr uint32_t A_BYTES = KB * TC_BM * 64;
    constexpr uint32_t B_BYTES = KB * BN * 64;
    constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
    constexpr int HALF = BN / 2;  // accumulator columns per epilogue thread
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    // full[ST] empty[ST] tfull[2] tempty[2] conv[ST]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * STAGE);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * ST + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // persistent: this CTA runs tiles blockIdx.x, + gridDim.x, ...; tile t =
    // (n tile, image, class, box row, box column), n tile slowest so the CTAs
    // in flight share one filter slice in L2
    const int txy = g.tiles_img;
    const int ntiles = g.ntiles;
    const int NG = g.RB / KB;                 // channel-block groups (one per tap sweep)
    const int D = g.seg;                      // stages per accumulation segment
    // all-zero tile skipping (sparse mode): zflag[img][group][tile] = 0 when the
    // tile's source box (all taps) is zero in the group's channels; a tile's
    // flags are loaded once per tile as a bit mask (NG <= 64, host-checked) by
    // every role, so skipped stages never enter the pipeline
    auto live_mask = [&](int img, int tt) {
        if (zflag == nullptr) return ~0ull;
        unsigned long long m = 0;
        for (int grp = 0; grp < NG; ++grp)
            m |= (unsigned long long)(__ldg(zflag + ((size_t)img * NG + grp) * txy + tt) != 0) << grp;
        return m;
    };
    // Segments are fixed runs of D stages of the FULL stage sequence (dense
    // order), so skipping leaves every segment's summation grouping -- and the
    // result -- bitwise equal to dense mode; a segment with no live stage is
    // skipped by the MMA issuer and the epilogue alike.
    auto seg_live = [&](unsigned long long lm, int ls, int taps, int nstage) {
        const int g0 = (ls * D) / taps, g1 = (min(ls * D + D, nstage) - 1) / taps;
        const unsigned long long span = (g1 - g0 == 63) ? ~0ull : ((2ull << (g1 - g0)) - 1) << g0;
        return (lm & span) != 0;
    };
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (ST + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * ST + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * ST + 2 + b); };
    auto conv_bar = [&](int s) { return bar0 + 8u * (2 * ST + 4 + s); };
    auto tile_coords = [&](int t, int& img, int& x0, int& y0, int& n0, int& tt, int& c) {
        const int nt = t / (g.N * txy);
        int r = t - nt * g.N * txy;
        img = r / txy;
        r -= img * txy;
        tt = r;
        c = 0;
        while (c + 1 < g.ncls && r >= g.cls[c + 1].tile0) ++c;
        r -= g.cls[c].tile0;
        const int ty = r / g.cls[c].tiles_x;
        x0 = (r - ty * g.cls[c].tiles_x) * g.bw;
        y0 = ty * g.bh;
        n0 = nt * BN;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
            mbar_init(conv_bar(s), 2);  // one arrival per converter warp (INK)
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), 8);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (blockIdx.x == 0 && cnt_tmp && exec_ctr) atomicAdd(exec_ctr, *cnt_tmp);
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

    if (warp >= 10) {
        // Converters (INK only; otherwise idle until the final barrier): A_lo = A_hi - tf32_trunc(A_hi), elementwise on the
        // swizzled tile (same positions, so the layout carries over), for every
        // live stage in pipeline order; then the MMA may read the stage.  No lo
        // copy of the source tensor exists in HBM.
        const int ct = threadIdx.x - 10 * 32;  // 0 .. 63
        int gi = 0;
        for (int t = INK ? (int)blockIdx.x : ntiles; t < ntiles; t += gridDim.x) {
            int img, x0, y0, n0, tt, c;
            tile_coords(t, img, x0, y0, n0, tt, c);
            const unsigned long long lm = live_mask(img, tt);
            const int taps = g.cls[c].ntap;
            for (int grp = 0; grp < NG; ++grp) {
                if (!((lm >> grp) & 1ull)) continue;
                for (int j = 0; j < taps; ++j, ++gi) {
                    const int s = gi % ST;
                    mbar_wait(full_bar(s), (gi / ST) & 1);
                    const float4* hi = reinterpret_cast<const float4*>(smem + s * STAGE);
                    float4* lo = reinterpret_cast<float4*>(smem + s * STAGE + A_BYTES);
#pragma unroll
                    for (int q = ct; q < (int)(A_BYTES / 16); q += 64) {
                        const float4 x = hi[q];
                        float4 l;
                        l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
                        l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
                        l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
                        l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
                        lo[q] = l;
                    }
                    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor core
                    __syncwarp();
                    if (lane == 0) mbar_arrive(conv_bar(s));
                }
            }
        }
    } else if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_hi)) : "memory");
            if (!INK) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lo)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
            int gi = 0;  // stage counter across this CTA's tiles (the smem ring continues)
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int img, x0, y0, n0, tt, c;
                tile_coords(t, img, x0, y0, n0, tt, c);
                const TcClass& C = g.cls[c];
                const unsigned long long lm = live_mask(img, tt);
                for (int grp = 0; grp < NG; ++grp) {
                    if (!((lm >> grp) & 1ull)) continue;
                    const int rb = grp * KB;
                    for (int j = 0; j < C.ntap; ++j, ++gi) {
                        const int s = gi % ST;
                        if (gi >= ST) mbar_wait(empty_bar(s), ((gi / ST) - 1) & 1);
                        const uint32_t st = sbase + s * STAGE;
                        mbar_expect_tx(full_bar(s), INK ? STAGE - A_BYTES : STAGE);  // INK: A_lo computed in smem
                        const int sx = g.sstr * x0 + C.dx[j], sy = g.sstr * y0 + C.dy[j];
                        tma_load_5d(st, &map_hi, full_bar(s), 0, sx, sy, rb, img);
                        if (!INK) tma_load_5d(st + A_BYTES, &map_lo, full_bar(s), 0, sx, sy, rb, img);
                        const int brow = C.tap[j] * g.RB + rb;
                        tma_load_3d(st + 2 * A_BYTES, &map_bhi, full_bar(s), 0, n0, brow);
                        tma_load_3d(st + 2 * A_BYTES + B_BYTES, &map_blo, full_bar(s), 0, n0, brow);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tf32_idesc<BN>();
            int gi = 0, gseg = 0;
            for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
                int img, x0, y0, n0, tt, c;
                tile_coords(t, img, x0, y0, n0, tt, c);
                const int taps = g.cls[c].ntap, nstage = NG * taps, nseg = (nstage + D - 1) / D;
                const unsigned long long lm = live_mask(img, tt);
                int ne = 0;  // live segments of this tile
                for (int ls = 0; ls < nseg; ++ls) {
                    if (!seg_live(lm, ls, taps, nstage)) continue;
                    const int sg = gseg + ne++, buf = sg & 1;
                    if (sg >= 2) mbar_wait(tempty_bar(buf), ((sg >> 1) - 1) & 1);
                    const uint32_t tm = tmem + buf * BN;
                    bool first = true;
                    for (int it = ls * D; it < min(ls * D + D, nstage); ++it) {
                        if (!((lm >> (it / taps)) & 1ull)) continue;
                        const int s = gi % ST;
                        mbar_wait(full_bar(s), (gi / ST) & 1);
                        if (INK) mbar_wait(conv_bar(s), (gi / ST) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint32_t st = sbase + s * STAGE;
#pragma unroll
                        for (int k = 0; k < 2 * KB; ++k) {  // two K=8 steps (32 bytes) per 16-channel block
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
                        first = false;
                        umma_commit(empty_bar(s));
                        ++gi;
                    }
                    umma_commit(tfull_bar(buf));
                }
                gseg += ne;
            }
        }
        __syncwarp();
    } else {
        // Epilogue warps 2..9: TMEM lane quarter q = warp % 4 (the warp's
        // accessible lanes) = output pixels 32q..32q+31; column half h.
        // Each segment's partial sums are drained into fp32 registers
        // (round-to-nearest adds), which bounds the length of the tensor
        // core's truncating accumulation chain; the store of
        // a tile overlaps the next tile's MMAs.
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int m = q * 32 + lane;
        const int py = m / g.bw, px = m - py * g.bw;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const size_t plane = (size_t)g.Ho * g.Wo * 16;
        int gseg = 0;
        for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
            int img, x0, y0, n0, tt, c;
            tile_coords(t, img, x0, y0, n0, tt, c);
            const TcClass& C = g.cls[c];
            const int taps = C.ntap, nstage = NG * taps, nseg = (nstage + D - 1) / D;
            float acc[HALF];
#pragma unroll
            for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
            const unsigned long long lm = live_mask(img, tt);
            int ne = 0;  // an all-zero tile has none: outputs = epi(0)
            for (int ls = 0; ls < nseg; ++ls) {
                if (!seg_live(lm, ls, taps, nstage)) continue;
                const int sg = gseg + ne++, buf = sg & 1;
                mbar_wait_sleep(tfull_bar(buf), (sg >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    float v[16];
                    tmem_ld16(tmem + lane_off + buf * BN + h * HALF + 16 * j, v);
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[16 * j + e] += v[e];
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty_bar(buf));
            }
            gseg += ne;
            if (y0 + py < C.Hc && x0 + px < C.Wc) {
                const int y = C.oy + g.os * (y0 + py), x = C.ox + g.os * (x0 + px);
                float* out = dst + (size_t)img * g.out_img + ((size_t)y * g.Wo + x) * 16;
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    const int kb = ((n0 + h * HALF) >> 4) + j;
                    float* o = out + (size_t)kb * plane;
                    float v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = acc[16 * j + e];
                    if (epi.active()) {
                        const size_t base = (size_t)(o - dst);
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = epi.apply(v[e], base + e);
                    }
#pragma unroll
                    for (int e = 0; e < 16; e += 4)
                        *reinterpret_cast<float4*>(o + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * BN))
                     : "memory");
    }
}

// FilterKCRSblk (out-channel role `o`, reduction role `r`) -> K-major hi / lo
// copies [tap][r/16][o][16 r-lanes]; flags non-finite taps.
__global__ void tc_split_filter_kernel(const float* __restrict__ f, float* __restrict__ bhi,
                                       float* __restrict__ blo, int Co, int Cr, int R, int S,
                                       int* __restrict__ nonfinite) {
    const size_t n = (size_t)Co * Cr * R * S;
    int bad = 0;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        // destination index decomposition: ((tap * RB + rb) * Co + o) * 16 + rl
        const int rl = (int)(e & 15);
        size_t t = e >> 4;
        const int o = (int)(t % Co);
        t /= Co;
        const int rb = (int)(t % (Cr / 16));
        const int tap = (int)(t / (Cr / 16));
        const int v = tap / R, u = tap - v * R;
        const float x = __ldg(f + filter_index(Cr, S, R, 16, o, rb * 16 + rl, u, v));
        const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
        bhi[e] = x;
        blo[e] = x - h;
        bad |= !isfinite(x);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(nonfinite, 1);
}

// zflag[img][group][tile] = 1 when any source row of the tile's box -- the
// output rows (x sstr) widened by the taps' row offsets [ylo, yhi], clipped to
// the image -- holds a nonzero in the group's KB channel blocks (rowflag from
// the split pass; whole image rows, so the skip is row-granular).
__global__ void tc_zero_tiles_kernel(const uint8_t* __restrict__ rowflag, uint8_t* __restrict__ zflag, int N, int CB,
                                     int KB, int Hs, int tiles_x, int tiles_y, int bh, int ylo, int yhi, int sstr) {
    const int NG = CB / KB, txy = tiles_x * tiles_y;
    const long nflags = (long)N * NG * txy;
    for (long f = blockIdx.x * (long)blockDim.x + threadIdx.x; f < nflags; f += (long)gridDim.x * blockDim.x) {
        const int tt = (int)(f % txy);
        const int grp = (int)((f / txy) % NG);
        const int img = (int)(f / ((long)txy * NG));
        const int ty = tt / tiles_x;
        const int ya = max(sstr * ty * bh + ylo, 0), yb = min(sstr * (ty * bh + bh - 1) + yhi, Hs - 1);
        uint8_t nz = 0;
        for (int cb = grp * KB; cb < grp * KB + KB && !nz; ++cb)
            for (int y = ya; y <= yb && !nz; ++y) nz = rowflag[((size_t)img * CB + cb) * Hs + y];
        zflag[f] = nz;
    }
}

// ---------------------------------------------------------------- host
// K-major filter copy [taps*RB][Co][16], box = 16 x bn x kb.
bool make_filter_map(CUtensorMap* m, const float* p, int rows, int Co, int bn, int kb = 1) {
    cuuint64_t dims[3] = {16, (cuuint64_t)Co, (cuuint64_t)rows};
    cuuint64_t strides[2] = {64, (cuuint64_t)Co * 64};
    cuuint32_t box[3] = {16, (cuuint32_t)bn, (cuuint32_t)kb};
    cuuint32_t es[3] = {1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(p), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The 128-pixel box (bw x bh, powers of two) with the least padded area.
void choose_box(int Ho, int Wo, int* bw, int* bh) {
    long best = -1;
    for (int w = 128; w >= 1; w >>= 1) {
        const int h = 128 / w;
        const long area = (long)((Wo + w - 1) / w) * w * ((Ho + h - 1) / h) * h;
        if (best < 0 || area < best) {
            best = area;
            *bw = w;
            *bh = h;
        }
    }
}

template <int BN, int KB, bool INK>
cudaError_t launch_bn(const CUtensorMap& mhi, const CUtensorMap& mlo, const CUtensorMap& mbhi, const CUtensorMap& mblo, const TcGeo& g, int N, float* dst, const int* nonfinite,
                      const unsigned long long* cnt, unsigned long long* exec_ctr, const Epi& epi, cudaStream_t st,
                      const uint8_t* zflag) {
    constexpr size_t STAGE = KB * (2 * TC_BM * 64 + 2 * BN * 64);
    // 4 stages (3 stages at BN = 128 with two CTAs per SM measured 1-3% slower);
    // 2-block stages: as many stages as fit 200 KB
    constexpr int ST = KB == 1 ? 4 : (int)((200 * 1024) / STAGE);
    const size_t smem = ST * STAGE + 1024 + 256;
    static PerDeviceOnce attr;
    int attr_dev = 0;
    if (attr.needed(attr_dev)) {
        cudaError_t e = cudaFuncSetAttribute(tc_conv_kernel<BN, ST, KB, INK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(tc_conv_kernel<BN, ST, KB, INK>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
        attr.done(attr_dev);
    }
    TcGeo gg = g;
    gg.N = N;
    gg.ntiles = N * g.tiles_img * (g.Co / BN);
    // persistent CTAs: as many as fit per SM (2 for BN <= 128: their
    // prologues / stores overlap each other's main loops), or fewer tiles
    // (measured, VGG conv1_2 FWD at BN = 64: 1 CTA/SM 75, 2 CTAs/SM 117 TFLOP/s)
    const int per_sm = (int)((228u * 1024u) / (smem + 1024u)) >= 2 ? 2 : 1;
    static const int persist_env = std::getenv("SPC_TC_CTAS") ? std::atoi(std::getenv("SPC_TC_CTAS")) : 0;
    int ctas = persist_env > 0 ? persist_env : 148 * per_sm;
    if (ctas > gg.ntiles) ctas = gg.ntiles;
    dim3 grid((unsigned)ctas);
    tc_conv_kernel<BN, ST, KB, INK><<<grid, TC_CONV_THREADS, smem, st>>>(mhi, mlo, mbhi, mblo, gg, dst, nonfinite, cnt,
                                                                          exec_ctr, epi, zflag);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- CTA pairs
// tc_pair_kernel: the same FWD/BWI GEMM on a CTA pair (cluster of 2,
// tcgen05.mma.cta_group::2, M = 256): each CTA of the pair loads its own
// 128-pixel A tile and HALF of the BN filter rows, and the pair's leader issues
// one M=256 MMA over both shared memories -- the filter bytes per SM halve, so
// a stage is 32 KB instead of 48 and the ring is 6 stages deep.  Both CTAs'
// TMA loads signal the leader's full barrier; the leader's MMA completion is
// multicast to both CTAs' empty / TMEM-full barriers; both epilogues release a
// TMEM buffer on the leader's barrier.  Tiles pair up within one N tile (the
// filter half must match); one output class (FWD any stride, BWI stride 1).
template <int BN, int ST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_pair_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                   const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo, TcGeo g,
                   float* __restrict__ dst, const int* __restrict__ nonfinite,
                   const unsigned long long* __restrict__ cnt_tmp, unsigned long long* __restrict__ exec_ctr, Epi epi,
                   const uint8_t* __restrict__ zflag) {
    if (__ldg(nonfinite) != 0) return;  // uniform over the pair (same flag)
    constexpr uint32_t A_BYTES = TC_BM * 64;
    constexpr uint32_t BH_BYTES = (BN / 2) * 64;  // this CTA's half of the filter rows
    constexpr uint32_t STAGE = 2 * A_BYTES + 2 * BH_BYTES;
    constexpr int HALF = BN / 2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * STAGE);  // full[ST] empty[ST] tfull[2] tempty[2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 4);
    const uint32_t rank = cluster_rank();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int txy = g.tiles_img;
    const int per_nt = g.N * txy;               // tiles per N tile
    const int pairs_nt = (per_nt + 1) / 2;
    const int npairs = pairs_nt * (g.Co / BN);
    const int pair0 = blockIdx.x >> 1, pstep = gridDim.x >> 1;
    const int NG = g.RB;
    const int D = g.seg;
    const TcClass& C = g.cls[0];
    const int taps = C.ntap, nstage = NG * taps, nseg = (nstage + D - 1) / D;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (ST + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * ST + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * ST + 2 + b); };
    // pair p -> (n tile, this CTA's tile); the partner of a last odd tile recomputes it (no store)
    auto tile_of = [&](int p, uint32_t r, int& img, int& tt, int& x0, int& y0, int& n0, bool& own) {
        const int nt = p / pairs_nt, pp = p - nt * pairs_nt;
        int t = 2 * pp + (int)r;
        own = t < per_nt;
        if (!own) t = per_nt - 1;
        img = t / txy;
        tt = t - img * txy;
        const int ty = tt / C.tiles_x;
        x0 = (tt - ty * C.tiles_x) * g.bw;
        y0 = ty * g.bh;
        n0 = nt * BN;
    };
    auto mask_of = [&](int img, int tt) {
        if (zflag == nullptr) return ~0ull;
        unsigned long long m = 0;
        for (int grp = 0; grp < NG; ++grp)
            m |= (unsigned long long)(__ldg(zflag + ((size_t)img * NG + grp) * txy + tt) != 0) << grp;
        return m;
    };
    // the pair's live mask: both tiles' flags (identical in both CTAs)
    auto pair_mask = [&](int p) {
        int img, tt, x0, y0, n0;
        bool own;
        tile_of(p, 0, img, tt, x0, y0, n0, own);
        unsigned long long m = mask_of(img, tt);
        tile_of(p, 1, img, tt, x0, y0, n0, own);
        return m | mask_of(img, tt);
    };
    auto seg_live = [&](unsigned long long lm, int ls) {
        const int g0 = (ls * D) / taps, g1 = (min(ls * D + D, nstage) - 1) / taps;
        const unsigned long long span = (g1 - g0 == 63) ? ~0ull : ((2ull << (g1 - g0)) - 1) << g0;
        return (lm & span) != 0;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), 16);  // 8 epilogue warps x 2 CTAs (leader's barrier)
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (blockIdx.x == 0 && cnt_tmp && exec_ctr) atomicAdd(exec_ctr, *cnt_tmp);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(tmem_cols(2 * BN))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // both CTAs' barriers initialised before any cross-CTA arrive / TMA
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_hi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lo)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
            int gi = 0;
            for (int p = pair0; p < npairs; p += pstep) {
                int img, tt, x0, y0, n0;
                bool own;
                tile_of(p, rank, img, tt, x0, y0, n0, own);
                const unsigned long long lm = pair_mask(p);
                for (int grp = 0; grp < NG; ++grp) {
                    if (!((lm >> grp) & 1ull)) continue;
                    for (int j = 0; j < taps; ++j, ++gi) {
                        const int s = gi % ST;
                        if (gi >= ST) mbar_wait(empty_bar(s), ((gi / ST) - 1) & 1);
                        const uint32_t st = sbase + s * STAGE;
                        // the leader expects both CTAs' bytes on its own barrier
                        if (rank == 0) mbar_expect_tx(full_bar(s), 2 * STAGE);
                        const int sx = g.sstr * x0 + C.dx[j], sy = g.sstr * y0 + C.dy[j];
                        tma_load_5d_pair(st, &map_hi, full_bar(s), 0, sx, sy, grp, img);
                        tma_load_5d_pair(st + A_BYTES, &map_lo, full_bar(s), 0, sx, sy, grp, img);
                        const int brow = C.tap[j] * g.RB + grp;
                        const int nb = n0 + (int)rank * (BN / 2);
                        tma_load_3d_pair(st + 2 * A_BYTES, &map_bhi, full_bar(s), 0, nb, brow);
                        tma_load_3d_pair(st + 2 * A_BYTES + BH_BYTES, &map_blo, full_bar(s), 0, nb, brow);
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            // instruction descriptor: M = 256 (the pair), N = BN, tf32, K-major
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(BN >> 3) << 17) |
                                   ((uint32_t)(256 >> 4) << 24);
            int gi = 0, gseg = 0;
            for (int p = pair0; p < npairs; p += pstep) {
                const unsigned long long lm = pair_mask(p);
                int ne = 0;
                for (int ls = 0; ls < nseg; ++ls) {
                    if (!seg_live(lm, ls)) continue;
                    const int sg = gseg + ne++, buf = sg & 1;
                    if (sg >= 2) mbar_wait(tempty_bar(buf), ((sg >> 1) - 1) & 1);
                    const uint32_t tm = tmem + buf * BN;
                    bool first = true;
                    for (int it = ls * D; it < min(ls * D + D, nstage); ++it) {
                        if (!((lm >> (it / taps)) & 1ull)) continue;
                        const int s = gi % ST;
                        mbar_wait(full_bar(s), (gi / ST) & 1);
                        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                        const uint32_t st = sbase + s * STAGE;
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
                        first = false;
                        umma_commit_pair(empty_bar(s));
                        ++gi;
                    }
                    umma_commit_pair(tfull_bar(buf));
                }
                gseg += ne;
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int m = q * 32 + lane;
        const int py = m / g.bw, px = m - py * g.bw;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const size_t plane = (size_t)g.Ho * g.Wo * 16;
        int gseg = 0;
        for (int p = pair0; p < npairs; p += pstep) {
            int img, tt, x0, y0, n0;
            bool own;
            tile_of(p, rank, img, tt, x0, y0, n0, own);
            const unsigned long long lm = pair_mask(p);
            float acc[HALF];
#pragma unroll
            for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
            int ne = 0;
            for (int ls = 0; ls < nseg; ++ls) {
                if (!seg_live(lm, ls)) continue;
                const int sg = gseg + ne++, buf = sg & 1;
                mbar_wait_sleep(tfull_bar(buf), (sg >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    float v[16];
                    tmem_ld16(tmem + lane_off + buf * BN + h * HALF + 16 * j, v);
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[16 * j + e] += v[e];
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                     map_to_rank0(tempty_bar(buf)))
                                 : "memory");
            }
            gseg += ne;
            if (own && y0 + py < C.Hc && x0 + px < C.Wc) {
                const int y = y0 + py, x = x0 + px;
                float* out = dst + (size_t)img * g.out_img + ((size_t)y * g.Wo + x) * 16;
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    const int kb = ((n0 + h * HALF) >> 4) + j;
                    float* o = out + (size_t)kb * plane;
                    float v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = acc[16 * j + e];
                    if (epi.active()) {
                        const size_t base = (size_t)(o - dst);
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = epi.apply(v[e], base + e);
                    }
#pragma unroll
                    for (int e = 0; e < 16; e += 4)
                        *reinterpret_cast<float4*>(o + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    cluster_sync_all();  // the partner no longer arrives on / reads this CTA's barriers and smem
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * BN))
                     : "memory");
    }
}

template <int BN>
cudaError_t launch_pair(const CUtensorMap& mhi, const CUtensorMap& mlo, const CUtensorMap& mbhi,
                        const CUtensorMap& mblo, const TcGeo& g, int N, float* dst, const int* nonfinite,
                        const unsigned long long* cnt, unsigned long long* exec_ctr, const Epi& epi, cudaStream_t st,
                        const uint8_t* zflag) {
    constexpr size_t STAGE = 2 * TC_BM * 64 + 2 * (BN / 2) * 64;
    constexpr int ST = (int)((200 * 1024) / STAGE) > 8 ? 8 : (int)((200 * 1024) / STAGE);
    const size_t smem = ST * STAGE + 1024 + 256;
    static PerDeviceOnce attr;
    int attr_dev = 0;
    if (attr.needed(attr_dev)) {
        cudaError_t e = cudaFuncSetAttribute(tc_pair_kernel<BN, ST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr.done(attr_dev);
    }
    TcGeo gg = g;
    gg.N = N;
    const long per_nt = (long)N * g.tiles_img;
    const long npairs = ((per_nt + 1) / 2) * (g.Co / BN);
    long ctas = 148;
    if (ctas > 2 * npairs) ctas = 2 * npairs;
    tc_pair_kernel<BN, ST><<<(unsigned)ctas, TC_THREADS, smem, st>>>(mhi, mlo, mbhi, mblo, gg, dst, nonfinite, cnt,
                                                                     exec_ctr, epi, zflag);
    note_launch();
    return cudaGetLastError();
}

// ---------------------------------------------------------------- 64-channel 3x3 halo kernel
// tc_halo9_kernel (3x3 stride 1, BN = 64): the small-N tile is both L2-bound
// (each tap reloads a shifted 128-pixel A box: VGG conv1_2 moved 13.6 TB/s
// through L2 at 40% tensor-pipe activity) and MMA-issue-bound (6 short MMAs per
// barrier round trip).  Here a stage is ONE 16-channel block: a halo box of
// (RW + 2) rows x P pixels loaded once (the M = 128 rows are RW = 128 / P
// output rows x pitch P, the last two columns of each row not outputs), plus
// the filter slices of all 9 taps; the MMA issuer then runs 9 taps x 2 K steps
// x 3 products = 54 MMAs on it, the A operand of tap (dv, du) being the 128
// consecutive halo rows from row dv * P + du (the descriptor start moves by
// 64-byte rows; SWIZZLE_64B keys on the address bits, so base offset 0).
struct TcHalo9Geo {
    int Ho, Wo, P, RW, tiles_x, tiles_y, RB, fwd, N, ntiles;
    size_t out_img;
};

template <int P>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_halo9_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                    const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                    TcHalo9Geo g, float* __restrict__ dst, const int* __restrict__ nonfinite,
                    const unsigned long long* __restrict__ cnt_tmp, unsigned long long* __restrict__ exec_ctr,
                    Epi epi, const uint8_t* __restrict__ zflag) {
    if (__ldg(nonfinite) != 0) return;
    constexpr int BN = 64, RW = 128 / P, HALF = BN / 2;
    constexpr uint32_t HROWS = (RW + 2) * P;                                // halo rows loaded
    constexpr uint32_t A_HALF = ((HROWS + 8) * 64 + 1023) & ~1023u;       // + rows garbage columns read past it
    constexpr uint32_t B_TAP = BN * 64;
    constexpr uint32_t STAGE = 2 * A_HALF + 2 * 9 * B_TAP;
    constexpr uint32_t STAGE_TX = 2 * HROWS * 64 + 2 * 9 * B_TAP;
    constexpr int ST = 2;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + ST * STAGE);  // full[ST] empty[ST] tfull[2] tempty[2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 4);
    const uint32_t sbase = smem_u32(smem), bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (ST + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * ST + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * ST + 2 + b); };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int txy = g.tiles_x * g.tiles_y;
    const int NG = g.RB;
    auto tile_coords = [&](int t, int& img, int& tt, int& x0, int& y0) {
        img = t / txy;
        tt = t - img * txy;
        const int ty = tt / g.tiles_x;
        x0 = (tt - ty * g.tiles_x) * (P - 2);
        y0 = ty * RW;
    };
    auto live_mask = [&](int img, int tt) {
        if (zflag == nullptr) return ~0ull;
        unsigned long long m = 0;
        for (int grp = 0; grp < NG; ++grp)
            m |= (unsigned long long)(__ldg(zflag + ((size_t)img * NG + grp) * txy + tt) != 0) << grp;
        return m;
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (blockIdx.x == 0 && cnt_tmp && exec_ctr) atomicAdd(exec_ctr, *cnt_tmp);
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
        if (lane == 0) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_hi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lo)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
            int gi = 0;
            for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                int img, tt, x0, y0;
                tile_coords(t, img, tt, x0, y0);
                const unsigned long long lm = live_mask(img, tt);
                for (int rb = 0; rb < g.RB; ++rb) {
                    if (!((lm >> rb) & 1ull)) continue;
                    const int s = gi % ST;
                    if (gi >= ST) mbar_wait(empty_bar(s), ((gi / ST) - 1) & 1);
                    const uint32_t st = sbase + s * STAGE;
                    mbar_expect_tx(full_bar(s), STAGE_TX);
                    tma_load_5d(st, &map_hi, full_bar(s), 0, x0 - 1, y0 - 1, rb, img);
                    tma_load_5d(st + A_HALF, &map_lo, full_bar(s), 0, x0 - 1, y0 - 1, rb, img);
                    // shift (dv, du) reads source (y + dv - 1, x + du - 1): FWD tap (dv, du); BWI the
                    // transposed filter's tap (2 - dv, 2 - du) (kernel_impl.hpp:85-89)
                    for (int sft = 0; sft < 9; ++sft) {
                        const int brow = (g.fwd ? sft : 8 - sft) * g.RB + rb;
                        tma_load_3d(st + 2 * A_HALF + sft * B_TAP, &map_bhi, full_bar(s), 0, 0, brow);
                        tma_load_3d(st + 2 * A_HALF + (9 + sft) * B_TAP, &map_blo, full_bar(s), 0, 0, brow);
                    }
                    ++gi;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idesc = tf32_idesc<BN>();
            int gi = 0, sg = 0;
            for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
                int img, tt, x0, y0;
                tile_coords(t, img, tt, x0, y0);
                const unsigned long long lm = live_mask(img, tt);
                // one segment per channel block (54 MMAs)
                for (int rb = 0; rb < g.RB; ++rb, ++sg) {
                    if (!((lm >> rb) & 1ull)) {
                        --sg;
                        continue;
                    }
                    const int buf = sg & 1;
                    if (sg >= 2) mbar_wait(tempty_bar(buf), ((sg >> 1) - 1) & 1);
                    const int s = gi % ST;
                    mbar_wait(full_bar(s), (gi / ST) & 1);
                    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                    const uint32_t st = sbase + s * STAGE;
                    const uint32_t tm = tmem + buf * BN;
#pragma unroll
                    for (int sft = 0; sft < 9; ++sft) {
                        const uint32_t aoff = (uint32_t)(((sft / 3) * P + (sft % 3)) * 64);
                        const uint32_t bh = st + 2 * A_HALF + sft * B_TAP;
#pragma unroll
                        for (int k = 0; k < 2; ++k) {
                            const uint64_t ahi = sw64_desc(st + aoff + 32 * k);
                            const uint64_t alo = sw64_desc(st + A_HALF + aoff + 32 * k);
                            const uint64_t bhi = sw64_desc(bh + 32 * k);
                            const uint64_t blo = sw64_desc(bh + 9 * B_TAP + 32 * k);
                            umma_tf32(tm, alo, bhi, idesc, (sft == 0 && k == 0) ? 0u : 1u);
                            umma_tf32(tm, ahi, blo, idesc, 1u);
                            umma_tf32(tm, ahi, bhi, idesc, 1u);
                        }
                    }
                    umma_commit(empty_bar(s));
                    umma_commit(tfull_bar(buf));
                    ++gi;
                }
            }
        }
        __syncwarp();
    } else {
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int m = q * 32 + lane;
        const int py = m / P, px = m - py * P;
        const uint32_t lane_off = (uint32_t)(q * 32) << 16;
        const size_t plane = (size_t)g.Ho * g.Wo * 16;
        int sg = 0;
        for (int t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
            int img, tt, x0, y0;
            tile_coords(t, img, tt, x0, y0);
            const unsigned long long lm = live_mask(img, tt);
            float acc[HALF];
#pragma unroll
            for (int j = 0; j < HALF; ++j) acc[j] = 0.0f;
            for (int rb = 0; rb < g.RB; ++rb) {
                if (!((lm >> rb) & 1ull)) continue;
                const int buf = sg & 1;
                mbar_wait_sleep(tfull_bar(buf), (sg >> 1) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    float v[16];
                    tmem_ld16(tmem + lane_off + buf * BN + h * HALF + 16 * j, v);
#pragma unroll
                    for (int e = 0; e < 16; ++e) acc[16 * j + e] += v[e];
                }
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) mbar_arrive(tempty_bar(buf));
                ++sg;
            }
            const int y = y0 + py, x = x0 + px;
            if (px < P - 2 && y < g.Ho && x < g.Wo) {
                float* out = dst + (size_t)img * g.out_img + ((size_t)y * g.Wo + x) * 16;
#pragma unroll
                for (int j = 0; j < HALF / 16; ++j) {
                    float* o = out + (size_t)(h * (HALF / 16) + j) * plane;
                    float v[16];
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = acc[16 * j + e];
                    if (epi.active()) {
                        const size_t base = (size_t)(o - dst);
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = epi.apply(v[e], base + e);
                    }
#pragma unroll
                    for (int e = 0; e < 16; e += 4)
                        *reinterpret_cast<float4*>(o + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(tmem_cols(2 * 64))
                     : "memory");
    }
}

template <int P>
cudaError_t launch_halo9(const CUtensorMap& mhi, const CUtensorMap& mlo, const CUtensorMap& mbhi,
                         const CUtensorMap& mblo, const TcHalo9Geo& g, float* dst, const int* nonfinite,
                         const unsigned long long* cnt, unsigned long long* exec_ctr, const Epi& epi, cudaStream_t st,
                         const uint8_t* zflag) {
    constexpr int RW = 128 / P;
    constexpr size_t A_HALF = (((size_t)(RW + 2) * P + 8) * 64 + 1023) & ~(size_t)1023;
    constexpr size_t STAGE = 2 * A_HALF + 2 * 9 * 64 * 64;
    const size_t smem = 2 * STAGE + 1024 + 256;
    static PerDeviceOnce attr;
    int attr_dev = 0;
    if (attr.needed(attr_dev)) {
        cudaError_t e = cudaFuncSetAttribute(tc_halo9_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr.done(attr_dev);
    }
    int ctas = 148;
    if (ctas > g.ntiles) ctas = g.ntiles;
    tc_halo9_kernel<P><<<ctas, TC_THREADS, smem, st>>>(mhi, mlo, mbhi, mblo, g, dst, nonfinite, cnt, exec_ctr, epi,
                                                      zflag);
    note_launch();
    return cudaGetLastError();
}

// Pitch for the halo kernel: P - 2 output columns per row, least padded area.
int choose_pitch(int Ho, int Wo) {
    long best = -1;
    int bp = 64;
    for (int P : {64, 32, 16}) {
        const int rw = 128 / P;
        const long area = (long)((Wo + P - 3) / (P - 2)) * P * ((Ho + rw - 1) / rw) * rw;
        if (best < 0 || area < best) {
            best = area;
            bp = P;
        }
    }
    return bp;
}

}  // namespace

bool tc_conv_supported(bool fwd, const DevShape& sh, int V) {
    (void)fwd;
    if (V != 16) return false;
    if (sh.O != sh.P || (sh.O != 1 && sh.O != 2)) return false;
    if (!((sh.R == 3 && sh.S == 3) || (sh.R == 1 && sh.S == 1))) return false;
    if (sh.padW != (sh.R - 1) / 2 || sh.padH != (sh.S - 1) / 2) return false;
    const int Co = fwd ? sh.K : sh.C;
    if (Co % 64) return false;
    return tc::encode_fn() != nullptr;
}

cudaError_t launch_tc_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi) {
    const int Co = fwd ? sh.K : sh.C, Cr = fwd ? sh.C : sh.K;
    const int Hs = fwd ? sh.H : sh.Hp, Ws = fwd ? sh.W : sh.Wp;
    const int Ho = fwd ? sh.Hp : sh.H, Wo = fwd ? sh.Wp : sh.W;
    const int taps = sh.R * sh.S;
    const size_t nsrc = (size_t)sh.N * Cr * Hs * Ws;
    const size_t nfilt = (size_t)Co * Cr * taps;
    // scratch: [flag, pad][counter][filter hi][filter lo][src lo (3x3 only: 1x1 splits A in shared memory)]
    const bool ink = sh.R == 1 && sh.S == 1;
    const size_t bytes = 256 + 2 * nfilt * 4 + (ink ? 0 : nsrc * 4);
    uint8_t* scratch = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&scratch, bytes, st);
    if (e != cudaSuccess) return e;
    int* nonfinite = reinterpret_cast<int*>(scratch);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(scratch + 128);
    float* bhi = reinterpret_cast<float*>(scratch + 256);
    float* blo = bhi + nfilt;
    float* lo = ink ? nullptr : blo + nfilt;
    tc_zero_kernel<<<1, 1, 0, st>>>(nonfinite, cnt);
    tc_split_filter_kernel<<<(unsigned)((nfilt + 255) / 256 < 148 * 8 ? (nfilt + 255) / 256 : 148 * 8), 256, 0, st>>>(
        filt, bhi, blo, Co, Cr, sh.R, sh.S, nonfinite);
    note_launch(2);

    // Output classes and tap tables (TcGeo): FWD (any stride) and BWI stride 1
    // are one class over the whole output; BWI stride 2 splits the output into
    // its 4 parity classes (P/include/spconv/tensor.hpp:57-66 restated per class).
    const int str = sh.O;  // O == P (tc_conv_supported)
    TcGeo g;
    std::memset(&g, 0, sizeof(g));
    g.Ho = Ho;
    g.Wo = Wo;
    g.Co = Co;
    g.RB = Cr / 16;
    g.out_img = (size_t)Co * Ho * Wo;
    g.sstr = fwd ? str : 1;
    g.os = (!fwd && str == 2) ? 2 : 1;
    g.ncls = (!fwd && str == 2) ? 4 : 1;
    int ylo = 1 << 20, yhi = -(1 << 20);  // tap row-offset extents (zero-tile flags)
    {
        // one box shape for every class (the classes of BWI stride 2 differ by at most one row / column)
        const int Hc0 = (Ho + g.os - 1) / g.os, Wc0 = (Wo + g.os - 1) / g.os;
        choose_box(Hc0, Wc0, &g.bw, &g.bh);
        int tile0 = 0;
        for (int c = 0; c < g.ncls; ++c) {
            TcClass& C = g.cls[c];
            const int cy = g.ncls == 4 ? c >> 1 : 0, cx = g.ncls == 4 ? c & 1 : 0;
            C.oy = cy;
            C.ox = cx;
            C.Hc = (Ho - cy + g.os - 1) / g.os;
            C.Wc = (Wo - cx + g.os - 1) / g.os;
            C.tiles_x = (C.Wc + g.bw - 1) / g.bw;
            C.tiles_y = (C.Hc + g.bh - 1) / g.bh;
            C.tile0 = tile0;
            tile0 += C.tiles_x * C.tiles_y;
            C.ntap = 0;
            for (int v = 0; v < sh.S; ++v)
                for (int u = 0; u < sh.R; ++u) {
                    int dy, dx;
                    if (fwd) {  // source = str * out + tap - pad (kernel_impl.hpp:82-84)
                        dy = v - sh.padH;
                        dx = u - sh.padW;
                    } else {    // out = str * y' + tap - pad  =>  y' = (out + pad - tap) / str
                        const int ny = cy + sh.padH - v, nx = cx + sh.padW - u;
                        if (((ny % str) + str) % str || ((nx % str) + str) % str) continue;
                        dy = ny / str;
                        dx = nx / str;
                    }
                    C.tap[C.ntap] = v * sh.R + u;
                    C.dy[C.ntap] = dy;
                    C.dx[C.ntap] = dx;
                    ++C.ntap;
                    ylo = std::min(ylo, dy);
                    yhi = std::max(yhi, dy);
                }
        }
        g.tiles_img = tile0;
    }
    // SPC_TC_SEG overrides the segment length (accuracy / speed experiments)
    static const int seg_env = std::getenv("SPC_TC_SEG") ? std::atoi(std::getenv("SPC_TC_SEG")) : 0;
    g.seg = seg_env > 0 ? seg_env : 8;  // error 1.2-1.4e-6 measured

    CUtensorMap mhi, mlo, mbhi, mblo;
    // N tile 256 when Co allows (128-wide tiles to fill the last round of
    // persistent CTAs measured slower: VGG conv3_2 185 -> 156, conv4 170 -> 155)
    const int bn = Co % 256 == 0 ? 256 : (Co % 128 == 0 ? 128 : 64);
    // BN = 128: two 16-channel blocks per pipeline stage (K = 32: twice the
    // MMAs per barrier round trip; measured VGG conv2_2 140 -> 180 TF/s).  BN =
    // 64 keeps one block per stage and two CTAs per SM (2-block stages there:
    // 117 -> 103), BN = 256 one (a 96 KB stage would leave 2 stages).
    static const int kb_env = std::getenv("SPC_TC_KB") ? std::atoi(std::getenv("SPC_TC_KB")) : 0;
    const int kb = (kb_env == 1 || bn != 128 || (Cr / 16) % 2) ? 1 : 2;
    if (!make_act_map(&mhi, src, sh.N, Cr / 16, Hs, Ws, g.bw, g.bh, kb, g.sstr) ||
        !make_act_map(&mlo, ink ? src : lo, sh.N, Cr / 16, Hs, Ws, g.bw, g.bh, kb, g.sstr) ||
        !make_filter_map(&mbhi, bhi, taps * (Cr / 16), Co, bn, kb) ||
        !make_filter_map(&mblo, blo, taps * (Cr / 16), Co, bn, kb)) {
        cudaFreeAsync(scratch, st);
        return cudaErrorInvalidValue;
    }
    // sparse mode: all-zero tile flags from row flags the split pass marks
    // (SPC_TC_SKIP=0 disables the skip)
    static const int skip_env = std::getenv("SPC_TC_SKIP") ? std::atoi(std::getenv("SPC_TC_SKIP")) : 1;
    uint8_t* zflag = nullptr;
    uint8_t* rowflag = nullptr;
    const bool skip = sparse && skip_env && (Cr / 16) / kb <= 64 && g.ncls == 1;
    const size_t nrows = (size_t)sh.N * (Cr / 16) * Hs;
    const size_t nflags = skip ? (size_t)sh.N * ((Cr / 16) / kb) * g.tiles_img : 0;
    if (skip) {
        e = cudaMallocAsync((void**)&rowflag, nrows + nflags, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(rowflag, 0, nrows, st);
        if (e != cudaSuccess) {
            cudaFreeAsync(scratch, st);
            return e;
        }
        zflag = rowflag + nrows;
    }
    tc_split_src_kernel<<<148 * 8, 256, 0, st>>>(src, lo, nsrc / 4, Hs, Ws, Ho, Wo, sh.R, sh.S, sh.padW, sh.padH,
                                                 fwd ? 0 : 1, (unsigned)(Co / 16), (sparse && exec_ctr) ? cnt : nullptr,
                                                 nonfinite, sh.O, rowflag);
    note_launch();
    if (skip) {
        const size_t blocks = (nflags + 255) / 256;
        tc_zero_tiles_kernel<<<(unsigned)(blocks < 148 * 8 ? blocks : 148 * 8), 256, 0, st>>>(
            rowflag, zflag, sh.N, Cr / 16, kb, Hs, g.cls[0].tiles_x, g.cls[0].tiles_y, g.bh, ylo, yhi, g.sstr);
        note_launch();
    }
    unsigned long long* ex = (sparse && exec_ctr) ? exec_ctr : nullptr;
    // 64-channel 3x3 stride-1 outputs: the halo kernel, one channel block (all 9
    // taps) per stage (SPC_TC_HALO=0 disables)
    static const int halo_env = std::getenv("SPC_TC_HALO") ? std::atoi(std::getenv("SPC_TC_HALO")) : 1;
    if (halo_env && bn == 64 && Co == 64 && sh.R == 3 && sh.S == 3 && str == 1 && g.ncls == 1 && !ink) {
        TcHalo9Geo hg;
        hg.Ho = Ho;
        hg.Wo = Wo;
        hg.P = choose_pitch(Ho, Wo);
        hg.RW = 128 / hg.P;
        hg.tiles_x = (Wo + hg.P - 3) / (hg.P - 2);
        hg.tiles_y = (Ho + hg.RW - 1) / hg.RW;
        hg.RB = Cr / 16;
        hg.fwd = fwd ? 1 : 0;
        hg.N = sh.N;
        hg.ntiles = sh.N * hg.tiles_x * hg.tiles_y;
        hg.out_img = g.out_img;
        CUtensorMap hhi, hlo;
        if (!make_act_map(&hhi, src, sh.N, Cr / 16, Hs, Ws, hg.P, hg.RW + 2, 1) ||
            !make_act_map(&hlo, lo, sh.N, Cr / 16, Hs, Ws, hg.P, hg.RW + 2, 1)) {
            if (rowflag) cudaFreeAsync(rowflag, st);
            cudaFreeAsync(scratch, st);
            return cudaErrorInvalidValue;
        }
        // the zero-tile flags are per box tile of the generic geometry: not usable here
        e = hg.P == 64   ? launch_halo9<64>(hhi, hlo, mbhi, mblo, hg, dst, nonfinite, cnt, ex, epi, st, nullptr)
            : hg.P == 32 ? launch_halo9<32>(hhi, hlo, mbhi, mblo, hg, dst, nonfinite, cnt, ex, epi, st, nullptr)
                         : launch_halo9<16>(hhi, hlo, mbhi, mblo, hg, dst, nonfinite, cnt, ex, epi, st, nullptr);
        if (e == cudaSuccess)
            e = launch_tile_conv_when(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi, nonfinite, 1);
        if (rowflag) cudaFreeAsync(rowflag, st);
        cudaFreeAsync(scratch, st);
        return e;
    }
    // CTA pairs (SPC_TC_PAIR=0 disables): 3x3 / 1x1 without the in-smem split,
    // one output class, one block per stage
    static const int pair_env = std::getenv("SPC_TC_PAIR") ? std::atoi(std::getenv("SPC_TC_PAIR")) : 1;
    // (measured: +5-8% on the BN = 256 VGG layers, conv3_2 179 -> 190 TF/s; a BN = 128 pair with one block
    // per stage lost to the single-CTA two-block stages, conv2_2 173 -> 132)
    if (pair_env && !ink && g.ncls == 1 && kb == 1 && bn == 256) {
        CUtensorMap mbhi2, mblo2;
        if (!make_filter_map(&mbhi2, bhi, taps * (Cr / 16), Co, bn / 2, 1) ||
            !make_filter_map(&mblo2, blo, taps * (Cr / 16), Co, bn / 2, 1)) {
            cudaFreeAsync(scratch, st);
            return cudaErrorInvalidValue;
        }
        e = launch_pair<256>(mhi, mlo, mbhi2, mblo2, g, sh.N, dst, nonfinite, cnt, ex, epi, st, zflag);
        if (e == cudaSuccess)
            e = launch_tile_conv_when(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi, nonfinite, 1);
        if (rowflag) cudaFreeAsync(rowflag, st);
        cudaFreeAsync(scratch, st);
        return e;
    }
#define SPC_TCL(BN_, KB_)                                                                                      \
    (ink ? launch_bn<BN_, KB_, true>(mhi, mlo, mbhi, mblo, g, sh.N, dst, nonfinite, cnt, ex, epi, st, zflag)    \
         : launch_bn<BN_, KB_, false>(mhi, mlo, mbhi, mblo, g, sh.N, dst, nonfinite, cnt, ex, epi, st, zflag))
    if (bn == 256)
        e = SPC_TCL(256, 1);
    else if (bn == 128)
        e = kb == 2 ? SPC_TCL(128, 2) : SPC_TCL(128, 1);
    else
        e = SPC_TCL(64, 1);
#undef SPC_TCL
    // non-finite source or filter: the FFMA tile kernel with the reference's exact skip semantics
    if (e == cudaSuccess) e = launch_tile_conv_when(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi, nonfinite, 1);
    if (rowflag) cudaFreeAsync(rowflag, st);
    cudaFreeAsync(scratch, st);
    return e;
}

}  // namespace spc
