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
// GEMM view (one CTA = one 128-pixel output box x BN output channels):
//   M = 128 output pixels: a BW x BH box of one image, BW*BH = 128
//   N = BN output channels (64 / 128 / 256)
//   reduction = (16-channel block rb, tap (v,u)): per step the A tile is the
//   source box shifted by the tap (TMA 5-D tiled load from ActNCHWc
//   [N][C/16][H][W][16]: 64-byte rows, SWIZZLE_64B, out-of-image pixels
//   zero-filled by TMA = the virtual padding), the B tile is the tap's
//   [BN][16] filter slice from a K-major copy the prep kernel writes.
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// MMA issuer (one elected thread), warps 2-9 = accumulator drain + epilogue.
// The MMAs accumulate a segment of `seg` pipeline stages into one of two TMEM
// buffers (2 x BN columns) while the epilogue warps add the other buffer's
// partial sums into fp32 registers; the last segment's drain is followed by
// the store (TMEM -> registers -> ActNCHWc, fused Epi).  4-stage mbarrier
// pipeline for the operands.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "pw_bww.h"
#include "tc_conv.h"
#include "tile_conv.h"

namespace spc {
namespace {

constexpr int TC_BM = 128;
constexpr int TC_ST = 4;          // pipeline stages
constexpr int TC_THREADS = 320;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
    } while (!ok);
}
// Same, with a back-off: for the epilogue warps, which wait a whole segment
// and would otherwise take issue slots from the producer / MMA threads.
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
        if (ok) break;
        __nanosleep(256);
    }
}
__device__ __forceinline__ void tma_load_5d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
        : "memory");
}
// UMMA shared-memory descriptor, K-major, SWIZZLE_64B: rows of 64 bytes,
// 8-row groups 512 bytes apart (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sw64_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
    d |= (uint64_t)1 << 16;              // LBO (unused for swizzled K-major)
    d |= (uint64_t)(512 >> 4) << 32;     // SBO
    d |= (uint64_t)1 << 46;              // version
    d |= (uint64_t)4 << 61;              // SWIZZLE_64B
    return d;
}
// Instruction descriptor: kind::tf32, D = f32, A/B K-major, M = 128, N = BN.
template <int BN>
__device__ __forceinline__ uint32_t tf32_idesc() {
    return (1u << 4)                        // D format f32
           | (2u << 7) | (2u << 10)         // A, B = tf32
           | ((uint32_t)(BN >> 3) << 17)    // N
           | ((uint32_t)(TC_BM >> 4) << 24);  // M
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
}

// Geometry of one launch, by value.
struct TcGeo {
    int Ho, Wo;        // output spatial extent
    int bw, bh;        // output box (bw * bh = 128)
    int tiles_x, tiles_y;
    int Co;            // output channels
    int RB;            // reduction blocks (input channels / 16)
    int R, S;          // filter columns, rows
    int sgn;           // +1 FWD (src = out + tap - pad), -1 BWI (src = out + pad - tap)
    int padW, padH;
    int seg;           // pipeline stages per TMEM accumulation segment
    size_t out_img;    // floats per output image
};

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_conv_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                   const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                   TcGeo g, float* __restrict__ dst, const int* __restrict__ nonfinite,
                   const unsigned long long* __restrict__ cnt_tmp, unsigned long long* __restrict__ exec_ctr,
                   Epi epi) {
    if (__ldg(nonfinite) != 0) return;  // the exact FFMA kernel runs instead
    constexpr uint32_t A_BYTES = TC_BM * 64;
    constexpr uint32_t B_BYTES = BN * 64;
    constexpr uint32_t STAGE = 2 * A_BYTES + 2 * B_BYTES;
    constexpr int HALF = BN / 2;  // accumulator columns per epilogue thread
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TC_ST * STAGE);  // full[ST] empty[ST] tfull[2] tempty[2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * TC_ST + 4);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x;
    const int img = tile / (g.tiles_x * g.tiles_y);
    const int trem = tile - img * g.tiles_x * g.tiles_y;
    const int ty = trem / g.tiles_x, tx = trem - ty * g.tiles_x;
    const int x0 = tx * g.bw, y0 = ty * g.bh;
    const int n0 = blockIdx.y * BN;
    const int niter = g.RB * g.R * g.S;
    const int D = g.seg;  // stages per accumulation segment
    const int nseg = (niter + D - 1) / D;
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar0 = smem_u32(bars);
    auto full_bar = [&](int s) { return bar0 + 8u * s; };
    auto empty_bar = [&](int s) { return bar0 + 8u * (TC_ST + s); };
    auto tfull_bar = [&](int b) { return bar0 + 8u * (2 * TC_ST + b); };
    auto tempty_bar = [&](int b) { return bar0 + 8u * (2 * TC_ST + 2 + b); };

    if (threadIdx.x == 0) {
        for (int s = 0; s < TC_ST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(tfull_bar(b), 1);
            mbar_init(tempty_bar(b), 8);  // one arrival per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (blockIdx.x == 0 && blockIdx.y == 0 && cnt_tmp && exec_ctr) atomicAdd(exec_ctr, *cnt_tmp);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(2 * BN)
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
            int rb = 0, v = 0, u = 0;
            for (int it = 0; it < niter; ++it) {
                const int s = it % TC_ST;
                if (it >= TC_ST) mbar_wait(empty_bar(s), ((it / TC_ST) - 1) & 1);
                const uint32_t st = sbase + s * STAGE;
                mbar_expect_tx(full_bar(s), STAGE);
                const int sx = x0 + g.sgn * (u - g.padW), sy = y0 + g.sgn * (v - g.padH);
                tma_load_5d(st, &map_hi, full_bar(s), 0, sx, sy, rb, img);
                tma_load_5d(st + A_BYTES, &map_lo, full_bar(s), 0, sx, sy, rb, img);
                const int brow = (v * g.R + u) * g.RB + rb;
                tma_load_3d(st + 2 * A_BYTES, &map_bhi, full_bar(s), 0, n0, brow);
                tma_load_3d(st + 2 * A_BYTES + B_BYTES, &map_blo, full_bar(s), 0, n0, brow);
                if (++u == g.R) {
                    u = 0;
                    if (++v == g.S) {
                        v = 0;
                        ++rb;
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
                const int s = it % TC_ST;
                mbar_wait(full_bar(s), (it / TC_ST) & 1);
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                const uint32_t st = sbase + s * STAGE;
                const uint32_t tm = tmem + buf * BN;
#pragma unroll
                for (int k = 0; k < 2; ++k) {  // two K=8 steps per 16-channel block (32 bytes each)
                    const uint64_t ahi = sw64_desc(st + 32 * k);
                    const uint64_t alo = sw64_desc(st + A_BYTES + 32 * k);
                    const uint64_t bhi = sw64_desc(st + 2 * A_BYTES + 32 * k);
                    const uint64_t blo = sw64_desc(st + 2 * A_BYTES + B_BYTES + 32 * k);
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
        // Epilogue warps 2..9: TMEM lane quarter q = warp % 4 (the warp's
        // accessible lanes) = output pixels 32q..32q+31; column half h.
        // Each segment's partial sums are drained into fp32 registers
        // (round-to-nearest adds), which bounds the length of the tensor
        // core's truncating accumulation chain.
        const int q = warp & 3, h = (warp - 2) >> 2;
        const int m = q * 32 + lane;
        const int py = m / g.bw, px = m - py * g.bw;
        const int y = y0 + py, x = x0 + px;
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
                float v[16];
                tmem_ld16(tmem + lane_off + buf * BN + h * HALF + 16 * j, v);
#pragma unroll
                for (int e = 0; e < 16; ++e) acc[16 * j + e] += v[e];
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tempty_bar(buf)) : "memory");
        }
        if (y < g.Ho && x < g.Wo) {
            const size_t plane = (size_t)g.Ho * g.Wo * 16;
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
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 1) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BN) : "memory");
    }
}

// lo = x - tf32_trunc(x) over the source; counts executed_vector_fmas the
// reference's way (P/src/oracle.cpp:160-230): every nonzero source element
// adds rows(y) * cols(x), scaled by Co/16 at the end; flags non-finite values.
__global__ void tc_split_src_kernel(const float* __restrict__ src, float* __restrict__ lo, size_t n4, int Hs,
                                    int Ws, int Ho, int Wo, int R, int S, int padW, int padH, int bwi,
                                    unsigned scale, unsigned long long* __restrict__ cnt,
                                    int* __restrict__ nonfinite) {
    unsigned long long acc = 0;
    int bad = 0;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n4; e += (size_t)gridDim.x * blockDim.x) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src) + e);
        float4 l;
        l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
        l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
        l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
        l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
        reinterpret_cast<float4*>(lo)[e] = l;
        bad |= !isfinite(x.x) | !isfinite(x.y) | !isfinite(x.z) | !isfinite(x.w);
        const unsigned nz = (x.x != 0.0f) + (x.y != 0.0f) + (x.z != 0.0f) + (x.w != 0.0f);
        if (nz && cnt) {
            const size_t pix = (e * 4) / 16;  // (image, channel block, y, x) pixel of the 16-lane vector
            const int xx = (int)(pix % Ws);
            const int yy = (int)((pix / Ws) % Hs);
            int rows = 0, cols = 0;
            for (int v = 0; v < S; ++v) {
                const int o = bwi ? yy + v - padH : yy + padH - v;  // stride 1
                rows += (o >= 0 && o < Ho) ? 1 : 0;
            }
            for (int u = 0; u < R; ++u) {
                const int o = bwi ? xx + u - padW : xx + padW - u;
                cols += (o >= 0 && o < Wo) ? 1 : 0;
            }
            acc += (unsigned long long)nz * rows * cols * scale;
        }
    }
    if (cnt) {
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if ((threadIdx.x & 31) == 0 && acc) atomicAdd(cnt, acc);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(nonfinite, 1);
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

__global__ void tc_zero_kernel(int* flag, unsigned long long* cnt) {
    *flag = 0;
    *cnt = 0;
}

// ---------------------------------------------------------------- host
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// ActNCHWc [N][CB][H][W][16] as a 5-D map, box = 16 ch x bw x bh x 1 x 1.
bool make_act_map(CUtensorMap* m, const float* p, int N, int CB, int H, int W, int bw, int bh) {
    cuuint64_t dims[5] = {16, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)CB, (cuuint64_t)N};
    cuuint64_t strides[4] = {64, (cuuint64_t)W * 64, (cuuint64_t)H * W * 64, (cuuint64_t)CB * H * W * 64};
    cuuint32_t box[5] = {16, (cuuint32_t)bw, (cuuint32_t)bh, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(p), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
// K-major filter copy [taps*RB][Co][16], box = 16 x bn x 1.
bool make_filter_map(CUtensorMap* m, const float* p, int rows, int Co, int bn) {
    cuuint64_t dims[3] = {16, (cuuint64_t)Co, (cuuint64_t)rows};
    cuuint64_t strides[2] = {64, (cuuint64_t)Co * 64};
    cuuint32_t box[3] = {16, (cuuint32_t)bn, 1};
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

template <int BN>
cudaError_t launch_bn(const CUtensorMap& mhi, const CUtensorMap& mlo, const CUtensorMap& mbhi,
                      const CUtensorMap& mblo, const TcGeo& g, int N, float* dst, const int* nonfinite,
                      const unsigned long long* cnt, unsigned long long* exec_ctr, const Epi& epi, cudaStream_t st) {
    constexpr size_t STAGE = 2 * TC_BM * 64 + 2 * BN * 64;
    const size_t smem = TC_ST * STAGE + 1024 + 256;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(tc_conv_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((unsigned)(N * g.tiles_x * g.tiles_y), (unsigned)(g.Co / BN));
    tc_conv_kernel<BN><<<grid, TC_THREADS, smem, st>>>(mhi, mlo, mbhi, mblo, g, dst, nonfinite, cnt, exec_ctr, epi);
    note_launch();
    return cudaGetLastError();
}

}  // namespace

bool tc_conv_supported(bool fwd, const DevShape& sh, int V) {
    (void)fwd;
    if (V != 16) return false;
    if (sh.O != 1 || sh.P != 1) return false;
    if (!((sh.R == 3 && sh.S == 3) || (sh.R == 1 && sh.S == 1))) return false;
    if (sh.padW != (sh.R - 1) / 2 || sh.padH != (sh.S - 1) / 2) return false;
    const int Co = fwd ? sh.K : sh.C;
    if (Co % 64) return false;
    return encode_fn() != nullptr;
}

cudaError_t launch_tc_conv(bool fwd, bool sparse, const DevShape& sh, const float* src, const float* filt,
                           float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi) {
    const int Co = fwd ? sh.K : sh.C, Cr = fwd ? sh.C : sh.K;
    const int Hs = fwd ? sh.H : sh.Hp, Ws = fwd ? sh.W : sh.Wp;
    const int Ho = fwd ? sh.Hp : sh.H, Wo = fwd ? sh.Wp : sh.W;
    const int taps = sh.R * sh.S;
    const size_t nsrc = (size_t)sh.N * Cr * Hs * Ws;
    const size_t nfilt = (size_t)Co * Cr * taps;
    // scratch: [flag, pad][counter][src lo][filter hi][filter lo]
    const size_t bytes = 256 + nsrc * 4 + 2 * nfilt * 4;
    uint8_t* scratch = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&scratch, bytes, st);
    if (e != cudaSuccess) return e;
    int* nonfinite = reinterpret_cast<int*>(scratch);
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(scratch + 128);
    float* lo = reinterpret_cast<float*>(scratch + 256);
    float* bhi = lo + nsrc;
    float* blo = bhi + nfilt;
    tc_zero_kernel<<<1, 1, 0, st>>>(nonfinite, cnt);
    tc_split_filter_kernel<<<(unsigned)((nfilt + 255) / 256 < 148 * 8 ? (nfilt + 255) / 256 : 148 * 8), 256, 0, st>>>(
        filt, bhi, blo, Co, Cr, sh.R, sh.S, nonfinite);
    tc_split_src_kernel<<<148 * 8, 256, 0, st>>>(src, lo, nsrc / 4, Hs, Ws, Ho, Wo, sh.R, sh.S, sh.padW, sh.padH,
                                                 fwd ? 0 : 1, (unsigned)(Co / 16), (sparse && exec_ctr) ? cnt : nullptr,
                                                 nonfinite);
    note_launch(3);

    TcGeo g;
    g.Ho = Ho;
    g.Wo = Wo;
    choose_box(Ho, Wo, &g.bw, &g.bh);
    g.tiles_x = (Wo + g.bw - 1) / g.bw;
    g.tiles_y = (Ho + g.bh - 1) / g.bh;
    g.Co = Co;
    g.RB = Cr / 16;
    g.R = sh.R;
    g.S = sh.S;
    g.sgn = fwd ? 1 : -1;
    g.padW = sh.padW;
    g.padH = sh.padH;
    g.out_img = (size_t)Co * Ho * Wo;
    // SPC_TC_SEG overrides the segment length (accuracy / speed experiments)
    static const int seg_env = std::getenv("SPC_TC_SEG") ? std::atoi(std::getenv("SPC_TC_SEG")) : 0;
    g.seg = seg_env > 0 ? seg_env : 8;  // error 1.2-1.4e-6 measured

    CUtensorMap mhi, mlo, mbhi, mblo;
    const int bn = Co % 256 == 0 ? 256 : (Co % 128 == 0 ? 128 : 64);
    if (!make_act_map(&mhi, src, sh.N, Cr / 16, Hs, Ws, g.bw, g.bh) ||
        !make_act_map(&mlo, lo, sh.N, Cr / 16, Hs, Ws, g.bw, g.bh) ||
        !make_filter_map(&mbhi, bhi, taps * (Cr / 16), Co, bn) ||
        !make_filter_map(&mblo, blo, taps * (Cr / 16), Co, bn)) {
        cudaFreeAsync(scratch, st);
        return cudaErrorInvalidValue;
    }
    unsigned long long* ex = (sparse && exec_ctr) ? exec_ctr : nullptr;
    if (bn == 256)
        e = launch_bn<256>(mhi, mlo, mbhi, mblo, g, sh.N, dst, nonfinite, cnt, ex, epi, st);
    else if (bn == 128)
        e = launch_bn<128>(mhi, mlo, mbhi, mblo, g, sh.N, dst, nonfinite, cnt, ex, epi, st);
    else
        e = launch_bn<64>(mhi, mlo, mbhi, mblo, g, sh.N, dst, nonfinite, cnt, ex, epi, st);
    // non-finite source or filter: the FFMA tile kernel with the reference's exact skip semantics
    if (e == cudaSuccess) e = launch_tile_conv_when(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi, nonfinite, 1);
    cudaFreeAsync(scratch, st);
    return e;
}

}  // namespace spc
