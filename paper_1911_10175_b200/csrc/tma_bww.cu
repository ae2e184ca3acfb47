// tma_bww.cu -- BWW, check = input, 3x3 stride 1 pad 1, V = 16: the tile
// kernel of tile_bww.cu with both operands staged by TMA.
//
// dG[k,c,v,u] = sum_{i,y',x'} D[i,c,y'+v-1,x'+u-1] * dY[i,k,y',x']
// (P/src/kernel_impl.hpp:209-336, P/src/kernels.cpp:238-302).
//
// Why: in tile_bww.cu every thread stages its share of each (item, image)
// stage with cp.async -- a 4-byte gather out of the 16-image ActCHWNn vectors
// for the checked planes -- and that address arithmetic plus the two CTA
// barriers per image were ~40% of the instructions of a warp step and ~30% of
// its L1 wavefronts (SASS of the production instantiation).  Here:
//   * a pre-pass rewrites the checked tensor from ActCHWNn into per-image
//     planes [N][C][H][Wpitch] (one read + one write of |D|, ~1% of the pass),
//   * one elected thread then stages a whole step with two TMA instructions:
//     a 4-D box of the planes (the halo'd region of the CTA's channels; pixels
//     outside the image are zero-filled = the virtual padding) and a 5-D box of
//     dY straight from ActNCHWc, its dimensions ordered (16, channel block, x,
//     y, image) so the tile lands pixel-major, [pixel][32*KK lane channels],
//   * full / empty mbarriers per stage replace the CTA barriers: warps drift
//     apart by up to NST-1 steps instead of meeting twice per image.
// The per-pixel zero test, the accumulation order inside a step and the
// split reduction are those of tile_bww.cu.
#include "common.cuh"
#include "tc_common.cuh"
#include "pw_bww.h"
#include "tile_bww.h"

#include <cstdlib>

#ifndef SPC_TMA_BWW_FFMA2_MIN
#define SPC_TMA_BWW_FFMA2_MIN SPC_FFMA2_MIN  // FMAs per lane in a pixel block from which the packed form is used
#endif

namespace spc {

using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::smem_u32;
using tc::tma_load_5d;

namespace {

// The spin is one PTX statement: a C++ loop around try_wait makes the
// compiler treat everything after it as possibly diverged (measured: 192
// registers instead of 124 for the same kernel body).
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@p bra D_%=;\n\t"
        "bra W_%=;\n"
        "D_%=:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

// ActCHWNn [NB][C][HW][16 images] -> planes [N][C][H][Wpitch] with pixel x
// stored at column x + 1 and column 0 = 0 (the left padding column): TMA needs
// a 16-byte aligned innermost start, and a region begins at x0 - 1 with x0 a
// multiple of 4 (measured: a misaligned innermost coordinate raises an illegal
// instruction; out-of-bounds ones are fine).  Columns past W are never read:
// the tensor map's x extent is W + 1.
__global__ void __launch_bounds__(256) chwnn_to_planes_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                              int N, int C, int H, int W, int Wpitch,
                                                              const int* __restrict__ sel, int want,
                                                              int* __restrict__ finite_out) {
    // finite_out: this pass is also the finiteness scan of the checked tensor (flag preset to 1,
    // cleared on Inf / NaN) -- it reads every element anyway; it then runs ungated
    if (finite_out == nullptr && sel != nullptr && __ldg(sel) != want) return;
    __shared__ float s[256][17];
    int bad = 0;
    const int HW = H * W;
    const int nb = blockIdx.z, c = blockIdx.y, p0 = blockIdx.x * 256;
    const int npx = HW - p0 < 256 ? HW - p0 : 256;
    const float4* in = reinterpret_cast<const float4*>(src + (((size_t)nb * C + c) * HW + p0) * 16);
    for (int e = threadIdx.x; e < npx * 4; e += 256) {
        const float4 v = __ldg(in + e);
        float* r = &s[e >> 2][(e & 3) * 4];
        r[0] = v.x; r[1] = v.y; r[2] = v.z; r[3] = v.w;
        bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    }
    if (finite_out != nullptr && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(finite_out, 0);
    __syncthreads();
    const int nimg = N - nb * 16 < 16 ? N - nb * 16 : 16;
    if ((int)threadIdx.x < npx) {
        const int p = p0 + threadIdx.x;
        const int y = p / W, x = p - y * W;
        float* o = dst + (((size_t)(nb * 16) * C + c) * H + y) * Wpitch + x + 1;
        const size_t img = (size_t)C * H * Wpitch;
#pragma unroll 4
        for (int j = 0; j < nimg; ++j) o[j * img] = s[threadIdx.x][j];
        if (x == 0) {
            for (int j = 0; j < nimg; ++j) o[j * img - 1] = 0.0f;
        }
    }
}

template <int KK, int CB, int NWC, int TH, int TW, int NSTAGE = 4>
struct TGeom {
    static constexpr int TAPS = 9;
    static constexpr int CRH = TH + 2, CRW = TW + 2;
    // the staged box starts at plane column (x0 & ~3) (= pixel x0 - 1 when x0 % 4 == 0)
    static constexpr int XOFF_MAX = (TW % 4 == 0) ? 0 : 4 - (TW % 4 == 2 ? 2 : 1);
    static constexpr int NQ = (CRW + XOFF_MAX + 3) / 4;
    static constexpr int CRWP = NQ * 4;
    static constexpr int PLANE = CRH * CRWP;
    static constexpr int CHW = CRH * CRW;
    static constexpr int NWORD = (CHW + 31) / 32;
    static constexpr int NCH = NWC * CB;
    static constexpr int NT = NWC * 32;
    static constexpr int NST = NSTAGE;
    static constexpr int OBYTES = TH * TW * 32 * KK * 4;
    static constexpr int CBYTES = NCH * PLANE * 4;
    static constexpr int CBYTES_PAD = (CBYTES + 127) / 128 * 128;
    static constexpr int STAGE = OBYTES + CBYTES_PAD;
    static constexpr int SMEM = NST * STAGE + 2 * NST * 8;  // + full / empty barriers
};

template <int KK, int CB, int NWC, int TH, int TW, int MINB, bool SPARSE, int NSTAGE = 4>
__global__ void __launch_bounds__(NWC * 32, MINB)
    tma_bww_kernel(const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapY, DevShape sh,
                   float* __restrict__ partial, int splits, unsigned long long* __restrict__ exec_ctr,
                   const int* __restrict__ sel, int want) {
    static_assert(NWC <= 15, "one named barrier (ids 1..15) per warp");
    using G = TGeom<KK, CB, NWC, TH, TW, NSTAGE>;
    if (sel != nullptr && __ldg(sel) != want) return;
    constexpr int TAPS = G::TAPS, CRH = G::CRH, CRW = G::CRW, CRWP = G::CRWP, PLANE = G::PLANE;
    constexpr int CHW = G::CHW, NWORD = G::NWORD, NCH = G::NCH, NST = G::NST;

    extern __shared__ __align__(1024) uint8_t smem[];  // no static shared memory in this kernel: offset 0
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bars = sbase + NST * G::STAGE;  // full[NST], empty[NST]
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (NST + s); };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mc0 = blockIdx.x * NCH;      // first checked (input) channel of the CTA
    const int lc0 = blockIdx.y * 32 * KK;  // first lane (output) channel of the CTA
    const int l0 = lc0 + lane * KK;

    const int tiles_x = (sh.Wp + TW - 1) / TW;
    const int ntiles = tiles_x * ((sh.Hp + TH - 1) / TH);
    const int items = ntiles * sh.N;  // step = (tile, image), image fastest
    const int it0 = (int)((long)items * blockIdx.z / splits), it1 = (int)((long)items * (blockIdx.z + 1) / splits);

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), NWC);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    float acc[CB][TAPS][KK];
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int f = 0; f < TAPS; ++f)
#pragma unroll
            for (int j = 0; j < KK; ++j) acc[a][f][j] = 0.0f;

    // producer cursor (thread 0): the step whose loads are issued next
    int pt = it0 / sh.N, pn = it0 - pt * sh.N, pit = it0;
    auto issue = [&](int li) {  // li = local index of step `pit`
        const int s = li % NST;
        const int y0 = (pt / tiles_x) * TH, x0 = (pt % tiles_x) * TW;
        const uint32_t dst = sbase + s * G::STAGE;
        mbar_expect_tx(full_bar(s), G::OBYTES + G::CBYTES);
        tma_load_5d(dst, &mapY, full_bar(s), 0, lc0 / 16, x0, y0, pn);
        tma_load_4d(dst + G::OBYTES, &mapD, full_bar(s), x0 & ~3, y0 - 1, mc0, pn);
        ++pit;
        if (++pn == sh.N) {
            pn = 0;
            ++pt;
        }
    };
    if (threadIdx.x == 0) {
        for (int d = 0; d < NST - 1 && pit < it1; ++d) issue(d);
    }

    // lane pixel offsets inside a plane (fixed for every step)
    int qoff[NWORD];
#pragma unroll
    for (int w = 0; w < NWORD; ++w) {
        const int q = lane + 32 * w;
        qoff[w] = q < CHW ? (q / CRW) * CRWP + q % CRW : 0;
    }
    uint32_t cnt = 0;
    uint32_t wt[NWORD];
    int ct = it0 / sh.N, cn = it0 - ct * sh.N;  // consumer cursor
    bool fresh = true;
    int xoff = 0;  // column of pixel x0 - 1 inside the staged box (0 when TW % 4 == 0)

#pragma unroll 1
    for (int it = it0; it < it1; ++it) {
        const int li = it - it0;
        const int s = li % NST;
        if (threadIdx.x == 0 && pit < it1) {
            // the stage refilled now was read by local step li - 1
            if (li >= 1) mbar_wait(empty_bar((li - 1) % NST), ((li - 1) / NST) & 1);
            issue(li + NST - 1);
        }
        if (fresh) {
            // valid (tap, output pixel) pairs of this lane's checked pixels, for counting
            const int y0 = (ct / tiles_x) * TH, x0 = (ct % tiles_x) * TW;
#pragma unroll
            for (int w = 0; w < NWORD; ++w) {
                const int q = lane + 32 * w;
                uint32_t ny = 0, nx = 0;
                if (q < CHW) {
                    const int ry = q / CRW, rx = q % CRW;
#pragma unroll
                    for (int v = 0; v < 3; ++v) {
                        const int num = ry - v;
                        if (num >= 0 && num < TH && y0 + num < sh.Hp) ++ny;
                    }
#pragma unroll
                    for (int u = 0; u < 3; ++u) {
                        const int num = rx - u;
                        if (num >= 0 && num < TW && x0 + num < sh.Wp) ++nx;
                    }
                }
                wt[w] = ny * nx;
            }
            if constexpr (TW % 4 != 0) xoff = x0 & 3;
            fresh = false;
        }
        if (++cn == sh.N) {
            cn = 0;
            ++ct;
            fresh = true;
        }
        mbar_wait(full_bar(s), (li / NST) & 1);
        // a warp-wide aligned barrier: tells ptxas the warp is converged after the
        // spin (without it the ballots compile to BRA.DIV paths and 194 registers)
        asm volatile("barrier.sync.aligned %0, 32;" ::"r"(warp + 1) : "memory");

        const float* base = reinterpret_cast<const float*>(smem + s * G::STAGE);
#ifdef SPC_TMA_NOCOMP  // probe: the staging pipeline alone (results are wrong)
        if (sh.N > 0) {
            acc[0][0][0] += base[lane];
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_bar(s));
            continue;
        }
#endif
        float O[TH * TW][KK];
        const float* Ob = base + lane * KK;
#pragma unroll
        for (int q = 0; q < TH * TW; ++q) {
            if constexpr (KK == 4) {
                const float4 t = *reinterpret_cast<const float4*>(Ob + q * 32 * KK);
                O[q][0] = t.x; O[q][1] = t.y; O[q][2] = t.z; O[q][3] = t.w;
            } else {
                const float2 t = *reinterpret_cast<const float2*>(Ob + q * 32 * KK);
                O[q][0] = t.x; O[q][1] = t.y;
            }
        }
        const float* Cb = base + G::OBYTES / 4;
#pragma unroll
        for (int cc = 0; cc < CB; ++cc) {
            const float* Pl = Cb + (warp * CB + cc) * PLANE + xoff;
            uint32_t m[NWORD];
            if (SPARSE) {
#pragma unroll
                for (int w = 0; w < NWORD; ++w) {
                    const float v = (lane + 32 * w < CHW) ? Pl[qoff[w]] : 0.0f;
                    const bool nz = v != 0.0f;
                    cnt += nz ? wt[w] : 0u;
                    m[w] = __ballot_sync(0xffffffffu, nz);
#if defined(TRY_MV1)
                    asm volatile("mov.b32 %0, %0;" : "+r"(m[w]));
#elif defined(TRY_MV2)
                    m[w] = __shfl_sync(0xffffffffu, m[w], 0);
#endif
                }
            }
            // region rows as broadcast vector loads, one row ahead (16-byte vectors; 8-byte
            // when the tile width leaves the region start only 8-byte aligned)
            constexpr int VW = (TW % 4 == 0) ? 4 : 2;
            constexpr int NV = (CRW + VW - 1) / VW;
            float cur[NV * VW], nxt[NV * VW];
            auto load_row = [&](float (&r)[NV * VW], int ry) {
#pragma unroll
                for (int h = 0; h < NV; ++h) {
                    if constexpr (VW == 4) {
                        const float4 t = *reinterpret_cast<const float4*>(Pl + ry * CRWP + 4 * h);
                        r[4 * h] = t.x; r[4 * h + 1] = t.y; r[4 * h + 2] = t.z; r[4 * h + 3] = t.w;
                    } else {
                        const float2 t = *reinterpret_cast<const float2*>(Pl + ry * CRWP + 2 * h);
                        r[2 * h] = t.x; r[2 * h + 1] = t.y;
                    }
                }
            };
            load_row(cur, 0);
#pragma unroll
            for (int ry = 0; ry < CRH; ++ry) {
                if (ry + 1 < CRH) load_row(nxt, ry + 1);
#pragma unroll
                for (int rx = 0; rx < CRW; ++rx) {
                    const int p = ry * CRW + rx;
                    if (!SPARSE || ((m[p >> 5] >> (p & 31)) & 1u)) {
                        const float d = cur[rx];
                        int ntap = 0;  // folds to a constant per unrolled pixel
#pragma unroll
                        for (int v = 0; v < 3; ++v)
#pragma unroll
                            for (int u = 0; u < 3; ++u) {
                                const int ny = ry - v, nx = rx - u;
                                ntap += !(ny < 0 || nx < 0 || ny >= TH || nx >= TW);
                            }
#pragma unroll
                        for (int v = 0; v < 3; ++v) {
#pragma unroll
                            for (int u = 0; u < 3; ++u) {
                                const int ny = ry - v, nx = rx - u;
                                if (ny < 0 || nx < 0 || ny >= TH || nx >= TW) continue;
                                fma_lane<KK, SPC_TMA_BWW_FFMA2_MIN>(acc[cc][v * 3 + u], d, O[ny * TW + nx], ntap);
                            }
                        }
                    }
                }
                if (ry + 1 < CRH) {
#pragma unroll
                    for (int h = 0; h < NV * VW; ++h) cur[h] = nxt[h];
                }
            }
        }
        // generic-proxy reads of this stage (the LDS above) must be ordered before the async-proxy
        // TMA write that refills it: the empty barrier's release does not cross proxies
        // (tma_pw_bww.cu measured the race on short steps; same protocol here)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(s));
    }

    // partial[z][c][tap][k]: warps own disjoint checked channels
    float* pz = partial + (size_t)blockIdx.z * sh.C * TAPS * sh.K;
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int f = 0; f < TAPS; ++f) {
            float* dstp = pz + ((size_t)(mc0 + warp * CB + a) * TAPS + f) * sh.K + l0;
            if constexpr (KK == 4) {
                *reinterpret_cast<float4*>(dstp) = make_float4(acc[a][f][0], acc[a][f][1], acc[a][f][2], acc[a][f][3]);
            } else {
                *reinterpret_cast<float2*>(dstp) = make_float2(acc[a][f][0], acc[a][f][1]);
            }
        }
    if (SPARSE && exec_ctr) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (2 * KK));
    }
}

// Sum the splits in fixed order and scatter into FilterKCRSblk (K, C).
__global__ void tma_bww_reduce(DevShape sh, const float* __restrict__ partial, int splits, float* __restrict__ dst,
                               const int* __restrict__ sel, int want) {
    if (sel != nullptr && __ldg(sel) != want) return;
    const size_t E = (size_t)sh.C * 9 * sh.K;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < E; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int z = 0; z < splits; ++z) s += partial[(size_t)z * E + e];
        const int k = (int)(e % sh.K);
        const int f = (int)((e / sh.K) % 9);
        const int c = (int)(e / ((size_t)sh.K * 9));
        dst[filter_index(sh.C, 3, 3, 16, k, c, f % 3, f / 3)] = s;
    }
}

template <int KK, int CB, int NWC, int TH, int TW, int MINB, int NSTAGE = 4>
cudaError_t launch_cfg(bool sparse, const DevShape& sh, const float* chk, const float* oth, float* dst,
                       unsigned long long* exec_ctr, const int* sel, int want, cudaStream_t st, int* scan_flag) {
    using G = TGeom<KK, CB, NWC, TH, TW, NSTAGE>;
    if (!tc::encode_fn()) return cudaErrorNotSupported;
    const int Wpitch = (sh.W + 1 + 3) / 4 * 4;
    const size_t plane_floats = (size_t)sh.N * sh.C * sh.H * Wpitch;
    const long items = (long)sh.N * ((sh.Wp + TW - 1) / TW) * ((sh.Hp + TH - 1) / TH);
    const long base = (long)(sh.C / G::NCH) * (sh.K / (32 * KK));
    static const long env_ctas = std::getenv("SPC_BWW_CTAS") ? std::atol(std::getenv("SPC_BWW_CTAS")) : 0;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long target_ctas = env_ctas > 0 ? env_ctas : (base >= 16 && base <= 128) ? nsm * 18L : nsm * 6L;
    long splits = (target_ctas + base - 1) / base;
    static const bool wave_off = std::getenv("SPC_BWW_WAVE") && std::atoi(std::getenv("SPC_BWW_WAVE")) == 0;
    if (env_ctas <= 0 && !wave_off && base <= 128) {
        // wave quantisation (the many-wave shapes): among the split counts within -25% / +10%
        // of the target, take the one whose grid fills its last wave best (MINB CTAs per SM;
        // conv3_2: 42 splits = 9.08 waves -> 37 splits = 8.00 waves).  Measured 3-4% faster on
        // VGG conv2_2 .. conv4_1; the few-wave shapes (base > 128) lose 8-10% with fewer
        // splits and keep the plain target.
        const long slots = (long)nsm * MINB;
        long best = splits;
        double best_eff = 0.0;
        for (long s = splits * 3 / 4 > 0 ? splits * 3 / 4 : 1; s <= splits + splits / 10; ++s) {
            const long g = base * s;
            const double eff = (double)g / (double)(((g + slots - 1) / slots) * slots);
            if (eff >= best_eff - 1e-9) {  // ties: the larger grid
                best_eff = eff;
                best = s;
            }
        }
        splits = best;
    }
    if (splits > items) splits = items;
    const size_t E = (size_t)sh.C * 9 * sh.K;
    const long cap = (long)((256ull << 20) / (E * sizeof(float)));
    if (splits > cap) splits = cap;
    if (splits < 1) splits = 1;

    float* planes = nullptr;
    float* partial = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&planes, plane_floats * sizeof(float), st);
    if (e != cudaSuccess) return e;
    e = cudaMallocAsync((void**)&partial, (size_t)splits * E * sizeof(float), st);
    if (e != cudaSuccess) {
        cudaFreeAsync(planes, st);
        return e;
    }
    const int HW = sh.H * sh.W;
    if (scan_flag != nullptr) launch_set_flag(scan_flag, st);
    chwnn_to_planes_kernel<<<dim3((HW + 255) / 256, sh.C, (sh.N + 15) / 16), 256, 0, st>>>(chk, planes, sh.N, sh.C,
                                                                                             sh.H, sh.W, Wpitch, sel,
                                                                                             want, scan_flag);
    note_launch();

    CUtensorMap mapD, mapY;
    bool ok = true;
    {
        cuuint64_t dims[4] = {(cuuint64_t)sh.W + 1, (cuuint64_t)sh.H, (cuuint64_t)sh.C, (cuuint64_t)sh.N};
        cuuint64_t strides[3] = {(cuuint64_t)Wpitch * 4, (cuuint64_t)sh.H * Wpitch * 4,
                                 (cuuint64_t)sh.C * sh.H * Wpitch * 4};
        cuuint32_t box[4] = {(cuuint32_t)G::CRWP, (cuuint32_t)G::CRH, (cuuint32_t)G::NCH, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        ok = ok && tc::encode_fn()(&mapD, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, planes, dims, strides, box, es,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    {
        // dY ActNCHWc [N][K/16][Hp][Wp][16] with the dimensions ordered (16, channel block, x, y, image)
        const cuuint64_t hw = (cuuint64_t)sh.Hp * sh.Wp;
        cuuint64_t dims[5] = {16, (cuuint64_t)(sh.K / 16), (cuuint64_t)sh.Wp, (cuuint64_t)sh.Hp, (cuuint64_t)sh.N};
        cuuint64_t strides[4] = {hw * 64, 64, (cuuint64_t)sh.Wp * 64, (cuuint64_t)(sh.K / 16) * hw * 64};
        cuuint32_t box[5] = {16, (cuuint32_t)(2 * KK), (cuuint32_t)TW, (cuuint32_t)TH, 1};
        cuuint32_t es[5] = {1, 1, 1, 1, 1};
        ok = ok && tc::encode_fn()(&mapY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(oth), dims, strides,
                                   box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (!ok) {
        cudaFreeAsync(planes, st);
        cudaFreeAsync(partial, st);
        return cudaErrorInvalidValue;
    }
    dim3 grid(sh.C / G::NCH, sh.K / (32 * KK), (unsigned)splits);
    auto kern = sparse ? tma_bww_kernel<KK, CB, NWC, TH, TW, MINB, true, NSTAGE>
                       : tma_bww_kernel<KK, CB, NWC, TH, TW, MINB, false, NSTAGE>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
    kern<<<grid, G::NT, G::SMEM, st>>>(mapD, mapY, sh, partial, (int)splits, exec_ctr, sel, want);
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        unsigned rb = (unsigned)((E + 255) / 256);
        if (rb > 148 * 8) rb = 148 * 8;
        tma_bww_reduce<<<rb, 256, 0, st>>>(sh, partial, (int)splits, dst, sel, want);
        note_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(planes, st);
    cudaFreeAsync(partial, st);
    return e;
}

#ifdef SPC_DEV
// tuning variants (tools/bww_ab.py; DESIGN.md 4.2 has the measurements)
int tma_cfg() {
    static const int v = std::getenv("SPC_TMA_BWW_CFG") ? std::atoi(std::getenv("SPC_TMA_BWW_CFG")) : 0;
    return v;
}
#endif

}  // namespace

bool tma_bww_supported(bool check_input, const DevShape& sh, int V) {
    if (V != 16 || !check_input) return false;
    if (sh.R != 3 || sh.S != 3 || sh.O != 1 || sh.P != 1 || sh.padW != 1 || sh.padH != 1) return false;
#ifdef SPC_DEV
    if (sh.K % 64 || sh.C % 16) return false;
#else
    if (sh.K % 128 || sh.C % 16) return false;
#endif
    // TMA extents: strides below 2^40 bytes, coordinates in int
    if ((size_t)sh.N * sh.C * sh.H * sh.W >= (1ull << 32)) return false;
    return tc::encode_fn() != nullptr;
}

cudaError_t launch_tma_bww_when(bool sparse, const DevShape& sh, const float* chk, const float* oth, float* dst,
                                unsigned long long* exec_ctr, const int* sel, int want, cudaStream_t st,
                                int* scan_flag) {
#ifdef SPC_DEV
    if (sh.K % 128 != 0) {  // 64-channel lane blocks: KK = 2
        switch (tma_cfg()) {
        case 11: return launch_cfg<2, 2, 8, 7, 4, 2>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
        case 12: return launch_cfg<2, 2, 4, 7, 4, 4>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
        case 13: return launch_cfg<2, 4, 4, 7, 4, 3>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
        default: return launch_cfg<2, 1, 8, 7, 4, 2>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
        }
    }
    switch (tma_cfg()) {
    case 1: return launch_cfg<4, 2, 4, 7, 2, 3>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 2: return launch_cfg<4, 2, 4, 7, 4, 2>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 3: return launch_cfg<4, 1, 8, 7, 2, 2>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 4: return launch_cfg<4, 2, 8, 7, 2, 1>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 5: return launch_cfg<4, 1, 4, 7, 4, 4>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 7: return launch_cfg<4, 1, 8, 7, 2, 3>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 8: return launch_cfg<4, 1, 8, 7, 4, 2, 6>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    case 9: return launch_cfg<4, 1, 8, 7, 4, 2, 3>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
    default: break;
    }
#endif
    // KK = 4 lane channels per lane, one checked channel per warp, 8 warps, 7x4 tile, 2 CTAs / SM
    return launch_cfg<4, 1, 8, 7, 4, 2>(sparse, sh, chk, oth, dst, exec_ctr, sel, want, st, scan_flag);
}

}  // namespace spc
