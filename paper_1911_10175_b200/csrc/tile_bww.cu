// tile_bww.cu -- tuned sm_100a BWW kernels for V = 16 blocked layouts.
//
// dG[k,c,v,u] = sum_{i,y',x'} D[i,c,y'P+v-padH, x'O+u-padW] * dY[i,k,y',x']
// (P/src/kernel_impl.hpp:209-336, P/src/kernels.cpp:238-302).
//
// The checked tensor arrives in ActCHWNn ([N/16][C][H][W][16 images]) as the
// reference's API requires.  A CTA of NWC warps owns one output-pixel tile,
// 32*KK lane channels (the OTHER tensor's channels, KK per lane) and NWC*CB
// checked channels (CB per warp).  The checked region of those channels is
// staged in shared memory with 4-byte cp.async that transposes the 16-image
// vectors into per-(channel, image) pixel planes, so for one image:
//   * one conflict-free lane load + __ballot_sync gives the nonzero mask of 32
//     region pixels (warp-uniform: every lane consumes the same checked value,
//     `d != 0.0f`, -0 is zero and NaN is not, P/include/spconv/vec.hpp:120-128);
//   * each region row's values arrive by broadcast 128-bit loads, one row ahead
//     of the uniform branches that skip the FMAs a zero would have fed.
// The other operand's pixel tile for the current image sits in registers and
// is reused by all CB channels x R*S taps of the warp; the NWC warps load the
// same tile, so L1 serves all but the first.  Accumulators (CB x R*S x KK) are
// register-resident for the whole reduction -- no per-FMA reloads (the CPU
// BWW's bottleneck).
//
// check = input:       checked = D  (input pixels, halo'd region), other = dY tile
// check = output_grad: checked = dY (output tile),                  other = D region
//
// The reduction over images and pixels is split over CTAs (fixed item ranges);
// bww_tile_reduce sums the splits in fixed order: bitwise deterministic, no
// float atomics.  The final store writes FilterKCRSblk (K, C) for either check
// side, i.e. the reference's check=output_grad transpose (kernels.cpp:285-300)
// is fused into the reduction.
#include "common.cuh"
#include "jt_blocks.cuh"
#include "tile_bww.h"

namespace spc {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int KK>
__device__ __forceinline__ void ld_vec(float (&o)[KK], const float* p) {
    if constexpr (KK == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        o[0] = t.x; o[1] = t.y; o[2] = t.z; o[3] = t.w;
    } else if constexpr (KK == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        o[0] = t.x; o[1] = t.y;
    } else {
        o[0] = __ldg(p);
    }
}

}  // namespace

template <bool CHECK_INPUT, int KK, int CB, int NWC, int TH, int TW, int R, int S, int STR>
struct BwwGeom {
    static constexpr int PADH = (S - 1) / 2, PADW = (R - 1) / 2;
    static constexpr int TAPS = R * S;
    static constexpr int IRH = (TH - 1) * STR + S;  // input-pixel region of the output tile
    static constexpr int IRW = (TW - 1) * STR + R;
    static constexpr int CRH = CHECK_INPUT ? IRH : TH;  // checked region
    static constexpr int CRW = CHECK_INPUT ? IRW : TW;
    static constexpr int NQ = (CRW + 3) / 4;
    static constexpr int CRWP = NQ * 4;
    static constexpr int PLANE = CRH * CRWP;          // one (channel, image) plane
    static constexpr int CHW = CRH * CRW;
    static constexpr int NWORD = (CHW + 31) / 32;
    static constexpr int OTH = CHECK_INPUT ? TH : IRH;  // other-operand register tile
    static constexpr int OTW = CHECK_INPUT ? TW : IRW;
    static constexpr int NCH = NWC * CB;               // checked channels per CTA
    static constexpr int NT = NWC * 32;
    static constexpr int NST = 4;                      // pipeline stages (one image each)
    static constexpr int CFLOATS = NCH * PLANE;         // checked planes of one image
    static constexpr int OFLOATS = OTH * OTW * 32 * KK;  // other tile of one image
    static constexpr int STAGE = CFLOATS + OFLOATS;
    static constexpr int SMEM = NST * STAGE * 4;
};

// Static loop over the 32-pixel mask words of the jump-table path.
template <int W, int NW, class JB, class Acc, class Ov>
__device__ __forceinline__ void bww_jt_words(Acc& acc, const Ov& O, const float* vv, const uint32_t* m) {
    if constexpr (W < NW) {
        if (m[W]) JB::template Word<W>::run(acc, O, vv[W], m[W]);
        bww_jt_words<W + 1, NW, JB>(acc, O, vv, m);
    }
}

// JT = 100: jump-table dispatch over the nonzero checked pixels only
// (jt_blocks.cuh, generated); 0: one uniform branch per checked pixel; 200:
// "counted dense" -- every pixel's FMAs run while the ballots still count
// (stride 2: a checked pixel feeds ~2.25 taps, too few for a branch to pay;
// finite operands only, the dispatcher guards).  Same accumulation order in
// all three.  `sel`/`want`: device-side kernel choice.
template <bool CHECK_INPUT, int KK, int CB, int NWC, int TH, int TW, int R, int S, int STR, int JT, bool SPARSE>
__global__ void __launch_bounds__(NWC * 32) bww_tile_kernel(DevShape sh, const float* __restrict__ chk,
                                                            const float* __restrict__ oth,
                                                            float* __restrict__ partial, int splits,
                                                            unsigned long long* __restrict__ exec_ctr,
                                                            const int* __restrict__ sel, int want) {
    using G = BwwGeom<CHECK_INPUT, KK, CB, NWC, TH, TW, R, S, STR>;
    if (sel != nullptr && __ldg(sel) != want) return;
    constexpr int TAPS = G::TAPS, CRH = G::CRH, CRW = G::CRW, CRWP = G::CRWP, PLANE = G::PLANE;
    constexpr int CHW = G::CHW, NWORD = G::NWORD, NQ = G::NQ, OTH = G::OTH, OTW = G::OTW, NCH = G::NCH;

    extern __shared__ __align__(16) float smem[];  // NST x {checked [NCH][CRH][CRWP], other [OTH*OTW][32*KK]}

    const int Lc = CHECK_INPUT ? sh.K : sh.C;  // lane channels (other tensor)
    const int Mc = CHECK_INPUT ? sh.C : sh.K;  // checked channels
    const int Hc = CHECK_INPUT ? sh.H : sh.Hp, Wc = CHECK_INPUT ? sh.W : sh.Wp;  // checked dims
    const int Ho = CHECK_INPUT ? sh.Hp : sh.H, Wo = CHECK_INPUT ? sh.Wp : sh.W;  // other dims
    const int LcB = Lc / 16;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mc0 = blockIdx.x * NCH;        // first checked channel of the CTA
    const int lc0 = blockIdx.y * 32 * KK;    // first lane channel of the CTA
    const int l0 = lc0 + lane * KK;          // this lane's first lane channel

    const int tiles_x = (sh.Wp + TW - 1) / TW;
    const int ntiles = tiles_x * ((sh.Hp + TH - 1) / TH);
    const int nb = (sh.N + 15) / 16;
    const int items = nb * ntiles;
    const int it0 = (int)((long)items * blockIdx.z / splits), it1 = (int)((long)items * (blockIdx.z + 1) / splits);

    float acc[CB][TAPS][KK];
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int f = 0; f < TAPS; ++f)
#pragma unroll
            for (int j = 0; j < KK; ++j) acc[a][f][j] = 0.0f;

    auto origin = [&](int it, int& ib, int& y0, int& x0) {
        ib = (int)(it / ntiles);
        const int t = (int)(it % ntiles);
        y0 = (t / tiles_x) * TH;
        x0 = (t % tiles_x) * TW;
    };
    const int nlast = sh.N - (nb - 1) * 16;  // images in the last (possibly ragged) block
    auto nimg_of = [&](int it) { return it >= (nb - 1) * ntiles ? nlast : 16; };

    // One pipeline stage = one (item, image): the checked planes of that image
    // (4-byte cp.async out of the 16-image CHWNn vectors; .ca keeps the lines in
    // L1 for the item's other images) and the other operand's pixel tile
    // ([pixel][32*KK lane channels], 16-byte cp.async).  Each thread's element
    // descriptors (global offset without the image term, smem offset, valid)
    // are computed once per item.
    constexpr int NCE = (NCH * CRH * CRW + NWC * 32 - 1) / (NWC * 32);
    constexpr int NOE = (OTH * OTW * 8 * KK + NWC * 32 - 1) / (NWC * 32);
    uint32_t cgo[NCE], cso[NCE], ogo[NOE];
    uint32_t cvalid = 0, ovalid = 0;
    const size_t ostride_img = (size_t)LcB * Ho * Wo * 16;
    auto describe = [&](int it) {
        int ib, y0, x0;
        origin(it, ib, y0, x0);
        const int cy0 = CHECK_INPUT ? y0 * STR - G::PADH : y0;
        const int cx0 = CHECK_INPUT ? x0 * STR - G::PADW : x0;
        cvalid = 0;
#pragma unroll
        for (int e = 0; e < NCE; ++e) {
            const int idx = threadIdx.x + e * NWC * 32;
            const int rx = idx % CRW, ry = (idx / CRW) % CRH, cc = idx / (CRW * CRH);
            const int gy = cy0 + ry, gx = cx0 + rx;
            const bool ok = idx < NCH * CRH * CRW && gy >= 0 && gy < Hc && gx >= 0 && gx < Wc;
            cgo[e] = ok ? (uint32_t)(((((size_t)ib * Mc + mc0 + cc) * Hc + gy) * Wc + gx) * 16) : 0u;
            cso[e] = (uint32_t)(cc * PLANE + ry * CRWP + rx) * 4u;
            cvalid |= (ok ? 1u : 0u) << e;
        }
        const int oy0 = CHECK_INPUT ? y0 : y0 * STR - G::PADH;
        const int ox0 = CHECK_INPUT ? x0 : x0 * STR - G::PADW;
        ovalid = 0;
#pragma unroll
        for (int e = 0; e < NOE; ++e) {
            const int idx = threadIdx.x + e * NWC * 32;
            const int c4 = idx % (8 * KK), q = idx / (8 * KK);
            const int gy = oy0 + q / OTW, gx = ox0 + q % OTW;
            const int ch = lc0 + c4 * 4;
            const bool ok = idx < OTH * OTW * 8 * KK && gy >= 0 && gy < Ho && gx >= 0 && gx < Wo;
            ogo[e] = ok ? (uint32_t)((((size_t)(ib * 16) * LcB + ch / 16) * Ho * Wo + (size_t)gy * Wo + gx) * 16 +
                                     (ch % 16))
                        : 0u;
            ovalid |= (ok ? 1u : 0u) << e;
        }
    };
    auto stage = [&](int j, int buf) {
        float* base = smem + buf * G::STAGE;
        const uint32_t dc = smem_u32(base);
#pragma unroll
        for (int e = 0; e < NCE; ++e) {
            const int idx = threadIdx.x + e * NWC * 32;
            if (idx < NCH * CRH * CRW) {
                const bool ok = (cvalid >> e) & 1u;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dc + cso[e]),
                             "l"(chk + cgo[e] + (ok ? j : 0)), "r"(ok ? 4 : 0));
            }
        }
        const uint32_t doo = smem_u32(base + G::CFLOATS);
#pragma unroll
        for (int e = 0; e < NOE; ++e) {
            const int idx = threadIdx.x + e * NWC * 32;
            if (idx < OTH * OTW * 8 * KK) {
                const bool ok = (ovalid >> e) & 1u;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(doo + (uint32_t)idx * 16u),
                             "l"(oth + ogo[e] + (ok ? (size_t)j * ostride_img : 0)), "r"(ok ? 16 : 0));
            }
        }
    };

    // lane pixel offsets inside a plane (fixed for every item)
    int qoff[NWORD];
#pragma unroll
    for (int w = 0; w < NWORD; ++w) {
        const int q = lane + 32 * w;
        qoff[w] = q < CHW ? (q / CRW) * CRWP + q % CRW : 0;
    }
    uint32_t cnt = 0;

    // prefetch cursor runs NST-1 stages ahead of the consumer
    int pit = it0;
    int pj = 0;
    if (pit < it1) describe(pit);
    auto advance = [&]() {
        if (++pj >= nimg_of(pit)) {
            pj = 0;
            if (++pit < it1) describe(pit);
        }
    };
    for (int d = 0; d < G::NST - 1; ++d) {
        if (pit < it1) {
            stage(pj, d);
            advance();
        }
        cp_async_commit();
    }
    int sbuf = G::NST - 1;  // stage buffer the next prefetch fills
    int cbufi = 0;          // stage buffer the consumer reads
    for (int it = it0; it < it1; ++it) {
        int ib, y0, x0;
        origin(it, ib, y0, x0);
        const int nimg = nimg_of(it);

        // valid (tap, partner) weight of this lane's checked pixels, for counting
        uint32_t wt[NWORD];
#pragma unroll
        for (int w = 0; w < NWORD; ++w) {
            const int q = lane + 32 * w;
            uint32_t ny = 0, nx = 0;
            if (q < CHW) {
                const int ry = q / CRW, rx = q % CRW;
                if (CHECK_INPUT) {  // (tap, output pixel) pairs with the output inside the image
#pragma unroll
                    for (int v = 0; v < S; ++v) {
                        const int num = ry - v;
                        if (num >= 0 && num % STR == 0 && num / STR < TH && y0 + num / STR < sh.Hp) ++ny;
                    }
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int num = rx - u;
                        if (num >= 0 && num % STR == 0 && num / STR < TW && x0 + num / STR < sh.Wp) ++nx;
                    }
                } else if (y0 + ry < sh.Hp && x0 + rx < sh.Wp) {  // taps whose input pixel is inside
#pragma unroll
                    for (int v = 0; v < S; ++v) {
                        const int y = (y0 + ry) * STR + v - G::PADH;
                        if (y >= 0 && y < sh.H) ++ny;
                    }
#pragma unroll
                    for (int u = 0; u < R; ++u) {
                        const int x = (x0 + rx) * STR + u - G::PADW;
                        if (x >= 0 && x < sh.W) ++nx;
                    }
                }
            }
            wt[w] = ny * nx;
        }

#pragma unroll 1
        for (int j = 0; j < nimg; ++j) {
            if (pit < it1) {
                stage(pj, sbuf);
                advance();
            }
            cp_async_commit();
            cp_async_wait<G::NST - 1>();
            __syncthreads();

            const float* base = smem + cbufi * G::STAGE;
            float O[OTH * OTW][KK];
            const float* Ob = base + G::CFLOATS + lane * KK;
#pragma unroll
            for (int q = 0; q < OTH * OTW; ++q) {
                if constexpr (KK == 4) {
                    const float4 t = *reinterpret_cast<const float4*>(Ob + q * 32 * KK);
                    O[q][0] = t.x; O[q][1] = t.y; O[q][2] = t.z; O[q][3] = t.w;
                } else if constexpr (KK == 2) {
                    const float2 t = *reinterpret_cast<const float2*>(Ob + q * 32 * KK);
                    O[q][0] = t.x; O[q][1] = t.y;
                } else {
                    O[q][0] = Ob[q * 32 * KK];
                }
            }
#pragma unroll
            for (int cc = 0; cc < CB; ++cc) {
                const float* Pl = base + (warp * CB + cc) * PLANE;
                uint32_t m[NWORD];
                float vv[NWORD];
                if (SPARSE) {
#pragma unroll
                    for (int w = 0; w < NWORD; ++w) {
                        vv[w] = (lane + 32 * w < CHW) ? Pl[qoff[w]] : 0.0f;
                        const bool nz = vv[w] != 0.0f;
                        cnt += nz ? wt[w] : 0u;
                        m[w] = __ballot_sync(0xffffffffu, nz);
                    }
                }
                using JB = BwwJtBlocks<CHECK_INPUT, KK, TH, TW, R, S, STR>;
                if constexpr (SPARSE && JT == 100 && JB::available) {
                    bww_jt_words<0, NWORD, JB>(acc[cc], O, vv, m);
                } else {
                float4 cur[NQ], nxt[NQ];
#pragma unroll
                for (int h = 0; h < NQ; ++h) cur[h] = *reinterpret_cast<const float4*>(Pl + 4 * h);
#pragma unroll
                for (int ry = 0; ry < CRH; ++ry) {
                    if (ry + 1 < CRH) {
#pragma unroll
                        for (int h = 0; h < NQ; ++h)
                            nxt[h] = *reinterpret_cast<const float4*>(Pl + (ry + 1) * CRWP + 4 * h);
                    }
#pragma unroll
                    for (int rx = 0; rx < CRW; ++rx) {
                        const int p = ry * CRW + rx;
                        if (!SPARSE || JT == 200 || ((m[p >> 5] >> (p & 31)) & 1u)) {
                            const float4 q4 = cur[rx >> 2];
                            const float d =
                                (rx & 3) == 0 ? q4.x : (rx & 3) == 1 ? q4.y : (rx & 3) == 2 ? q4.z : q4.w;
                            int ntap = 0;  // folds to a constant per unrolled pixel
#pragma unroll
                            for (int v = 0; v < S; ++v)
#pragma unroll
                                for (int u = 0; u < R; ++u) {
                                    const int ny = ry - v, nx = rx - u;
                                    ntap += !CHECK_INPUT || !(ny < 0 || nx < 0 || ny % STR || nx % STR ||
                                                              ny / STR >= TH || nx / STR >= TW);
                                }
#pragma unroll
                            for (int v = 0; v < S; ++v) {
#pragma unroll
                                for (int u = 0; u < R; ++u) {
                                    int q;
                                    if (CHECK_INPUT) {
                                        const int ny = ry - v, nx = rx - u;
                                        if (ny < 0 || nx < 0 || ny % STR || nx % STR || ny / STR >= TH ||
                                            nx / STR >= TW)
                                            continue;
                                        q = (ny / STR) * OTW + nx / STR;
                                    } else {
                                        q = (ry * STR + v) * OTW + rx * STR + u;
                                    }
                                    fma_lane(acc[cc][v * R + u], d, O[q], ntap);
                                }
                            }
                        }
                    }
                    if (ry + 1 < CRH) {
#pragma unroll
                        for (int h = 0; h < NQ; ++h) cur[h] = nxt[h];
                    }
                }
                }  // in-line path
            }
            __syncthreads();  // stage buffer free for reuse
            sbuf = sbuf + 1 == G::NST ? 0 : sbuf + 1;
            cbufi = cbufi + 1 == G::NST ? 0 : cbufi + 1;
        }
    }
    cp_async_wait<0>();

    // partial[z][m][tap][l]: warps own disjoint checked channels
    float* pz = partial + (size_t)blockIdx.z * Mc * TAPS * Lc;
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int f = 0; f < TAPS; ++f) {
            float* dstp = pz + ((size_t)(mc0 + warp * CB + a) * TAPS + f) * Lc + l0;
            if constexpr (KK == 4) {
                *reinterpret_cast<float4*>(dstp) = make_float4(acc[a][f][0], acc[a][f][1], acc[a][f][2], acc[a][f][3]);
            } else if constexpr (KK == 2) {
                *reinterpret_cast<float2*>(dstp) = make_float2(acc[a][f][0], acc[a][f][1]);
            } else {
                dstp[0] = acc[a][f][0];
            }
        }
    if (SPARSE && exec_ctr) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (2 * KK));
    }
}

// Sum the splits in fixed order and scatter into FilterKCRSblk (K, C).
template <bool CHECK_INPUT>
__global__ void bww_tile_reduce(DevShape sh, const float* __restrict__ partial, int splits, float* __restrict__ dst,
                                const int* __restrict__ sel = nullptr, int want = 0) {
    if (sel != nullptr && __ldg(sel) != want) return;
    const int TAPS = sh.R * sh.S;
    const int Lc = CHECK_INPUT ? sh.K : sh.C, Mc = CHECK_INPUT ? sh.C : sh.K;
    const size_t E = (size_t)Mc * TAPS * Lc;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < E; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int z = 0; z < splits; ++z) s += partial[(size_t)z * E + e];
        const int l = (int)(e % Lc);
        const int f = (int)((e / Lc) % TAPS);
        const int m = (int)(e / ((size_t)Lc * TAPS));
        const int k = CHECK_INPUT ? l : m, c = CHECK_INPUT ? m : l;
        dst[filter_index(sh.C, sh.S, sh.R, 16, k, c, f % sh.R, f / sh.R)] = s;
    }
}

// ---------------------------------------------------------------- dispatch
// Launch kernel variant(s) then the fixed-order split reduction.  With
// JTSEL, sparse mode launches both the per-pixel-branch kernel and the
// jump-table kernel; a density probe on the checked tensor picks one on the
// device (the other exits at entry), no host synchronisation.
template <bool CI, int KK, int CB, int NWC, int TH, int TW, int R, int S, int STR, bool JTSEL = false,
          bool COUNTED_DENSE = false>
static cudaError_t launch_bww_cfg(bool sparse, const DevShape& sh, const float* chk, const float* oth,
                                  float* dst, unsigned long long* exec_ctr, cudaStream_t st,
                                  const int* xsel = nullptr, int xwant = 0) {
    using G = BwwGeom<CI, KK, CB, NWC, TH, TW, R, S, STR>;
    const int Lc = CI ? sh.K : sh.C, Mc = CI ? sh.C : sh.K;
    const long items = (long)((sh.N + 15) / 16) * ((sh.Wp + TW - 1) / TW) * ((sh.Hp + TH - 1) / TH);
    const long base = (long)(Mc / G::NCH) * (Lc / (32 * KK));
    // Split count: aim for ~6 CTAs per SM; 3x3 s1 layers with 16-128 base
    // CTAs (VGG conv2_2..conv4_1) measured 4-10% faster at ~18 per SM
    // (SPC_BWW_CTAS sweep, profiles/r01_tune.md).  Fixed per shape, so the
    // summation order stays deterministic.
    static const long env_ctas = std::getenv("SPC_BWW_CTAS") ? std::atol(std::getenv("SPC_BWW_CTAS")) : 0;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long target_ctas =
        env_ctas > 0 ? env_ctas : (R == 3 && STR == 1 && base >= 16 && base <= 128) ? nsm * 18L : nsm * 6L;
    long splits = (target_ctas + base - 1) / base;
    if (splits > items) splits = items;
    const size_t E = (size_t)Mc * R * S * Lc;
    // bounded split-partial workspace: splits x |dG| <= 256 MB (stream-ordered pool memory)
    const long cap = (long)((256ull << 20) / (E * sizeof(float)));
    if (splits > cap) splits = cap;
    if (splits < 1) splits = 1;
    float* partial = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)splits * E * sizeof(float), st);
    if (e != cudaSuccess) return e;
    dim3 grid(Mc / G::NCH, Lc / (32 * KK), (unsigned)splits);
    if (sparse && JTSEL) {
        int* sel = stream_flags(st) ? stream_flags(st) + FLAG_BWW_SEL : nullptr;
        if (sel == nullptr) {
            cudaFreeAsync(partial, st);
            return cudaErrorMemoryAllocation;
        }
        const size_t n = (size_t)((sh.N + 15) / 16) * Mc * (CI ? sh.H * sh.W : sh.Hp * sh.Wp) * 16;
        launch_density_probe(chk, n, 15, sel, st);
        auto k0 = bww_tile_kernel<CI, KK, CB, NWC, TH, TW, R, S, STR, 0, true>;
        auto k1 = bww_tile_kernel<CI, KK, CB, NWC, TH, TW, R, S, STR, 100, true>;
        cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        k0<<<grid, G::NT, G::SMEM, st>>>(sh, chk, oth, partial, (int)splits, exec_ctr, sel, 0);
        k1<<<grid, G::NT, G::SMEM, st>>>(sh, chk, oth, partial, (int)splits, exec_ctr, sel, 1);
        note_launch(2);
    } else {
        auto kern = sparse ? bww_tile_kernel<CI, KK, CB, NWC, TH, TW, R, S, STR, COUNTED_DENSE ? 200 : 0, true>
                           : bww_tile_kernel<CI, KK, CB, NWC, TH, TW, R, S, STR, 0, false>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        kern<<<grid, G::NT, G::SMEM, st>>>(sh, chk, oth, partial, (int)splits, exec_ctr, xsel, xwant);
        note_launch();
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        unsigned rb = (unsigned)((E + 255) / 256);
        if (rb > 148 * 8) rb = 148 * 8;
        bww_tile_reduce<CI><<<rb, 256, 0, st>>>(sh, partial, (int)splits, dst, xsel, xwant);
        note_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(partial, st);
    return e;
}

#ifdef SPC_DEV
// Development entry: alternative BWW tile configurations (tools/tune.py --comp bww).
cudaError_t launch_tile_bww_variant(int variant, bool check_input, bool sparse, const DevShape& sh, const float* chk,
                                    const float* oth, float* dst, unsigned long long* exec_ctr, cudaStream_t st) {
    const int Lc = check_input ? sh.K : sh.C, Mc = check_input ? sh.C : sh.K;
    if (sh.R != 3 || sh.O != 1) return cudaErrorInvalidValue;
#define SPC_BV(ID, CI, KK, CB, NWC, TH, TW)                                                                  \
    case ID:                                                                                                 \
        if (check_input != CI || Lc % (32 * KK) || Mc % (CB * NWC)) return cudaErrorInvalidValue;           \
        return launch_bww_cfg<CI, KK, CB, NWC, TH, TW, 3, 3, 1>(sparse, sh, chk, oth, dst, exec_ctr, st);
    switch (variant) {
        SPC_BV(0, true, 4, 1, 8, 4, 4)
        SPC_BV(1, true, 4, 1, 4, 4, 4)
        SPC_BV(2, true, 4, 1, 8, 4, 7)
        SPC_BV(3, true, 4, 1, 8, 7, 4)
        SPC_BV(4, true, 2, 2, 8, 4, 4)
        SPC_BV(5, true, 2, 2, 8, 4, 7)
        SPC_BV(6, true, 2, 2, 8, 7, 7)
        SPC_BV(7, true, 4, 1, 8, 2, 4)
        SPC_BV(8, true, 2, 1, 8, 7, 7)
        SPC_BV(9, true, 4, 2, 4, 4, 4)
        SPC_BV(10, true, 2, 4, 4, 4, 4)
        SPC_BV(11, true, 4, 1, 8, 4, 8)
        SPC_BV(12, true, 4, 1, 4, 4, 7)
        SPC_BV(13, true, 2, 2, 4, 4, 7)
        SPC_BV(20, false, 4, 1, 8, 2, 4)
        SPC_BV(21, false, 2, 2, 8, 4, 4)
        SPC_BV(22, false, 4, 1, 8, 4, 4)
        SPC_BV(23, false, 2, 1, 8, 4, 7)
        SPC_BV(24, false, 4, 1, 4, 2, 4)
        // round 2: more checked channels per warp (CB) against the shared-memory bound
        SPC_BV(30, true, 4, 2, 8, 7, 4)
        SPC_BV(31, true, 4, 2, 4, 7, 4)
        SPC_BV(32, true, 2, 4, 4, 7, 4)
        SPC_BV(33, true, 2, 4, 8, 7, 4)
        SPC_BV(34, true, 2, 2, 8, 7, 4)
        SPC_BV(35, true, 4, 2, 8, 4, 4)
        SPC_BV(36, true, 4, 3, 8, 4, 4)
        default: return cudaErrorInvalidValue;
    }
#undef SPC_BV
}
#endif  // SPC_DEV

bool tile_bww_supported(bool check_input, const DevShape& sh, int V) {
    if (V != 16) return false;
    // the staging descriptors hold 32-bit element offsets (tile_bww_kernel
    // cgo / ogo); larger tensors take the shape-general kernel (size_t)
    const size_t chwnn = (size_t)((sh.N + 15) / 16) * 16 * sh.C * sh.H * sh.W;
    const size_t dy = (size_t)((sh.N + 15) / 16) * 16 * sh.K * sh.Hp * sh.Wp;
    if (chwnn >= (1ull << 32) || dy >= (1ull << 32)) return false;
    const int Lc = check_input ? sh.K : sh.C, Mc = check_input ? sh.C : sh.K;
    if (Lc % 64 || Mc % 16) return false;
    if (sh.R != sh.S || sh.O != sh.P) return false;
    if (sh.padW != (sh.R - 1) / 2 || sh.padH != (sh.S - 1) / 2) return false;
    if ((sh.R == 3 || sh.R == 1) && (sh.O == 1 || sh.O == 2)) return true;
    return false;
}

cudaError_t launch_tile_bww(bool check_input, bool sparse, const DevShape& sh, const float* chk, const float* oth,
                            float* dst, unsigned long long* exec_ctr, cudaStream_t st) {
    const int Lc = check_input ? sh.K : sh.C;
    const bool kk4 = Lc % 128 == 0;
#define SPC_B(CI, KK, CB, NWC, TH, TW, R, STR) \
    return launch_bww_cfg<CI, KK, CB, NWC, TH, TW, R, R, STR>(sparse, sh, chk, oth, dst, exec_ctr, st)
    if (check_input) {
        if (sh.R == 3 && sh.O == 1) {
            // tools/tune.py --comp bww sweeps (profiles/r01_tune.md).  The
            // jump-table BWW variant (JTSEL) measured slower than per-pixel
            // branches at every sparsity of the VGG sweep; branches only.
            if (kk4) SPC_B(true, 4, 1, 8, 7, 4, 3, 1);
            SPC_B(true, 2, 2, 4, 4, 7, 3, 1);
        }
        if (sh.R == 3) {
            if (kk4) SPC_B(true, 4, 2, 4, 2, 4, 3, 2);
            SPC_B(true, 2, 4, 4, 2, 4, 3, 2);
        }
        if (sh.O == 1) {
            if (kk4) SPC_B(true, 4, 4, 4, 4, 8, 1, 1);
            SPC_B(true, 2, 4, 4, 4, 8, 1, 1);
        }
        if (kk4) SPC_B(true, 4, 4, 4, 4, 8, 1, 2);
        SPC_B(true, 2, 4, 4, 4, 8, 1, 2);
    }
    if (sh.R == 3 && sh.O == 1) {
        SPC_B(false, 2, 1, 8, 4, 7, 3, 1);
    }
    if (sh.R == 3) {
        if (kk4) SPC_B(false, 4, 2, 4, 2, 2, 3, 2);
        SPC_B(false, 2, 2, 4, 2, 4, 3, 2);
    }
    if (sh.O == 1) {
        if (kk4) SPC_B(false, 4, 4, 4, 4, 8, 1, 1);
        SPC_B(false, 2, 4, 4, 4, 8, 1, 1);
    }
    if (kk4) SPC_B(false, 4, 4, 4, 4, 8, 1, 2);
    SPC_B(false, 2, 4, 4, 4, 8, 1, 2);
#undef SPC_B
}

// 3x3 stride-2 check=input BWW runs counted dense unless SPC_BWW_S2_SKIP=1 (A/B).  The caller
// must then have folded BOTH operands' finiteness into *sel (0 * Inf would be NaN where the
// reference skips): tile_bww_counted_dense() tells it so.
static bool counted_dense_s2() {
    static const bool skip = std::getenv("SPC_BWW_S2_SKIP") && std::atoi(std::getenv("SPC_BWW_S2_SKIP")) == 1;
    return !skip;
}
bool tile_bww_counted_dense(bool check_input, const DevShape& sh) {
    return check_input && sh.R == 3 && sh.S == 3 && sh.O == 2 && sh.P == 2 && counted_dense_s2();
}

// The default stride-1 configurations gated on a device word (*sel == want):
// the exact FFMA BWW behind the tensor-core variant for Inf/NaN operands.
cudaError_t launch_tile_bww_when(bool check_input, bool sparse, const DevShape& sh, const float* chk,
                                 const float* oth, float* dst, unsigned long long* exec_ctr, cudaStream_t st,
                                 const int* sel, int want, bool both_finite_gated) {
    const bool kk4 = (check_input ? sh.K : sh.C) % 128 == 0;
#define SPC_B(CI, KK, CB, NWC, TH, TW, R) \
    return launch_bww_cfg<CI, KK, CB, NWC, TH, TW, R, R, 1>(sparse, sh, chk, oth, dst, exec_ctr, st, sel, want)
#define SPC_B2(CI, KK, CB, NWC, TH, TW, R) \
    return launch_bww_cfg<CI, KK, CB, NWC, TH, TW, R, R, 2>(sparse, sh, chk, oth, dst, exec_ctr, st, sel, want)
#define SPC_B2D(CI, KK, CB, NWC, TH, TW, R)                                                                          \
    return launch_bww_cfg<CI, KK, CB, NWC, TH, TW, R, R, 2, false, true>(sparse, sh, chk, oth, dst, exec_ctr, st, sel, \
                                                                         want)
    if (sh.O == 2) {  // the stride-2 configurations of launch_tile_bww
        if (check_input) {
            if (sh.R == 3) {
                // counted dense (tile_bww_counted_dense): measured 627 -> ~430 us on ResNet-50's
                // stage-2 3x3 stride-2 BWW at s = 0.6 (the per-pixel branches cost more than they skip)
                if (both_finite_gated && counted_dense_s2()) {
                    if (kk4) SPC_B2D(true, 4, 2, 4, 2, 4, 3);
                    SPC_B2D(true, 2, 4, 4, 2, 4, 3);
                }
                if (kk4) SPC_B2(true, 4, 2, 4, 2, 4, 3);
                SPC_B2(true, 2, 4, 4, 2, 4, 3);
            }
            if (kk4) SPC_B2(true, 4, 4, 4, 4, 8, 1);
            SPC_B2(true, 2, 4, 4, 4, 8, 1);
        }
        if (sh.R == 3) {
            if (kk4) SPC_B2(false, 4, 2, 4, 2, 2, 3);
            SPC_B2(false, 2, 2, 4, 2, 4, 3);
        }
        if (kk4) SPC_B2(false, 4, 4, 4, 4, 8, 1);
        SPC_B2(false, 2, 4, 4, 4, 8, 1);
    }
    if (check_input) {
        if (sh.R == 3) {
            if (kk4) SPC_B(true, 4, 1, 8, 7, 4, 3);
            SPC_B(true, 2, 2, 4, 4, 7, 3);
        }
        if (kk4) SPC_B(true, 4, 4, 4, 4, 8, 1);
        SPC_B(true, 2, 4, 4, 4, 8, 1);
    }
    if (sh.R == 3) SPC_B(false, 2, 1, 8, 4, 7, 3);
    if (kk4) SPC_B(false, 4, 4, 4, 4, 8, 1);
    SPC_B(false, 2, 4, 4, 4, 8, 1);
#undef SPC_B
#undef SPC_B2
#undef SPC_B2D
}

}  // namespace spc
