// row_bww.cu -- BWW with check = input for 3x3 stride-1 pad-1 layers (V = 16):
// a row-streaming register window with dispatch over the nonzeros only.
//
// dG[k,c,v,u] = sum_{i,y',x'} D[i,c,y'+v-1,x'+u-1] * dY[i,k,y',x']
// (P/src/kernel_impl.hpp:209-336 bww_task_impl<VB, CheckInput=true>,
//  P/src/kernels.cpp:238-302).
//
// Why a new kernel (round-1 tile_bww.cu is kept for the other geometries):
// there, every warp reloaded a 7x4-pixel dY tile (28 LDS.128) per image for a
// single checked channel, so shared-memory bandwidth, not the FMA pipe, bounded
// it (ncu: L1 70%, FMA 41% at s = 0.6), and every checked pixel paid a
// branch whether zero or not.  Here:
//   * A warp owns CB checked channels c and 32*KK lane channels k (the other
//     operand's; every lane consumes the same checked value, so the zero test
//     is warp-uniform).  A work item is one image x one TW-wide column strip
//     of the output, swept top to bottom over the whole image height.
//   * The dY rows live in a 3-row REGISTER WINDOW (3 x TW pixels x KK
//     channels): each dY value is read from shared memory once per warp and
//     reused by the CB channels x 3 row taps it meets, so the shared-memory
//     bytes per FMA drop by CB (x3 vs the round-1 kernel's per-image reload).
//   * Per input row the warp loads its CB x (TW+2) checked values with one
//     conflict-free LDS per lane, takes ONE __ballot_sync (the nonzero mask of
//     the whole row for all its channels, the paper's per-vector zero check),
//     and walks the bits with one warp-uniform branch each into a block of
//     static-register FFMA2s (acc[c][tap] += d * dY[tap's output pixel]); a
//     zero costs its branch only.  (Dispatching set bits through a jump table
//     -- brx per nonzero -- measured 4-6x slower.)
//   * Rows are staged by a cp.async pipeline (NST rows deep, one barrier per
//     row): the dY row as 16-byte copies of the ActNCHWc channel vectors, the
//     checked row's (TW+2) pixels per channel out of ActCHWNn.
//   * Exactness: output pixels outside the image read zero-filled window
//     slots instead of being skipped, so d * 0 terms are added (exact for
//     finite d).  A device scan of D selects, when D holds Inf/NaN, the
//     round-1 tile kernel (exact skip semantics) instead -- both launched, the
//     non-matching one exits at entry (no host sync).
//   * executed_vector_fmas is counted exactly like the reference's
//     (popcount x valid targets x K/V), per lane from the row's mask.
//   * The reduction over (image, strip) items is split over CTAs in fixed
//     item ranges; the partials are summed in fixed order (deterministic).
#include <type_traits>

#include "common.cuh"
#include "tile_bww.h"

namespace spc {

namespace {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int KK, int CB, int NW, int TW>
struct RowGeom {
    static constexpr int RW = TW + 2;   // region columns of a strip (1-pixel halo each side)
    static constexpr int NB = CB * RW;  // mask bits of one warp row
    static constexpr int NCH = NW * CB; // checked channels per CTA
    static constexpr int LK = 32 * KK;  // lane channels per CTA
    static constexpr int DROW = 8;      // padded region row in shared memory
    static constexpr int DFLOATS = NCH * DROW;
    static constexpr int OFLOATS = TW * LK;
    static constexpr int ROW = DFLOATS + OFLOATS;  // one row's staging
    static constexpr int RB = 3;                   // rows per pipeline stage (= the window's 3 phases)
    static constexpr int STAGE = RB * ROW;
    static constexpr int NST = 6;
    static constexpr int ND = (RB * NCH * RW + NW * 32 - 1) / (NW * 32);      // D copies per thread per stage
    static constexpr int NO = (RB * TW * LK / 4 + NW * 32 - 1) / (NW * 32);   // dY copies per thread per stage
    static constexpr int NT = NW * 32;
    static constexpr int SMEM = NST * STAGE * 4;
    static_assert(NB <= 32, "one mask word per warp row");
    static_assert(RW <= DROW, "region row must fit the padded row");
    static_assert(KK == 2 || KK == 4, "KK");
};

// acc[cc][tap] += d * window[slot(v)][t] for the (v, u) taps whose output
// pixel t = r - u lies in the strip; J = cc * RW + r, PH = step % 3.
template <int KK, int CB, int TW, int PH, int J>
__device__ __forceinline__ void row_block(float2 (&acc)[CB][9][KK / 2], const float2 (&win)[3][TW][KK / 2],
                                          float d) {
    constexpr int RW = TW + 2;
    constexpr int cc = J / RW, r = J % RW;
    const float2 dd = make_float2(d, d);
#pragma unroll
    for (int v = 0; v < 3; ++v) {
        const int slot = (PH - v + 3) % 3;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            const int t = r - u;
            if (t < 0 || t >= TW) continue;
#pragma unroll
            for (int j = 0; j < KK / 2; ++j) acc[cc][v * 3 + u][j] = __ffma2_rn(dd, win[slot][t][j], acc[cc][v * 3 + u][j]);
        }
    }
}

// Walk the row's mask bits in a fixed order: one warp-uniform branch per bit
// (the ballot result is uniform), the bit's FFMA2 block when set.  Straight-
// line code with forward branches only: an indirect jump per nonzero
// (brx through a jump table) measured 4-6x slower on the B200 (branch
// resolution + instruction fetch per nonzero).
template <int KK, int CB, int TW, int PH, int J>
__device__ __forceinline__ void row_bits_pre(uint32_t m, const float (&dv)[CB * (TW + 2)],
                                             float2 (&acc)[CB][9][KK / 2], const float2 (&win)[3][TW][KK / 2]) {
    if constexpr (J < CB * (TW + 2)) {
        if (m & (1u << J)) row_block<KK, CB, TW, PH, J>(acc, win, dv[J]);
        row_bits_pre<KK, CB, TW, PH, J + 1>(m, dv, acc, win);
    }
}

}  // namespace

template <int KK, int CB, int NW, int TW, bool SPARSE>
__global__ void __launch_bounds__(NW * 32) row_bww_kernel(DevShape sh, const float* __restrict__ chk,
                                                          const float* __restrict__ oth,
                                                          float* __restrict__ partial, int splits,
                                                          unsigned long long* __restrict__ exec_ctr,
                                                          const int* __restrict__ sel, int want) {
    using G = RowGeom<KK, CB, NW, TW>;
    if (sel != nullptr && __ldg(sel) != want) return;
    constexpr int RW = G::RW, NB = G::NB, NCH = G::NCH, LK = G::LK, NST = G::NST, NT = G::NT;
    extern __shared__ __align__(16) float smem[];  // NST x {D rows [NCH][DROW], dY row [TW][LK]}

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mc0 = blockIdx.x * NCH;  // first checked channel (c) of the CTA
    const int lc0 = blockIdx.y * LK;   // first lane channel (k) of the CTA
    const int H = sh.H, W = sh.W, Hp = sh.Hp, Wp = sh.Wp;
    const int steps = H + 1;  // per item: dY rows 0..H-1 enter the window, D rows 0..H-1 are swept
    const int spi = (steps + G::RB - 1) / G::RB;  // pipeline stages per item
    const int nstrips = (Wp + TW - 1) / TW;
    const int items = sh.N * nstrips;
    const int it0 = (int)((long)items * blockIdx.z / splits), it1 = (int)((long)items * (blockIdx.z + 1) / splits);
    const long G_stages = (long)(it1 - it0) * spi;
    const int KB = sh.K / 16;

    // Staging of rows s = j*RB .. j*RB+RB-1 (<= H) of item it into buffer b:
    // the checked row y = s - 1 (ActCHWNn, 4-byte copies) and the dY row s
    // (ActNCHWc, 16-byte copies), zero-filled outside the image.  Each thread
    // owns fixed (row, channel, pixel) slots; their item-dependent global
    // offsets are computed once per item (describe), a stage only adds its row.
    uint32_t d_off[G::ND], o_off[G::NO];  // element offsets (tensors < 2^32 floats, checked at launch)
    uint32_t d_ok = 0, o_ok = 0;
    int d_r[G::ND], o_r[G::NO];
    auto describe = [&](int it) {
        const int i = it / nstrips, x0 = (it % nstrips) * TW;
        d_ok = 0;
#pragma unroll
        for (int k = 0; k < G::ND; ++k) {
            const int e = threadIdx.x + k * NT;
            const int r = e / (NCH * RW), q = e % (NCH * RW);
            const int cc = q / RW, rr = q % RW;
            const int x = x0 - 1 + rr;
            const bool ok = e < G::RB * NCH * RW && x >= 0 && x < W;
            d_r[k] = e < G::RB * NCH * RW ? r : 1 << 20;
            // element (i, c, y = s - 1, x) of ActCHWNn minus the row term
            d_off[k] = ok ? (uint32_t)(((((size_t)(i >> 4) * sh.C + mc0 + cc) * H - 1) * W + x) * 16 + (i & 15)) : 0u;
            d_ok |= (ok ? 1u : 0u) << k;
        }
        o_ok = 0;
#pragma unroll
        for (int k = 0; k < G::NO; ++k) {
            const int e = threadIdx.x + k * NT;
            const int r = e / (TW * LK / 4), q = e % (TW * LK / 4);
            const int t = q / (LK / 4), c4 = q % (LK / 4);
            const int x = x0 + t;
            const bool ok = e < G::RB * TW * LK / 4 && x < Wp;
            o_r[k] = e < G::RB * TW * LK / 4 ? r : 1 << 20;
            o_off[k] = ok ? (uint32_t)(((((size_t)i * KB + (lc0 + c4 * 4) / 16) * Hp) * Wp + x) * 16 + (c4 % 4) * 4)
                          : 0u;
            o_ok |= (ok ? 1u : 0u) << k;
        }
    };
    auto stage = [&](int j, int b) {
        float* base = smem + b * G::STAGE;
        const int s0 = j * G::RB;
#pragma unroll
        for (int k = 0; k < G::ND; ++k) {
            const int e = threadIdx.x + k * NT;
            if (d_r[k] >= G::RB) continue;
            const int s = s0 + d_r[k];
            if (s < 1 || s > H) continue;
            const bool ok = (d_ok >> k) & 1u;
            const int q = e % (NCH * RW);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(
                             smem_addr(base + d_r[k] * G::ROW + (q / RW) * G::DROW + q % RW)),
                         "l"(chk + (ok ? d_off[k] + (uint32_t)(s * W * 16) : 0u)), "r"(ok ? 4 : 0));
        }
#pragma unroll
        for (int k = 0; k < G::NO; ++k) {
            const int e = threadIdx.x + k * NT;
            if (o_r[k] >= G::RB) continue;
            const int s = s0 + o_r[k];
            if (s >= Hp) continue;
            const bool ok = (o_ok >> k) & 1u;
            const int q = e % (TW * LK / 4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(
                             smem_addr(base + o_r[k] * G::ROW + G::DFLOATS + q * 4)),
                         "l"(oth + (ok ? o_off[k] + (uint32_t)(s * Wp * 16) : 0u)), "r"(ok ? 16 : 0));
        }
    };

    float2 acc[CB][9][KK / 2];
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int f = 0; f < 9; ++f)
#pragma unroll
            for (int j = 0; j < KK / 2; ++j) acc[a][f][j] = make_float2(0.0f, 0.0f);
    float2 win[3][TW][KK / 2];
    uint32_t cnt = 0;

    // pipeline prologue: the producer cursor runs NST-1 stages ahead
    long p_g = 0;
    int p_it = it0, p_j = 0, p_buf = 0;
    if (G_stages > 0) describe(p_it);
    for (int d = 0; d < NST - 1; ++d) {
        if (p_g < G_stages) {
            stage(p_j, p_buf);
            if (++p_j == spi) {
                p_j = 0;
                if (++p_it < it1) describe(p_it);
            }
            ++p_buf;
            ++p_g;
        }
        asm volatile("cp.async.commit_group;\n" ::);
    }

    // per-lane constants of the current item
    int x0 = 0, cv = 0;
    const int lr = lane % RW, lcc = lane / RW;

    auto step = [&](auto PHc, const float* base, int s) {
        constexpr int PH = decltype(PHc)::value;
        // 1. dY row s enters the window (zeros below the image)
#pragma unroll
        for (int t = 0; t < TW; ++t) {
            if (s < Hp) {
                const float* p = base + G::DFLOATS + t * LK + lane * KK;
                if constexpr (KK == 4) {
                    const float4 q = *reinterpret_cast<const float4*>(p);
                    win[PH][t][0] = make_float2(q.x, q.y);
                    win[PH][t][1] = make_float2(q.z, q.w);
                } else {
                    win[PH][t][0] = *reinterpret_cast<const float2*>(p);
                }
            } else {
#pragma unroll
                for (int j = 0; j < KK / 2; ++j) win[PH][t][j] = make_float2(0.0f, 0.0f);
            }
        }
        if (s == 0) return;
        // 2. checked row y = s - 1: one ballot for the warp's CB channels x RW pixels
        const int y = s - 1;
        const float* drow = base + warp * CB * G::DROW;
        const float val = lane < NB ? drow[lcc * G::DROW + lr] : 0.0f;
        const int x = x0 - 1 + lr;
        const bool nz = SPARSE ? (lane < NB && val != 0.0f) : (lane < NB && x >= 0 && x < W);
        const int rv = (y + 1 < Hp) + (y < Hp) + (y >= 1 && y - 1 < Hp);
        cnt += nz ? (uint32_t)(rv * cv) : 0u;
        const uint32_t m = __ballot_sync(0xffffffffu, nz);
        if (m == 0) return;
        // the row's values as broadcast 128-bit loads, all issued before the first FMA
        // (measured faster than fetching each set bit's value with a shuffle)
        float dv[NB];
#pragma unroll
        for (int a = 0; a < CB; ++a)
#pragma unroll
            for (int h = 0; h < (RW + 3) / 4; ++h) {
                const float4 q = *reinterpret_cast<const float4*>(drow + a * G::DROW + 4 * h);
                const float e4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int z = 0; z < 4; ++z)
                    if (4 * h + z < RW) dv[a * RW + 4 * h + z] = e4[z];
            }
        row_bits_pre<KK, CB, TW, PH, 0>(m, dv, acc, win);
    };

    // consumer cursor (item, stage) advanced incrementally: no divisions per row
    int c_it = it0, c_j = 0, c_buf = 0;
    for (long g = 0; g < G_stages; ++g) {
        asm volatile("cp.async.wait_group %0;\n" ::"n"(NST - 2));
        __syncthreads();  // stage g visible to all; everyone is past stage g-1, its buffer is free
        if (p_g < G_stages) {
            stage(p_j, p_buf);
            if (++p_j == spi) {
                p_j = 0;
                if (++p_it < it1) describe(p_it);
            }
            p_buf = p_buf + 1 == NST ? 0 : p_buf + 1;
            ++p_g;
        }
        asm volatile("cp.async.commit_group;\n" ::);
        if (c_j == 0) {  // new item: strip origin, per-lane valid-column count, zero the row -1 slot
            x0 = (c_it % nstrips) * TW;
            cv = 0;
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int t = lr - u;
                cv += (t >= 0 && t < TW && x0 + t < Wp) ? 1 : 0;
            }
#pragma unroll
            for (int t = 0; t < TW; ++t)
#pragma unroll
                for (int j = 0; j < KK / 2; ++j) win[2][t][j] = make_float2(0.0f, 0.0f);
        }
        const float* base = smem + c_buf * G::STAGE;
        const int s0 = c_j * G::RB;
        step(std::integral_constant<int, 0>{}, base, s0);
        if (s0 + 1 <= H) step(std::integral_constant<int, 1>{}, base + G::ROW, s0 + 1);
        if (s0 + 2 <= H) step(std::integral_constant<int, 2>{}, base + 2 * G::ROW, s0 + 2);
        if (++c_j == spi) { c_j = 0; ++c_it; }
        c_buf = c_buf + 1 == NST ? 0 : c_buf + 1;
    }
    asm volatile("cp.async.wait_group 0;\n" ::);

    // partial[z][c][tap][k]: warps own disjoint checked channels
    float* pz = partial + (size_t)blockIdx.z * sh.C * 9 * sh.K;
#pragma unroll
    for (int a = 0; a < CB; ++a)
#pragma unroll
        for (int f = 0; f < 9; ++f) {
            float* dstp = pz + ((size_t)(mc0 + warp * CB + a) * 9 + f) * sh.K + lc0 + lane * KK;
            if constexpr (KK == 4) {
                *reinterpret_cast<float4*>(dstp) = make_float4(acc[a][f][0].x, acc[a][f][0].y, acc[a][f][1].x,
                                                               acc[a][f][1].y);
            } else {
                *reinterpret_cast<float2*>(dstp) = acc[a][f][0];
            }
        }
    if (exec_ctr) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, cnt);
        if (lane == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (2 * KK));
    }
}

// Sum the splits in fixed order, scatter into FilterKCRSblk (K, C).
__global__ void row_bww_reduce(DevShape sh, const float* __restrict__ partial, int splits, float* __restrict__ dst,
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

bool row_bww_supported(bool check_input, const DevShape& sh, int V) {
    return check_input && V == 16 && sh.R == 3 && sh.S == 3 && sh.O == 1 && sh.P == 1 && sh.padW == 1 &&
           sh.padH == 1 && sh.K % 64 == 0 && sh.C % 16 == 0 &&
           (size_t)((sh.N + 15) / 16) * 16 * sh.C * sh.H * sh.W < (1ull << 32) &&
           (size_t)sh.N * sh.K * sh.Hp * sh.Wp < (1ull << 32);
}


template <int KK, int CB, int NW, int TW>
static cudaError_t launch_row_cfg(bool sparse, const DevShape& sh, const float* chk, const float* oth, float* dst,
                                  unsigned long long* exec_ctr, const int* sel, cudaStream_t st) {
    using G = RowGeom<KK, CB, NW, TW>;
    if (sh.C % G::NCH || sh.K % G::LK) return cudaErrorInvalidValue;
    // 32-bit element offsets inside the kernel
    if ((size_t)((sh.N + 15) / 16) * 16 * sh.C * sh.H * sh.W >= (1ull << 32) ||
        (size_t)sh.N * sh.K * sh.Hp * sh.Wp >= (1ull << 32))
        return cudaErrorInvalidValue;
    auto kern = sparse ? row_bww_kernel<KK, CB, NW, TW, true> : row_bww_kernel<KK, CB, NW, TW, false>;
    static PerDeviceOnce attr[2];
    int ad = 0;
    if (attr[sparse].needed(ad)) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
        attr[sparse].done(ad);
    }
    int dev = 0, nsm = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::NT, G::SMEM);
    if (per_sm < 1) per_sm = 1;
    const long items = (long)sh.N * ((sh.Wp + TW - 1) / TW);
    const long base = (long)(sh.C / G::NCH) * (sh.K / G::LK);
    // whole waves of resident CTAs: the largest split count with
    // base * splits <= waves * (SMs x CTAs/SM), at most one split per item;
    // the partial buffer stays bounded (splits x |dG| <= 256 MB)
    const long slots = (long)nsm * per_sm;
    long waves = (base + slots - 1) / slots;
    if (waves < 1) waves = 1;
    long splits = waves * slots / base;
    if (splits > items) splits = items;
    const size_t E = (size_t)sh.C * 9 * sh.K;
    const long cap = (long)((256ull << 20) / (E * sizeof(float)));
    if (splits > cap) splits = cap > 0 ? cap : 1;
    if (splits < 1) splits = 1;
    float* partial = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)splits * E * sizeof(float), st);
    if (e != cudaSuccess) return e;
    dim3 grid(sh.C / G::NCH, sh.K / G::LK, (unsigned)splits);
    kern<<<grid, G::NT, G::SMEM, st>>>(sh, chk, oth, partial, (int)splits, exec_ctr, sel, 1);
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        unsigned rb = (unsigned)((E + 255) / 256);
        if (rb > (unsigned)nsm * 8) rb = (unsigned)nsm * 8;
        row_bww_reduce<<<rb, 256, 0, st>>>(sh, partial, (int)splits, dst, sel, 1);
        note_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(partial, st);
    return e;
}

// The row kernel for a finite D (sel = 1); the caller enqueues the exact
// kernel for sel = 0.  KK=4 (128 lane channels) only runs when forced
// (SPC_ROW_BWW=1): it measured slower than the tile kernel;
// variants of round 2's sweep (shuffled values instead of the preloaded row,
// CB = 2, KK = 2 on 128-channel layers) were slower still and are not built.
cudaError_t launch_row_bww_when(bool sparse, const DevShape& sh, const float* chk, const float* oth, float* dst,
                                unsigned long long* exec_ctr, const int* sel, cudaStream_t st) {
    if (sh.K % 128 == 0)
        return launch_row_cfg<4, 4, 4, 4>(sparse, sh, chk, oth, dst, exec_ctr, sel, st);
    return launch_row_cfg<2, 4, 4, 4>(sparse, sh, chk, oth, dst, exec_ctr, sel, st);
}

}  // namespace spc
