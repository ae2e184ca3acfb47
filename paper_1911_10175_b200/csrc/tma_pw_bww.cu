// tma_pw_bww.cu -- BWW for 1x1 convs (stride 1 / 2), check = input, V = 16, finite dY:
// the GEMM of pw_bww.cu with both operands staged by TMA.
//
// dG[k, c] = sum over images i and output pixels o of dY[i, k, o] * D[i, c, s(o)]
// (P/src/kernel_impl.hpp:209-336 for R = S = 1): M = K, N = C, reduction r = (i, o).
//
// pw_bww.cu stages dY with a 4-byte transposing cp.async per element -- 8 gathers with
// their index arithmetic per thread per 16-r chunk -- and ran at 22-25 TFLOP/s.  Here
// one stage is one output pixel x one 16-image block (16 reduction rows), and both
// operands arrive by TMA exactly as they lie in memory:
//   A[r][BK]  dY (ActNCHWc): a box of (16 channels, BK/16 channel blocks, 1 pixel,
//             16 images) -- the tensor map orders the dimensions (16, block, pixel,
//             image), so the rows land image-major with the BK channels contiguous;
//   B[c][16]  D (ActCHWNn): a box of (16 image lanes, 1 pixel, BC channels), 64-byte
//             rows under SWIZZLE_64B so that the 16 lanes of a warp reading rows
//             c = tx + 16 j at the same 16-byte chunk hit 8 distinct bank groups.
// One elected thread issues the two loads per stage behind full / empty mbarriers
// (no CTA barrier, no staging instructions in the compute warps); the compute loop
// is a plain 8 x 8 register-blocked FFMA2 GEMM: per 4 r, 8 LDS.128 of D (one per c
// row) + 8 of dY feed 128 FFMA2.  (A first version transposed D into ActNCHWc in a
// pre-pass so that both tiles were [r][channel]: the pre-pass alone cost 60-100 us
// of a 250-400 us pass.)  Same policy as pw_bww.cu: every FMA executes ("counted
// dense": a zero test per element never paid for 1x1 on B200), zero products are
// exact for finite dY, and the dispatcher runs pw_bww.cu's EXACT instantiation when
// dY holds Inf / NaN.  executed_vector_fmas stays the reference's exact count
// (nonzero staged D elements x K/16).  Splits + a fixed-order reduce: bitwise
// deterministic.
#include <cstdlib>

#include "common.cuh"
#include "pw_bww.h"
#include "tc_common.cuh"

namespace spc {

using tc::mbar_arrive;
using tc::mbar_expect_tx;
using tc::mbar_init;
using tc::smem_u32;

namespace {

constexpr int TP_RT = 16;   // reduction rows per stage: one output pixel x 16 images
constexpr int TP_NST = 4;   // stages

__device__ __forceinline__ void tp_mbar_wait(uint32_t bar, uint32_t parity) {
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
__device__ __forceinline__ void tp_tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                               int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
        : "memory");
}

template <int BK, int BC, bool COUNT>
__global__ void __launch_bounds__((BK / 8) * (BC / 8), 2)
    tma_pw_bww_kernel(const __grid_constant__ CUtensorMap mapD, const __grid_constant__ CUtensorMap mapY, int NB,
                      int C, int K, int HWo, int Wo, int Ws, int str, float* __restrict__ partial, int splits,
                      unsigned long long* __restrict__ exec_ctr, const int* __restrict__ finite) {
    if (__ldg(finite) == 0) return;  // dY holds Inf / NaN: pw_bww.cu's EXACT kernel runs instead
    constexpr int NT = (BK / 8) * (BC / 8);
    constexpr int NWARP = NT / 32;
    static_assert(NWARP <= 15, "one named barrier (ids 1..15) per warp");
    constexpr int ABYTES = TP_RT * BK * 4, BBYTES = BC * TP_RT * 4, STAGE = ABYTES + BBYTES;
    extern __shared__ __align__(1024) uint8_t smem[];  // no static shared memory in this kernel: offset 0
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bars = sbase + TP_NST * STAGE;
    auto full_bar = [&](int s) { return bars + 8u * s; };
    auto empty_bar = [&](int s) { return bars + 8u * (TP_NST + s); };

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tx = tid % (BC / 8), ty = tid / (BC / 8);
    const int k_base = blockIdx.x * BK, c_base = blockIdx.y * BC;
    const long items = (long)NB * HWo;  // (16-image block, output pixel), pixel fastest
    const int it0 = (int)(items * blockIdx.z / splits), it1 = (int)(items * (blockIdx.z + 1) / splits);

    if (tid == 0) {
        for (int s = 0; s < TP_NST; ++s) {
            mbar_init(full_bar(s), 1);
            mbar_init(empty_bar(s), NWARP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();

    auto issue = [&](int it, int li) {
        const int s = li % TP_NST;
        const int nb = it / HWo, o = it - nb * HWo;
        const int oy = o / Wo, ox = o - oy * Wo;
        const uint32_t dst = sbase + s * STAGE;
        mbar_expect_tx(full_bar(s), STAGE);
        tp_tma_load_4d(dst, &mapY, full_bar(s), 0, k_base / 16, o, nb * 16);
        tp_tma_load_4d(dst + ABYTES, &mapD, full_bar(s), 0, (oy * str) * Ws + ox * str, c_base, nb);
    };
    int pit = it0;
    if (tid == 0) {
        for (int d = 0; d < TP_NST - 1 && pit < it1; ++d, ++pit) issue(pit, d);
    }

    // thread tile: k = ty*4 + {0..3} and BK/2 + ty*4 + {0..3}; c = tx + (BC/8) * j, j < 8
    float2 acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.0f, 0.0f);
    uint32_t nz = 0;
    // SWIZZLE_64B: the 16-byte chunk q of 64-byte row `row` sits at chunk q ^ ((row >> 1) & 3)
    int brow[8], bsw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int c = tx + (BC / 8) * j;
        brow[j] = c * TP_RT;
        bsw[j] = (c >> 1) & 3;
    }

#pragma unroll 1
    for (int it = it0; it < it1; ++it) {
        const int li = it - it0;
        const int s = li % TP_NST;
        if (tid == 0 && pit < it1) {
            if (li >= 1) tp_mbar_wait(empty_bar((li - 1) % TP_NST), ((li - 1) / TP_NST) & 1);
            issue(pit, li + TP_NST - 1);
            ++pit;
        }
        tp_mbar_wait(full_bar(s), (li / TP_NST) & 1);
        // tells ptxas the warp is converged after the spin (tma_bww.cu has the measurement)
        asm volatile("barrier.sync.aligned %0, 32;" ::"r"(warp + 1) : "memory");
        const float* A = reinterpret_cast<const float*>(smem + s * STAGE);           // [r][BK]
        const float* B = reinterpret_cast<const float*>(smem + s * STAGE + ABYTES);  // [c][16 r], swizzled
        if (COUNT && blockIdx.x == 0) {
            for (int t = tid; t < TP_RT * BC; t += NT) nz += B[t] != 0.0f;
        }
        const float* Ap = A + ty * 4;
#pragma unroll
        for (int r0 = 0; r0 < TP_RT; r0 += 4) {
            float4 b[8];  // row c_j, r0 .. r0+3
#pragma unroll
            for (int j = 0; j < 8; ++j)
                b[j] = *reinterpret_cast<const float4*>(B + brow[j] + (((r0 >> 2) ^ bsw[j]) << 2));
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int r = r0 + h;
                const float4 a0 = *reinterpret_cast<const float4*>(Ap + r * BK);
                const float4 a1 = *reinterpret_cast<const float4*>(Ap + r * BK + BK / 2);
                const float2 pr[4] = {make_float2(a0.x, a0.y), make_float2(a0.z, a0.w), make_float2(a1.x, a1.y),
                                      make_float2(a1.z, a1.w)};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float v = h == 0 ? b[j].x : h == 1 ? b[j].y : h == 2 ? b[j].z : b[j].w;
#pragma unroll
                    for (int i = 0; i < 4; ++i) acc[i][j] = __ffma2_rn(pr[i], make_float2(v, v), acc[i][j]);
                }
            }
        }
        // Generic-proxy reads (the LDS above) against the async-proxy TMA write that refills this
        // stage: the release on the empty barrier does not order them across proxies.  Measured:
        // without this fence ~1e-4 relative errors, different from run to run, on shapes whose CTAs
        // reuse their stages (56x56 images); with it, bitwise reproducible.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(s));
    }

    // partial[split][c][k] (pw_bww_reduce's layout)
    float* P = partial + (size_t)blockIdx.z * C * K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = k_base + (i < 2 ? ty * 4 + 2 * i : BK / 2 + ty * 4 + 2 * (i - 2));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = c_base + tx + (BC / 8) * j;
            *reinterpret_cast<float2*>(P + (size_t)c * K + k) = acc[i][j];
        }
    }
    if (COUNT && blockIdx.x == 0 && exec_ctr) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, nz);
        if (lane == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (K / 16));
    }
}

// fixed-order split sum -> FilterKCRSblk (K, C), R = S = 1 (gated like the kernel)
__global__ void tp_reduce(int C, int K, const float* __restrict__ partial, int splits, float* __restrict__ dst,
                          const int* __restrict__ finite) {
    if (__ldg(finite) == 0) return;
    const size_t E = (size_t)C * K;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < E; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int z = 0; z < splits; ++z) s += partial[(size_t)z * E + e];
        const int k = (int)(e % K), c = (int)(e / K);
        dst[((size_t)(k / 16) * (C / 16) + c / 16) * 256 + (c % 16) * 16 + k % 16] = s;
    }
}

template <int BK, int BC>
cudaError_t tp_launch(bool sparse, const DevShape& sh, const float* dchw, const float* dy, float* dst,
                      unsigned long long* exec_ctr, const int* finite, cudaStream_t st) {
    constexpr int NT = (BK / 8) * (BC / 8);
    constexpr int STAGE = TP_RT * (BK + BC) * 4;
    constexpr int SMEM = TP_NST * STAGE + 2 * TP_NST * 8;
    const int HW = sh.H * sh.W, HWo = sh.Hp * sh.Wp;
    const int NB = (sh.N + 15) / 16;
    const long items = (long)NB * HWo;
    const long tiles = (long)(sh.K / BK) * (sh.C / BC);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    long splits = ((long)nsm * 4 + tiles - 1) / tiles;  // 2 CTAs per SM, 2 waves
    if (splits > items) splits = items;
    if (splits < 1) splits = 1;
    float* partial = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)splits * sh.C * sh.K * sizeof(float), st);
    if (e != cudaSuccess) return e;

    CUtensorMap mapD, mapY;
    auto enc = tc::encode_fn();
    bool ok;
    {  // dY ActNCHWc [N][K/16][HWo][16]: (16, channel block, pixel, image); images past N read as zeros
        cuuint64_t dims[4] = {16, (cuuint64_t)(sh.K / 16), (cuuint64_t)HWo, (cuuint64_t)sh.N};
        cuuint64_t strides[3] = {(cuuint64_t)HWo * 64, 64, (cuuint64_t)(sh.K / 16) * HWo * 64};
        cuuint32_t box[4] = {16, (cuuint32_t)(BK / 16), 1, 16};
        cuuint32_t es[4] = {1, 1, 1, 1};
        ok = enc(&mapY, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(dy), dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (ok) {  // D ActCHWNn [NB][C][HW][16 images]: (16, pixel, channel, image block), 64-byte rows swizzled
        cuuint64_t dims[4] = {16, (cuuint64_t)HW, (cuuint64_t)sh.C, (cuuint64_t)NB};
        cuuint64_t strides[3] = {64, (cuuint64_t)HW * 64, (cuuint64_t)sh.C * HW * 64};
        cuuint32_t box[4] = {16, 1, (cuuint32_t)BC, 1};
        cuuint32_t es[4] = {1, 1, 1, 1};
        ok = enc(&mapD, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(dchw), dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    if (!ok) {
        cudaFreeAsync(partial, st);
        return cudaErrorInvalidValue;
    }
    auto kern = sparse ? tma_pw_bww_kernel<BK, BC, true> : tma_pw_bww_kernel<BK, BC, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    dim3 grid(sh.K / BK, sh.C / BC, (unsigned)splits);
    kern<<<grid, NT, SMEM, st>>>(mapD, mapY, NB, sh.C, sh.K, HWo, sh.Wp, sh.W, sh.O, partial, (int)splits, exec_ctr,
                                 finite);
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        unsigned rb = (unsigned)(((size_t)sh.C * sh.K + 255) / 256);
        if (rb > 148 * 8) rb = 148 * 8;
        tp_reduce<<<rb, 256, 0, st>>>(sh.C, sh.K, partial, (int)splits, dst, finite);
        note_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(partial, st);
    return e;
}

}  // namespace

bool tma_pw_bww_supported(const DevShape& sh) {
    static const bool off = std::getenv("SPC_TMA_PW_BWW") && std::atoi(std::getenv("SPC_TMA_PW_BWW")) == 0;
    if (off || tc::encode_fn() == nullptr) return false;
    if ((size_t)sh.N * sh.C * sh.H * sh.W >= (1ull << 32)) return false;
    return sh.C % 64 == 0 && sh.K % 64 == 0;
}

// runs when *finite == 1 (dY finite); exits at entry otherwise
cudaError_t launch_tma_pw_bww(bool sparse, const DevShape& sh, const float* dchw, const float* dy, float* dst,
                              unsigned long long* exec_ctr, const int* finite, cudaStream_t st) {
    const bool k128 = sh.K % 128 == 0, c128 = sh.C % 128 == 0;
    if (k128 && c128) return tp_launch<128, 128>(sparse, sh, dchw, dy, dst, exec_ctr, finite, st);
    if (k128) return tp_launch<128, 64>(sparse, sh, dchw, dy, dst, exec_ctr, finite, st);
    if (c128) return tp_launch<64, 128>(sparse, sh, dchw, dy, dst, exec_ctr, finite, st);
    return tp_launch<64, 64>(sparse, sh, dchw, dy, dst, exec_ctr, finite, st);
}

}  // namespace spc
