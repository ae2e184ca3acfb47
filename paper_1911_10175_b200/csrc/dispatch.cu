// dispatch.cu -- kernel selection (internal).
#include "dispatch.h"

#include <cstdlib>

#include "pw_bww.h"
#include "pw_conv.h"
#include "pw_gemm.h"
#include "tc_conv.h"
#include "tile_bww.h"
#include "tile_conv.h"

namespace spc {

// Arithmetic of the FWD/BWI passes (spc_set_math): FP32 FFMA (default) or the
// 3xTF32 tensor-core variant.  Per host thread, like spc_last_error.
static thread_local int g_math = SPC_MATH_FP32;
int math_mode() { return g_math; }
void set_math_mode(int m) { g_math = m; }

__global__ void epilogue_kernel(Epi epi, float* __restrict__ out, size_t n) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
        out[e] = epi.apply(out[e], e);
}

cudaError_t launch_epilogue(const Epi& epi, float* out, size_t n, cudaStream_t st) {
    if (!epi.active() || n == 0) return cudaSuccess;
    epilogue_kernel<<<148 * 8, 256, 0, st>>>(epi, out, n);
    note_launch();
    return cudaGetLastError();
}

// SPC_PW_GEMM=0 routes 1x1 FWD/BWI to the lane-per-channel pw_conv kernel (A/B testing)
static bool use_pw_gemm() {
    static const bool off = std::getenv("SPC_PW_GEMM") && std::atoi(std::getenv("SPC_PW_GEMM")) == 0;
    return !off;
}

bool conv_supports_gate(bool fwd, const DevShape& sh, int V) {
    static const bool force_generic = std::getenv("SPC_FORCE_GENERIC") && std::atoi(std::getenv("SPC_FORCE_GENERIC"));
    if (force_generic) return false;
    if (use_pw_gemm() && pw_gemm_supported(fwd, sh, V)) return false;  // the GEMM kernel has no Gate
    return pw_conv_supported(fwd, sh, V) || tile_conv_supported(fwd, sh, V);
}

cudaError_t launch_conv(bool fwd, bool sparse, const DevShape& sh, int V, const float* src, const float* filt,
                        float* dst, unsigned long long* exec_ctr, cudaStream_t st, const Epi& epi, const Gate& gate) {
    // SPC_FORCE_GENERIC=1 selects the shape-general kernels (A/B testing only)
    static const bool force_generic = std::getenv("SPC_FORCE_GENERIC") && std::atoi(std::getenv("SPC_FORCE_GENERIC"));
    // SPC_PW_OFF=1 routes 1x1 convs to the tile kernel (A/B testing only)
    static const bool pw_off = std::getenv("SPC_PW_OFF") && std::atoi(std::getenv("SPC_PW_OFF"));
    if (g_math == SPC_MATH_TF32X3 && gate.in_ready == nullptr && tc_conv_supported(fwd, sh, V))
        return launch_tc_conv(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi);
    // 1x1 stride-2 BWI: the GEMM kernel with one row per SOURCE pixel (each row also
    // writes its 2x2 cell's gap pixels as zeros): 375 / 356 / 461 us on ResNet-50's three
    // projection shortcuts against 662 / 843 / 1116 us for the tile kernel's per-pixel zero
    // skip, which had beaten the earlier output-pixel-row GEMM (1145 us: 3/4 of its FMAs
    // were spent on the stride gaps).  SPC_S2_BWI_GEMM=0 selects the tile kernel (A/B).
    const bool pw_s2_bwi = !fwd && sh.R == 1 && sh.S == 1 && sh.O == 2 && sh.P == 2;
    static const bool s2_gemm = !(std::getenv("SPC_S2_BWI_GEMM") && std::atoi(std::getenv("SPC_S2_BWI_GEMM")) == 0);
    const bool s2_bwi_tile = pw_s2_bwi && !s2_gemm && tile_conv_supported(fwd, sh, V);
    if (!force_generic && !pw_off && !s2_bwi_tile && use_pw_gemm() && pw_gemm_supported(fwd, sh, V)) {
        int* finite = stream_flags(st) ? stream_flags(st) + FLAG_FINITE : nullptr;
        cudaError_t e = finite ? cudaSuccess : cudaErrorMemoryAllocation;
        if (e != cudaSuccess) return e;
        launch_finite_all(filt, (size_t)sh.K * sh.C, finite, st);
        e = launch_pw_gemm(fwd, sparse, sh, src, filt, dst, exec_ctr, finite, st, epi);
        return e;
    }
    if (!force_generic && !pw_off && !s2_bwi_tile && pw_conv_supported(fwd, sh, V)) {
        int* finite = stream_flags(st) ? stream_flags(st) + FLAG_FINITE : nullptr;
        cudaError_t e = finite ? cudaSuccess : cudaErrorMemoryAllocation;
        if (e != cudaSuccess) return e;
        launch_filter_finite(filt, (size_t)sh.K * sh.C, finite, st);
        e = launch_pw_conv(fwd, sparse, sh, src, filt, dst, exec_ctr, st, finite, epi, gate);
        // filters with Inf/NaN: the per-element-skip tile kernel (exits otherwise)
        if (e == cudaSuccess) e = launch_tile_conv(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi, finite, 0, gate);
        return e;
    }
    if (!force_generic && tile_conv_supported(fwd, sh, V))
        return launch_tile_conv(fwd, sparse, sh, src, filt, dst, exec_ctr, st, epi, nullptr, 0, gate);
    cudaError_t e = launch_conv_generic(fwd, sparse, sh, V, src, filt, dst, exec_ctr, st);
    if (e != cudaSuccess) return e;
    const size_t n = (size_t)sh.N * (fwd ? (size_t)sh.K * sh.Hp * sh.Wp : (size_t)sh.C * sh.H * sh.W);
    return launch_epilogue(epi, dst, n, st);
}

cudaError_t launch_bww(bool check_input, bool sparse, const DevShape& sh, int V, const float* chk,
                       const float* oth, float* dst, unsigned long long* exec_ctr, cudaStream_t st) {
    static const bool force_generic = std::getenv("SPC_FORCE_GENERIC") && std::atoi(std::getenv("SPC_FORCE_GENERIC"));
    static const bool pw_off = std::getenv("SPC_PW_OFF") && std::atoi(std::getenv("SPC_PW_OFF"));
    if (g_math == SPC_MATH_TF32X3 && tc_bww_supported(sh, V))
        return launch_tc_bww(check_input, sparse, sh, chk, oth, dst, exec_ctr, st);
    if (!force_generic && !pw_off && pw_bww_supported(check_input, sh, V)) {
        int* finite = stream_flags(st) ? stream_flags(st) + FLAG_FINITE : nullptr;
        cudaError_t e = finite ? cudaSuccess : cudaErrorMemoryAllocation;
        if (e != cudaSuccess) return e;
        launch_finite_all(oth, (size_t)sh.N * sh.K * sh.Hp * sh.Wp, finite, st);  // dY (ActNCHWc)
        e = launch_pw_bww(sparse, sh, chk, oth, dst, exec_ctr, finite, st);
        return e;
    }
    // V=16 tile kernels (tile_bww.cu), except 3x3 s1 check=input with 64-channel
    // lane blocks (K % 128 != 0: VGG conv1_2, ResNet stage 1), where the
    // row-window kernel (row_bww.cu, KK=2) measured 4-22% faster at every
    // sparsity; on the 128-multiple layers it is 8-30% slower.
    // SPC_ROW_BWW=0 / 1 forces the tile / row kernel (A/B).  Both add d * 0 for taps whose partner pixel lies
    // outside the image (zero-filled staging), exact only for a FINITE checked
    // tensor: a device scan of it picks, for Inf/NaN, the shape-general
    // kernel (exact skips, P/src/kernel_impl.hpp:239-304).  All are enqueued;
    // the non-matching ones exit at entry (no host sync).
    static const int row_env = std::getenv("SPC_ROW_BWW") ? std::atoi(std::getenv("SPC_ROW_BWW")) : -1;
    const bool row_pick = row_env == 1 || (row_env == -1 && sh.K % 128 != 0);
    const bool use_row = !force_generic && row_pick && row_bww_supported(check_input, sh, V);
    // 3x3 s1 check=input with 128-multiple lane blocks: the TMA-staged tile kernel
    // (tma_bww.cu), 7-10% faster than the cp.async tile kernel at every sparsity
    // of the VGG sweep.  SPC_TMA_BWW=0 keeps the cp.async kernel (A/B); =2 (DEV
    // build) also takes the 64-channel layers from the row kernel.
    static const int tma_env = std::getenv("SPC_TMA_BWW") ? std::atoi(std::getenv("SPC_TMA_BWW")) : 1;
    const bool use_tma = !force_generic && (!use_row || tma_env == 2) && tma_env >= 1 && row_env != 1 &&
                         tma_bww_supported(check_input, sh, V);
    if (use_row || use_tma || (!force_generic && tile_bww_supported(check_input, sh, V))) {
        const size_t chk_n = (size_t)((sh.N + 15) / 16) * 16 *
                             (check_input ? (size_t)sh.C * sh.H * sh.W : (size_t)sh.K * sh.Hp * sh.Wp);
        int* finite = stream_flags(st) ? stream_flags(st) + FLAG_FINITE : nullptr;
        cudaError_t e = finite ? cudaSuccess : cudaErrorMemoryAllocation;
        if (e != cudaSuccess) return e;
        if (!use_tma) launch_finite_all(chk, chk_n, finite, st);  // the TMA kernel's pre-pass scans as it transposes
        const bool counted = !use_row && !use_tma && tile_bww_counted_dense(check_input, sh);
        if (counted)  // every FMA runs: dY must be finite too
            launch_finite_also(oth, (size_t)sh.N * sh.K * sh.Hp * sh.Wp, finite, st);
        e = use_row && !use_tma ? launch_row_bww_when(sparse, sh, chk, oth, dst, exec_ctr, finite, st)
            : use_tma ? launch_tma_bww_when(sparse, sh, chk, oth, dst, exec_ctr, finite, 1, st, finite)
                      : launch_tile_bww_when(check_input, sparse, sh, chk, oth, dst, exec_ctr, st, finite, 1, counted);
        if (e == cudaSuccess) {
            const int gs = bww_generic_splits(sh);
            const size_t E = (size_t)sh.K * sh.C * sh.S * sh.R;
            float* partial = nullptr;
            e = cudaMallocAsync((void**)&partial, (size_t)gs * E * sizeof(float), st);
            if (e == cudaSuccess) {
                e = launch_bww_generic(check_input, sparse, sh, V, chk, oth, partial, gs, dst, exec_ctr, st, finite, 0);
                cudaFreeAsync(partial, st);
            }
        }
        return e;
    }
    const int splits = bww_generic_splits(sh);
    const size_t E = (size_t)sh.K * sh.C * sh.S * sh.R;
    float* partial = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)splits * E * sizeof(float), st);
    if (e != cudaSuccess) return e;
    e = launch_bww_generic(check_input, sparse, sh, V, chk, oth, partial, splits, dst, exec_ctr, st);
    cudaFreeAsync(partial, st);
    return e;
}

}  // namespace spc
