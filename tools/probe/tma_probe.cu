// Standalone probe: does a 5-D TMA load with permuted (non-monotonic) strides work, and the 4-D halo box?
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
#include "../../paper_1911_10175_b200/csrc/tc_common.cuh"
using namespace spc::tc;

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                 ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar) : "memory");
}

__global__ void probe5(const __grid_constant__ CUtensorMap m, float* out, int nfl, int kb0, int x0, int y0, int n) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint32_t sb = smem_u32(smem), bar = sb + nfl * 4;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, nfl * 4);
        tma_load_5d(sb, &m, bar, 0, kb0, x0, y0, n);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < nfl; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}
__global__ void probe4(const __grid_constant__ CUtensorMap m, float* out, int nfl, int x0, int y0, int c0, int n) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint32_t sb = smem_u32(smem), bar = sb + nfl * 4;
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(bar, nfl * 4);
        tma_load_4d(sb, &m, bar, x0, y0, c0, n);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    for (int i = threadIdx.x; i < nfl; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)
int main(int argc, char** argv) {
    const int var = argc > 1 ? atoi(argv[1]) : 0;
    const int N = 2, K = 128, Hp = 14, Wp = 14, TH = 7, TW = 4, KB = K / 16;
    std::vector<float> h((size_t)N * K * Hp * Wp);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *out;
    CK(cudaMalloc(&d, h.size() * 4));
    CK(cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    const int nfl = TH * TW * 128;
    CK(cudaMalloc(&out, nfl * 4));
    CUtensorMap m;
    const cuuint64_t hw = (cuuint64_t)Hp * Wp;
    cuuint64_t dims[5] = {16, (cuuint64_t)KB, (cuuint64_t)Wp, (cuuint64_t)Hp, (cuuint64_t)N};
    cuuint64_t strides[4] = {hw * 64, 64, (cuuint64_t)Wp * 64, (cuuint64_t)KB * hw * 64};
    cuuint32_t box[5] = {16, 8, TW, TH, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode5 (permuted strides): %d\n", (int)r);
    if (r == CUDA_SUCCESS && var == 0) {
        CK(cudaFuncSetAttribute(probe5, cudaFuncAttributeMaxDynamicSharedMemorySize, nfl * 4 + 64));
        const int x0 = 12, y0 = 7, n = 1;
        probe5<<<1, 128, nfl * 4 + 64>>>(m, out, nfl, 0, x0, y0, n);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(nfl);
        CK(cudaMemcpy(o.data(), out, nfl * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int q = 0; q < TH * TW; ++q) for (int k = 0; k < 128; ++k) {
            int y = y0 + q / TW, x = x0 + q % TW;
            float want = (y < Hp && x < Wp) ? h[(((size_t)n * KB + k / 16) * Hp + y) * Wp * 16 + (size_t)x * 16 + k % 16] : 0.f;
            if (o[q * 128 + k] != want) { if (bad < 5) printf("5d mismatch q %d k %d got %f want %f\n", q, k, o[q * 128 + k], want); ++bad; }
        }
        printf("probe5: %d mismatches\n", bad);
    }
    // 4-D planes [N][C][H][Wpitch]
    const int C = 16, H = 14, W = 14, Wpitch = 16;
    std::vector<float> hp((size_t)N * C * H * Wpitch);
    for (size_t i = 0; i < hp.size(); ++i) hp[i] = (float)(i + 1);
    float* dp;
    CK(cudaMalloc(&dp, hp.size() * 4));
    CK(cudaMemcpy(dp, hp.data(), hp.size() * 4, cudaMemcpyHostToDevice));
    cuuint64_t d4[4] = {(cuuint64_t)(var == 1 ? Wpitch : W), (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
    cuuint64_t s4[3] = {(cuuint64_t)Wpitch * 4, (cuuint64_t)H * Wpitch * 4, (cuuint64_t)C * H * Wpitch * 4};
    cuuint32_t b4[4] = {8, 9, 8, 1};
    const int x0 = var == 2 ? 4 : var == 3 ? -1 : var == 5 ? 5 : var == 6 ? 12 : var == 7 ? 4 : var == 8 ? -4 : 11, y0 = (var == 4 || var == 7) ? -1 : 6;
    cuuint32_t e4[4] = {1, 1, 1, 1};
    CUtensorMap m4;
    r = encode_fn()(&m4, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dp, d4, s4, b4, e4, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode4: %d\n", (int)r);
    if (r == CUDA_SUCCESS) {
        const int nf4 = 8 * 9 * 8;
        CK(cudaFuncSetAttribute(probe4, cudaFuncAttributeMaxDynamicSharedMemorySize, nf4 * 4 + 64));
        const int c0 = 8, n = 1;
        probe4<<<1, 128, nf4 * 4 + 64>>>(m4, out, nf4, x0, y0, c0, n);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(nf4);
        CK(cudaMemcpy(o.data(), out, nf4 * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (int c = 0; c < 8; ++c) for (int ry = 0; ry < 9; ++ry) for (int rx = 0; rx < 8; ++rx) {
            int y = y0 + ry, x = x0 + rx;
            float want = (y >= 0 && y < H && x >= 0 && x < (var == 1 ? Wpitch : W)) ? hp[(((size_t)n * C + c0 + c) * H + y) * Wpitch + x] : 0.f;
            float got = o[(c * 9 + ry) * 8 + rx];
            if (got != want) { if (bad < 5) printf("4d mismatch c %d ry %d rx %d got %f want %f\n", c, ry, rx, got, want); ++bad; }
        }
        printf("probe4: %d mismatches\n", bad);
    }
    return 0;
}
