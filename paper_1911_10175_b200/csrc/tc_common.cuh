// tc_common.cuh -- tcgen05 / TMA / mbarrier helpers shared by the 3xTF32
// tensor-core kernels (tc_conv.cu FWD/BWI, tc_bww.cu BWW).  Inline PTX for
// sm_100a; the descriptor bit layouts follow the PTX ISA tcgen05 "shared
// memory descriptor" and "instruction descriptor" tables.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>

namespace spc {
namespace tc {

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
           | ((uint32_t)(128 >> 4) << 24);  // M = 128
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

// UMMA descriptor, MN-major, SWIZZLE_64B: atoms of 16 MN-elements (64 B) x 8
// K-rows (64 B apart); `lbo` = byte stride between MN atoms, `sbo` = byte
// stride between 8-row K groups.
__device__ __forceinline__ uint64_t sw64_mn_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr & 0x3FFFFu) >> 4);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)4 << 61;
    return d;
}
// Instruction descriptor: kind::tf32, D = f32, M = 128, N = bn; a_mn / b_mn
// select MN-major operands.
__device__ __forceinline__ uint32_t tf32_idesc_rt(int bn, int a_mn, int b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
           ((uint32_t)(bn >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// host: cuTensorMapEncodeTiled through the runtime's driver entry point
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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
// A [N][CB][H][W][16] fp32 tensor (ActNCHWc) as a 5-D map with box
// {16, b1 (x), b2 (y), b3 (channel blocks), 1}, SWIZZLE_64B, OOB -> 0.
// `str` = traversal stride over x and y (the box then spans str * b1 x str * b2
// source pixels and lands b1 x b2 of them).
inline bool make_act_map(CUtensorMap* m, const float* p, int N, int CB, int H, int W, int b1, int b2, int b3,
                         int str = 1) {
    cuuint64_t dims[5] = {16, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)CB, (cuuint64_t)N};
    cuuint64_t strides[4] = {64, (cuuint64_t)W * 64, (cuuint64_t)H * W * 64, (cuuint64_t)CB * H * W * 64};
    cuuint32_t box[5] = {16, (cuuint32_t)(b1 * str), (cuuint32_t)(b2 * str), (cuuint32_t)b3, 1};
    cuuint32_t es[5] = {1, (cuuint32_t)str, (cuuint32_t)str, 1, 1};
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(p), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// A contiguous 5-D fp32 tensor with dims d[0] (innermost, 16 floats = 64 B)
// .. d[4], box b[0..4], SWIZZLE_64B, OOB -> 0.
inline bool make_map5(CUtensorMap* m, const float* p, const int (&d)[5], const int (&b)[5]) {
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    cuuint64_t st = 4;
    for (int i = 0; i < 5; ++i) {
        dims[i] = (cuuint64_t)d[i];
        box[i] = (cuuint32_t)b[i];
        st *= (cuuint64_t)d[i];
        if (i < 4) strides[i] = st;
    }
    return encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(p), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---------------------------------------------------------------- shared by the tcgen05 kernels
constexpr int TC_BM = 128;
constexpr int TC_ST = 4;          // pipeline stages
constexpr int TC_THREADS = 320;       // BWW: TMA, MMA, 8 drain / epilogue warps
constexpr int TC_CONV_THREADS = 384;  // FWD/BWI: + 2 warps that split A into hi / lo in shared memory
// TMEM allocations are powers of two >= 32 columns
constexpr int tmem_cols(int n) { return n <= 32 ? 32 : n <= 64 ? 64 : n <= 128 ? 128 : n <= 256 ? 256 : 512; }

// CTA-pair (cluster of 2, cta_group::2) forms: the TMA loads signal the
// leader CTA's barrier (peer bit cleared), the MMA reads both CTAs' shared
// memory, the commit is multicast to both CTAs.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_to_rank0(uint32_t addr) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(addr));
    return r;
}
__device__ __forceinline__ void tma_load_5d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2, int c3, int c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(bar & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1,
                                                 int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar & 0xFEFFFFFFu)
        : "memory");
}
__device__ __forceinline__ void umma_tf32_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(bar)
        : "memory");
}

// Prep kernels shared by the FWD/BWI (tc_conv.cu) and BWW (tc_bww.cu)
// launchers, defined in tc_prep.cu.
__global__ void tc_split_src_kernel(const float* __restrict__ src, float* __restrict__ lo, size_t n4, int Hs,
                                    int Ws, int Ho, int Wo, int R, int S, int padW, int padH, int bwi,
                                    unsigned scale, unsigned long long* __restrict__ cnt,
                                    int* __restrict__ nonfinite, int str = 1,
                                    uint8_t* __restrict__ rowflag = nullptr);
__global__ void tc_zero_kernel(int* flag, unsigned long long* cnt);

}  // namespace tc
}  // namespace spc
