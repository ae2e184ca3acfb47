// pw_bww.cu -- BWW for 1x1 convs (stride 1/2), check = input, V = 16.
//
// dG[k, c] = sum over images i and output pixels o of D[i, c, s(o)] * dY[i, k, o]
// (P/src/kernel_impl.hpp:209-336 for R = S = 1), i.e. a GEMM dY[K x R] . D[C x R]^T
// with the reduction index r = (16-image block, output pixel, image lane).
//
// Like the 1x1 FWD/BWI kernel (pw_conv.cu), this executes every FMA: a checked
// D element feeds only a few FMAs per thread, and no zero-check granularity beat
// dense FMAs on B200 for 1x1.  Zero products are exact for finite dY; when dY
// holds Inf/NaN (0*Inf = NaN where the reference skips) the EXACT instantiation
// runs instead, which applies an FMA only where the checked D value is nonzero
// (device-side flag, both launched, one exits at entry).
// executed_vector_fmas is the reference's exact count (nonzero staged D
// elements x K/16).
//
// Mapping: SGEMM-style register blocking.  A CTA owns a BK x BC tile of dG and
// a fixed range of r; each thread an 8 x 8 (k x c) sub-tile (FFMA2 over k
// pairs, the c value broadcast).  Per r-chunk (one output pixel x 16 images)
// the CTA stages
//   Ds[c][r]        from ActCHWNn [nb][C][H][W][16]: 64 contiguous bytes per
//                   (c, pixel) -- 16-byte cp.async, no transpose;
//   Ys[k/2][r][2]   from ActNCHWc dY [N][K/16][H'][W'][16]: a 4-byte
//                   transposing cp.async per element, laid out so one LDS.128
//                   yields two k-pairs for two r (the FFMA2 operands);
// 4 stages deep.  Rows are padded so the per-thread LDS.128 are conflict-free.
// Partials per split, then a fixed-order reduction into FilterKCRSblk (K, C):
// bitwise deterministic, no float atomics.
#include <cstdint>

#include "common.cuh"
#include "pw_bww.h"

namespace spc {
namespace {

constexpr int PB_RT = 16;           // r per chunk: one output pixel x 16 images
constexpr int PB_NST = 4;           // pipeline depth
constexpr int PB_DS = PB_RT + 4;    // padded Ds row (floats)
constexpr int PB_YS = 2 * PB_RT + 4;  // padded Ys row (floats): 16 r x 2 k

__device__ __forceinline__ uint32_t pb_smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int BK, int BC, int STR, bool COUNT, bool EXACT>
__global__ void __launch_bounds__((BK / 8) * (BC / 8)) pw_bww_kernel(DevShape sh, const float* __restrict__ dchw,
                                                                    const float* __restrict__ dy,
                                                                    float* __restrict__ partial, int splits,
                                                                    unsigned long long* __restrict__ exec_ctr,
                                                                    const int* __restrict__ finite) {
    if ((__ldg(finite) != 0) == EXACT) return;  // EXACT runs only for a dY with Inf/NaN
    constexpr int NT = (BK / 8) * (BC / 8);
    extern __shared__ __align__(16) float smem[];
    float* Ds = smem;                                  // [NST][BC][PB_DS]
    float* Ys = smem + PB_NST * BC * PB_DS;            // [NST][BK/2][PB_YS]

    const int Hs = sh.H, Ws = sh.W, Wo = sh.Wp, HWo = sh.Hp * sh.Wp;
    const int KB = sh.K / 16;
    const int nb_total = (sh.N + 15) / 16;
    const int ktile = blockIdx.x, ctile = blockIdx.y, split = blockIdx.z;
    const int k_base = ktile * BK, c_base = ctile * BC;
    // this split's chunk range over (nb, o)
    const long nchunks = (long)nb_total * HWo;
    const long ch0 = nchunks * split / splits, ch1 = nchunks * (split + 1) / splits;
    const int nsteps = (int)(ch1 - ch0);

    const int tid = threadIdx.x;
    const int tx = tid % (BC / 8), ty = tid / (BC / 8);

    // staging of one chunk (nb, o) into buffer buf
    auto stage = [&](int step, int buf) {
        if (step < nsteps) {
            const long chk = ch0 + step;
            const int nb = (int)(chk / HWo), o = (int)(chk % HWo);
            const int oy = o / Wo, ox = o - oy * Wo;
            const int sidx = (oy * STR) * Ws + ox * STR;
            // Ds[c][r]: BC rows x 4 chunks of 16 B
            const uint32_t dbase = pb_smem_u32(Ds + (size_t)buf * BC * PB_DS);
            for (int t = tid; t < BC * 4; t += NT) {
                const int c = t >> 2, q = t & 3;
                const float* g = dchw + (((size_t)nb * sh.C + (c_base + c)) * Hs * Ws + sidx) * 16 + q * 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dbase + (uint32_t)(c * PB_DS + q * 4) * 4u),
                             "l"(g));
            }
            // Ys[k/2][r][2]: BK x 16 elements, 4-byte transposing copies (lane = image)
            const uint32_t ybase = pb_smem_u32(Ys + (size_t)buf * (BK / 2) * PB_YS);
            for (int t = tid; t < BK * 16; t += NT) {
                const int kk = t & 15, rest = t >> 4;  // kk fastest: 16 k of one (image, k-block) are contiguous
                const int lane = rest % 16, kb = rest / 16;
                const int k = kb * 16 + kk;  // within the tile
                const int img = nb * 16 + lane;
                const bool ok = img < sh.N;
                const float* g = dy + ((((size_t)(ok ? img : 0) * KB + (k_base + k) / 16) * HWo + o) * 16 + (k_base + k) % 16);
                const uint32_t d = ybase + (uint32_t)((k >> 1) * PB_YS + lane * 2 + (k & 1)) * 4u;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(g), "r"(ok ? 4 : 0));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };

    // accumulators: 4 k-pairs x 8 c, as float2 (k, k+1)
    float2 acc[4][8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.0f, 0.0f);
    // thread sub-tile: k pairs {ty*2, ty*2+1} and {BK/4 + ty*2, +1}; c = tx + (BC/8)*j, j < 8
    // (strided c rows: the 8 lanes of an LDS.128 phase hit 8 different 16-byte bank groups)
    const int kp0 = ty * 2, kp1 = BK / 4 + ty * 2;
    uint32_t nz = 0;

#pragma unroll
    for (int d = 0; d < PB_NST - 1; ++d) stage(d, d);
    for (int step = 0; step < nsteps; ++step) {
        stage(step + PB_NST - 1, (step + PB_NST - 1) % PB_NST);
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PB_NST - 1));
        __syncthreads();
        const float* D = Ds + (size_t)(step % PB_NST) * BC * PB_DS;
        const float* Y = Ys + (size_t)(step % PB_NST) * (BK / 2) * PB_YS;
        if (COUNT && ktile == 0) {
            // exact counter: nonzero checked elements of this chunk (each staged once per c-tile)
            for (int t = tid; t < BC * PB_RT; t += NT) nz += D[(t / PB_RT) * PB_DS + (t % PB_RT)] != 0.0f;
        }
#pragma unroll
        for (int r0 = 0; r0 < PB_RT; r0 += 4) {
            float4 b[8];  // c_j at r0..r0+3
#pragma unroll
            for (int j = 0; j < 8; ++j) b[j] = *reinterpret_cast<const float4*>(D + (tx + (BC / 8) * j) * PB_DS + r0);
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // r0 + 2h, r0 + 2h + 1
                float4 a[4];  // per k-pair row: {k,k+1 @ r}, {k,k+1 @ r+1}
                a[0] = *reinterpret_cast<const float4*>(Y + (kp0 + 0) * PB_YS + (r0 + 2 * h) * 2);
                a[1] = *reinterpret_cast<const float4*>(Y + (kp0 + 1) * PB_YS + (r0 + 2 * h) * 2);
                a[2] = *reinterpret_cast<const float4*>(Y + (kp1 + 0) * PB_YS + (r0 + 2 * h) * 2);
                a[3] = *reinterpret_cast<const float4*>(Y + (kp1 + 1) * PB_YS + (r0 + 2 * h) * 2);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 p0 = make_float2(a[i].x, a[i].y), p1 = make_float2(a[i].z, a[i].w);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float v0 = h ? b[j].z : b[j].x, v1 = h ? b[j].w : b[j].y;
                        if constexpr (EXACT) {  // skip zero checked values, as the reference does
                            if (v0 != 0.0f) acc[i][j] = __ffma2_rn(p0, make_float2(v0, v0), acc[i][j]);
                            if (v1 != 0.0f) acc[i][j] = __ffma2_rn(p1, make_float2(v1, v1), acc[i][j]);
                        } else {
                            acc[i][j] = __ffma2_rn(p0, make_float2(v0, v0), acc[i][j]);
                            acc[i][j] = __ffma2_rn(p1, make_float2(v1, v1), acc[i][j]);
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    // partial[split][c][k] (the reduce kernel's layout)
    float* P = partial + (size_t)split * sh.C * sh.K;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int kp = i < 2 ? kp0 + i : kp1 + (i - 2);
        const int k = k_base + 2 * kp;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = c_base + tx + (BC / 8) * j;
            *reinterpret_cast<float2*>(P + (size_t)c * sh.K + k) = acc[i][j];
        }
    }
    if (COUNT && ktile == 0 && exec_ctr) {
        const uint32_t total = __reduce_add_sync(0xffffffffu, nz);
        if ((tid & 31) == 0 && total) atomicAdd(exec_ctr, (unsigned long long)total * (sh.K / 16));
    }
}

// fixed-order split sum -> FilterKCRSblk (K, C), R = S = 1
__global__ void pw_bww_reduce(int C, int K, const float* __restrict__ partial, int splits, float* __restrict__ dst,
                              const int* __restrict__ only_if_nonfinite) {
    if (only_if_nonfinite != nullptr && __ldg(only_if_nonfinite) != 0) return;
    const size_t E = (size_t)C * K;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < E; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int z = 0; z < splits; ++z) s += partial[(size_t)z * E + e];
        const int k = (int)(e % K), c = (int)(e / K);
        dst[((size_t)(k / 16) * (C / 16) + c / 16) * 256 + (c % 16) * 16 + k % 16] = s;
    }
}

// flag = 1 when every element is finite (grid-stride; flag preset to 1)
__global__ void finite_all_kernel(const float* __restrict__ t, size_t n, int* flag) {
    int bad = 0;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n / 4; e += (size_t)gridDim.x * blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(t) + e);
        bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
    }
    for (size_t e = (n / 4) * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
         e += (size_t)gridDim.x * blockDim.x)
        bad |= !isfinite(t[e]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 0);
}
__global__ void set_one_kernel(int* flag) { *flag = 1; }

template <int BK, int BC, int STR>
cudaError_t pb_launch(bool sparse, const DevShape& sh, const float* dchw, const float* dy, float* dst,
                      unsigned long long* exec_ctr, const int* finite, cudaStream_t st, bool exact_only) {
    constexpr int NT = (BK / 8) * (BC / 8);
    const size_t smem = (size_t)PB_NST * (BC * PB_DS + (BK / 2) * PB_YS) * sizeof(float);
    const long tiles = (long)(sh.K / BK) * (sh.C / BC);
    const long nchunks = (long)((sh.N + 15) / 16) * sh.Hp * sh.Wp;
    long splits = (148L * 4 + tiles - 1) / tiles;  // ~2 CTAs per SM, 2 waves
    if (splits > nchunks) splits = nchunks;
    if (splits < 1) splits = 1;
    float* partial = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&partial, (size_t)splits * sh.C * sh.K * sizeof(float), st);
    if (e != cudaSuccess) return e;
    auto k0 = sparse ? pw_bww_kernel<BK, BC, STR, true, false> : pw_bww_kernel<BK, BC, STR, false, false>;
    auto k1 = sparse ? pw_bww_kernel<BK, BC, STR, true, true> : pw_bww_kernel<BK, BC, STR, false, true>;
    cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(sh.K / BK, sh.C / BC, (unsigned)splits);
    // exact_only: the finite case is tma_pw_bww.cu's (already enqueued); this is its Inf / NaN fallback
    if (!exact_only) k0<<<grid, NT, smem, st>>>(sh, dchw, dy, partial, (int)splits, exec_ctr, finite);
    k1<<<grid, NT, smem, st>>>(sh, dchw, dy, partial, (int)splits, exec_ctr, finite);
    note_launch(exact_only ? 1 : 2);
    e = cudaGetLastError();
    if (e == cudaSuccess) {
        unsigned rb = (unsigned)(((size_t)sh.C * sh.K + 255) / 256);
        if (rb > 148 * 8) rb = 148 * 8;
        pw_bww_reduce<<<rb, 256, 0, st>>>(sh.C, sh.K, partial, (int)splits, dst, exact_only ? finite : nullptr);
        note_launch();
        e = cudaGetLastError();
    }
    cudaFreeAsync(partial, st);
    return e;
}

}  // namespace

bool pw_bww_supported(bool check_input, const DevShape& sh, int V) {
    if (!check_input || V != 16 || sh.R != 1 || sh.S != 1 || sh.O != sh.P || sh.padW || sh.padH) return false;
    if (sh.O != 1 && sh.O != 2) return false;
    return sh.C % 64 == 0 && sh.K % 64 == 0;
}

cudaError_t launch_pw_bww(bool sparse, const DevShape& sh, const float* dchw, const float* dy, float* dst,
                          unsigned long long* exec_ctr, const int* finite, cudaStream_t st) {
    const bool k128 = sh.K % 128 == 0, c128 = sh.C % 128 == 0;
    // finite dY: the TMA-staged GEMM (tma_pw_bww.cu); this file's EXACT kernel stays its Inf / NaN fallback
    bool exact_only = false;
    if (tma_pw_bww_supported(sh)) {
        const cudaError_t e = launch_tma_pw_bww(sparse, sh, dchw, dy, dst, exec_ctr, finite, st);
        if (e != cudaSuccess) return e;
        exact_only = true;
    }
#define PB_L(BK, BC)                                                                                       \
    return sh.O == 1 ? pb_launch<BK, BC, 1>(sparse, sh, dchw, dy, dst, exec_ctr, finite, st, exact_only)  \
                     : pb_launch<BK, BC, 2>(sparse, sh, dchw, dy, dst, exec_ctr, finite, st, exact_only)
    if (k128 && c128) PB_L(128, 128);
    if (k128) PB_L(128, 64);
    if (c128) PB_L(64, 128);
    PB_L(64, 64);
#undef PB_L
}

void launch_set_flag(int* flag, cudaStream_t st) {
    set_one_kernel<<<1, 1, 0, st>>>(flag);
    note_launch();
}

// AND another tensor's finiteness into a flag launch_finite_all already wrote
void launch_finite_also(const float* t, size_t n, int* flag, cudaStream_t st) {
    finite_all_kernel<<<148 * 4, 256, 0, st>>>(t, n, flag);
    note_launch();
}

void launch_finite_all(const float* t, size_t n, int* flag, cudaStream_t st) {
    set_one_kernel<<<1, 1, 0, st>>>(flag);
    finite_all_kernel<<<148 * 4, 256, 0, st>>>(t, n, flag);
    note_launch(2);
}

}  // namespace spc
