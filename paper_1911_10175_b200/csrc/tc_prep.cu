// tc_prep.cu -- prep kernels shared by the 3xTF32 tensor-core launchers
// (tc_conv.cu FWD/BWI, tc_bww.cu BWW): the source split / exact counter /
// non-finite scan, and the scratch reset.
#include <cstdint>

#include "common.cuh"
#include "tc_common.cuh"

namespace spc {
namespace tc {

// lo = x - tf32_trunc(x) over the source; counts executed_vector_fmas the
// reference's way (P/src/oracle.cpp:160-230): every nonzero source element
// adds rows(y) * cols(x), scaled by Co/16 at the end; flags non-finite values.
__global__ void tc_split_src_kernel(const float* __restrict__ src, float* __restrict__ lo, size_t n4, int Hs,
                                    int Ws, int Ho, int Wo, int R, int S, int padW, int padH, int bwi,
                                    unsigned scale, unsigned long long* __restrict__ cnt,
                                    int* __restrict__ nonfinite, int str,
                                    uint8_t* __restrict__ rowflag) {
    unsigned long long acc = 0;
    int bad = 0;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n4; e += (size_t)gridDim.x * blockDim.x) {
        const float4 x = __ldg(reinterpret_cast<const float4*>(src) + e);
        if (rowflag) {
            // rowflag[(image, channel block, row)] = 1 once the row holds a nonzero
            // (zero-tile skip); a warp's 32 float4 nearly always share one row:
            // one store for the warp then, per-lane stores otherwise (benign races,
            // flags only go 0 -> 1)
            const size_t row = e / (4 * (size_t)Ws);
            const bool nz = x.x != 0.0f || x.y != 0.0f || x.z != 0.0f || x.w != 0.0f;
            const unsigned act = __activemask();
            const size_t row0 = __shfl_sync(act, row, __ffs(act) - 1);
            if (__all_sync(act, row == row0)) {
                if (__any_sync(act, nz) && (int)(threadIdx.x & 31) == __ffs(act) - 1) rowflag[row0] = 1;
            } else if (nz) {
                rowflag[row] = 1;
            }
        }
        if (lo) {
            float4 l;
            l.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
            l.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
            l.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
            l.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
            reinterpret_cast<float4*>(lo)[e] = l;
        }
        bad |= !isfinite(x.x) | !isfinite(x.y) | !isfinite(x.z) | !isfinite(x.w);
        const unsigned nz = (x.x != 0.0f) + (x.y != 0.0f) + (x.z != 0.0f) + (x.w != 0.0f);
        if (nz && cnt) {
            const size_t pix = (e * 4) / 16;  // (image, channel block, y, x) pixel of the 16-lane vector
            const int xx = (int)(pix % Ws);
            const int yy = (int)((pix / Ws) % Hs);
            int rows = 0, cols = 0;
            // FWD: output rows y' with y'*str + v - pad = y (oracle.cpp:160-190);
            // BWI: input rows y = y'*str + v - pad inside the image (:195-230)
            for (int v = 0; v < S; ++v) {
                if (bwi) {
                    const int o = yy * str + v - padH;
                    rows += (o >= 0 && o < Ho) ? 1 : 0;
                } else {
                    const int n = yy + padH - v;
                    rows += (n >= 0 && n % str == 0 && n / str < Ho) ? 1 : 0;
                }
            }
            for (int u = 0; u < R; ++u) {
                if (bwi) {
                    const int o = xx * str + u - padW;
                    cols += (o >= 0 && o < Wo) ? 1 : 0;
                } else {
                    const int n = xx + padW - u;
                    cols += (n >= 0 && n % str == 0 && n / str < Wo) ? 1 : 0;
                }
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

__global__ void tc_zero_kernel(int* flag, unsigned long long* cnt) {
    *flag = 0;
    *cnt = 0;
}
}  // namespace tc
}  // namespace spc
