// generic.cu -- shape-general sm_100a kernels for all three passes.
//
// These cover every geometry and vector width the reference accepts
// (V in {4, 8, 16}, any R/S/stride/padding).  The tuned V=16 tile kernels
// (tile_conv.cu, tile_bww.cu) take over for the shapes they support.
//
// Zero skipping is warp-uniform by construction: the lanes of a warp own
// different OUTPUT channels of the same output pixel, so every lane reads the
// same checked element d and `d != 0.0f` (IEEE: -0 is zero, NaN is not,
// P/include/spconv/vec.hpp:120-128) branches the whole warp together.
#include "common.cuh"

namespace spc {

// FWD (IsFwd) and BWI share one body with channel roles swapped, exactly as
// the reference shares conv_row_task<VB, IsFwd> (P/src/kernel_impl.hpp:51-202):
//   FWD: Y[i,k,y',x']  += D[i,c,y'P+v-padH, x'O+u-padW] * G[k,c,v,u]
//   BWI: dD[i,c,y,x]   += dY[i,k,y',x'] * Gt[c,k,v,u],  y = y'P+v-padH, x = x'O+u-padW
// One CTA per (image, output pixel) x block of output channels.
template <bool IsFwd, bool Sparse>
__global__ void __launch_bounds__(128) conv_generic_kernel(DevShape sh, int V, const float* __restrict__ src,
                                                           const float* __restrict__ filt,
                                                           float* __restrict__ dst,
                                                           unsigned long long* __restrict__ exec_ctr) {
    const int Co = IsFwd ? sh.K : sh.C, Ci = IsFwd ? sh.C : sh.K;
    const int Hs = IsFwd ? sh.H : sh.Hp, Ws = IsFwd ? sh.W : sh.Wp;
    const int Ho = IsFwd ? sh.Hp : sh.H, Wo = IsFwd ? sh.Wp : sh.W;
    long pix = blockIdx.x;
    const int xo = (int)(pix % Wo);
    pix /= Wo;
    const int yo = (int)(pix % Ho);
    const int i = (int)(pix / Ho);
    const int co = blockIdx.y * blockDim.x + threadIdx.x;
    const bool active = co < Co;
    float acc = 0.0f;
    unsigned cnt = 0;
    if (active) {
        const int cib = Ci / V;
        for (int v = 0; v < sh.S; ++v) {
            int ys;
            if (IsFwd) {
                ys = yo * sh.P + v - sh.padH;
                if (ys < 0 || ys >= Hs) continue;
            } else {
                const int num = yo + sh.padH - v;
                if (num < 0 || num % sh.P != 0) continue;
                ys = num / sh.P;
                if (ys >= Hs) continue;
            }
            for (int u = 0; u < sh.R; ++u) {
                int xs;
                if (IsFwd) {
                    xs = xo * sh.O + u - sh.padW;
                    if (xs < 0 || xs >= Ws) continue;
                } else {
                    const int num = xo + sh.padW - u;
                    if (num < 0 || num % sh.O != 0) continue;
                    xs = num / sh.O;
                    if (xs >= Ws) continue;
                }
                for (int cb = 0; cb < cib; ++cb) {
                    const float* sp = src + ((((size_t)i * cib + cb) * Hs + ys) * Ws + xs) * V;
                    const float* fp = filt + filter_index(Ci, sh.S, sh.R, V, co, cb * V, u, v);
                    for (int l = 0; l < V; ++l) {
                        const float d = sp[l];
                        if (Sparse && !(d != 0.0f)) continue;  // uniform across the warp
                        acc = fmaf(d, __ldg(fp + (size_t)l * V), acc);
                        ++cnt;
                    }
                }
            }
        }
        dst[act_index(Co, Ho, Wo, V, i, co, yo, xo)] = acc;
    }
    // one representative lane per V-vector of output channels counts vector FMAs
    warp_count_add(exec_ctr, (active && co % V == 0) ? cnt : 0u);
}

// BWW partial sums.  dG[k,c,v,u] = sum_{i,y',x'} D[i,c,y,x] * dY[i,k,y',x'].
// The checked tensor (ActCHWNn) supplies the uniform operand d; lanes own the
// other tensor's channels.  blockIdx.x = (checked channel m, v, u),
// blockIdx.y = lane-channel block, blockIdx.z = split of the (i, y') rows.
// Partial results go to partial[split][k][c][v][u] (plain order); bww_reduce
// sums the splits in fixed order, so results are deterministic.
template <bool CheckInput, bool Sparse>
__global__ void __launch_bounds__(128) bww_generic_partial(DevShape sh, int V, const float* __restrict__ chk,
                                                           const float* __restrict__ oth,
                                                           float* __restrict__ partial, int splits,
                                                           unsigned long long* __restrict__ exec_ctr,
                                                           const int* __restrict__ sel, int want) {
    if (sel != nullptr && __ldg(sel) != want) return;
    const int Lc = CheckInput ? sh.K : sh.C;  // lane channel count
    const int Mc = CheckInput ? sh.C : sh.K;  // checked channel count
    // grid-stride over the (m, v, u) x lane-block x split work units, so a
    // gated launch that is not selected costs a small grid, not one CTA per unit
    const int nlb = (Lc + blockDim.x - 1) / blockDim.x;
    const long units = (long)Mc * sh.S * sh.R * nlb * splits;
    for (long unit = blockIdx.x; unit < units; unit += gridDim.x) {
    long b = unit;
    const int zsplit = (int)(b % splits);
    b /= splits;
    const int lb = (int)(b % nlb);
    b /= nlb;
    const int u = (int)(b % sh.R);
    b /= sh.R;
    const int v = (int)(b % sh.S);
    const int m = (int)(b / sh.S);
    const int l = lb * blockDim.x + threadIdx.x;
    const bool active = l < Lc;
    const long rows = (long)sh.N * sh.Hp;
    const long r0 = rows * zsplit / splits, r1 = rows * (zsplit + 1) / splits;
    float acc = 0.0f;
    unsigned cnt = 0;
    if (active) {
        for (long r = r0; r < r1; ++r) {
            const int i = (int)(r / sh.Hp), yp = (int)(r % sh.Hp);
            const int y = yp * sh.P + v - sh.padH;
            if (y < 0 || y >= sh.H) continue;
            for (int xp = 0; xp < sh.Wp; ++xp) {
                const int x = xp * sh.O + u - sh.padW;
                if (x < 0 || x >= sh.W) continue;
                float d, o;
                if (CheckInput) {
                    d = chk[chwnn_index(sh.C, sh.H, sh.W, V, i, m, y, x)];
                    if (Sparse && !(d != 0.0f)) continue;
                    o = oth[act_index(sh.K, sh.Hp, sh.Wp, V, i, l, yp, xp)];
                } else {
                    d = chk[chwnn_index(sh.K, sh.Hp, sh.Wp, V, i, m, yp, xp)];
                    if (Sparse && !(d != 0.0f)) continue;
                    o = oth[act_index(sh.C, sh.H, sh.W, V, i, l, y, x)];
                }
                acc = fmaf(d, o, acc);
                ++cnt;
            }
        }
        const int k = CheckInput ? l : m, c = CheckInput ? m : l;
        const size_t E = (size_t)sh.K * sh.C * sh.S * sh.R;
        partial[(size_t)zsplit * E + (((size_t)k * sh.C + c) * sh.S + v) * sh.R + u] = acc;
    }
    warp_count_add(exec_ctr, (active && l % V == 0) ? cnt : 0u);
    }
}

// Fixed-order split reduction + scatter into FilterKCRSblk (K, C).  This also
// performs the reference's check=output_grad (c,k) fix-up
// (P/src/kernels.cpp:285-300) for free: partials are already in (k, c) order.
__global__ void bww_reduce_kernel(DevShape sh, int V, const float* __restrict__ partial, int splits,
                                  float* __restrict__ dst, const int* __restrict__ sel, int want) {
    if (sel != nullptr && __ldg(sel) != want) return;
    const size_t E = (size_t)sh.K * sh.C * sh.S * sh.R;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < E; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int z = 0; z < splits; ++z) s += partial[(size_t)z * E + e];
        size_t t = e;
        const int u = (int)(t % sh.R);
        t /= sh.R;
        const int v = (int)(t % sh.S);
        t /= sh.S;
        const int c = (int)(t % sh.C);
        const int k = (int)(t / sh.C);
        dst[filter_index(sh.C, sh.S, sh.R, V, k, c, u, v)] = s;
    }
}

// ---------------------------------------------------------------- launchers
cudaError_t launch_conv_generic(bool fwd, bool sparse, const DevShape& sh, int V, const float* src,
                                const float* filt, float* dst, unsigned long long* exec_ctr,
                                cudaStream_t st) {
    const int Co = fwd ? sh.K : sh.C;
    const int Ho = fwd ? sh.Hp : sh.H, Wo = fwd ? sh.Wp : sh.W;
    const int bs = Co >= 128 ? 128 : ((Co + 31) / 32) * 32;
    dim3 grid((unsigned)((long)sh.N * Ho * Wo), (unsigned)((Co + bs - 1) / bs));
    if (fwd) {
        if (sparse) conv_generic_kernel<true, true><<<grid, bs, 0, st>>>(sh, V, src, filt, dst, exec_ctr);
        else conv_generic_kernel<true, false><<<grid, bs, 0, st>>>(sh, V, src, filt, dst, exec_ctr);
    } else {
        if (sparse) conv_generic_kernel<false, true><<<grid, bs, 0, st>>>(sh, V, src, filt, dst, exec_ctr);
        else conv_generic_kernel<false, false><<<grid, bs, 0, st>>>(sh, V, src, filt, dst, exec_ctr);
    }
    note_launch();
    return cudaGetLastError();
}

int bww_generic_splits(const DevShape& sh) {
    const long rows = (long)sh.N * sh.Hp;
    long s = rows / 4;
    if (s < 1) s = 1;
    if (s > 64) s = 64;
    return (int)s;
}

cudaError_t launch_bww_generic(bool check_input, bool sparse, const DevShape& sh, int V, const float* chk,
                               const float* oth, float* partial, int splits, float* dst,
                               unsigned long long* exec_ctr, cudaStream_t st, const int* sel, int want) {
    const int Lc = check_input ? sh.K : sh.C;
    const int Mc = check_input ? sh.C : sh.K;
    const int bs = Lc >= 128 ? 128 : ((Lc + 31) / 32) * 32;
    const long units = (long)Mc * sh.S * sh.R * ((Lc + bs - 1) / bs) * splits;
    const unsigned grid = (unsigned)(units < 148L * 16 ? units : 148L * 16);
    if (check_input) {
        if (sparse) bww_generic_partial<true, true><<<grid, bs, 0, st>>>(sh, V, chk, oth, partial, splits, exec_ctr, sel, want);
        else bww_generic_partial<true, false><<<grid, bs, 0, st>>>(sh, V, chk, oth, partial, splits, exec_ctr, sel, want);
    } else {
        if (sparse) bww_generic_partial<false, true><<<grid, bs, 0, st>>>(sh, V, chk, oth, partial, splits, exec_ctr, sel, want);
        else bww_generic_partial<false, false><<<grid, bs, 0, st>>>(sh, V, chk, oth, partial, splits, exec_ctr, sel, want);
    }
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const size_t E = (size_t)sh.K * sh.C * sh.S * sh.R;
    const unsigned rb = (unsigned)((E + 255) / 256 < 148 * 4 ? (E + 255) / 256 : 148 * 4);
    bww_reduce_kernel<<<rb, 256, 0, st>>>(sh, V, partial, splits, dst, sel, want);
    note_launch();
    return cudaGetLastError();
}

}  // namespace spc
