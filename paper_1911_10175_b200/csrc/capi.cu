// capi.cu -- the extern "C" boundary: validation, planning, counters, dispatch.
//
// Validation restates the reference's contract checks so that the same bad
// calls fail the same way, before any device work:
//   conv_shape::validate      P/src/tensor.cpp:26-36
//   plan()                    P/src/planner.cpp:25-73
//   check_common              P/src/kernels.cpp:104-117
//   check_act / check_filter  P/src/kernels.cpp:119-142
//   per-entry C,K % V checks  P/src/kernels.cpp:172-173, 208-209, 244-245
#include <atomic>
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "dispatch.h"
#include "tile_bww.h"
#include "tile_conv.h"
#include "host_stage.h"
#include <nvtx3/nvToolsExt.h>
#include "../../include/spconv_b200_dev.h"

namespace spc {

static std::atomic<unsigned long long> g_launches{0};
void note_launch(unsigned n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static thread_local std::string g_err;

static spc_status fail(spc_status st, const std::string& msg) {
    g_err = msg;
    return st;
}
int* stream_flags(cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, int*> blocks;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> g(mu);
    int*& p = blocks[{dev, st}];
    if (!p && cudaMalloc((void**)&p, FLAG_COUNT * sizeof(int)) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
    }
    return p;
}

// For the other translation units (comm.cu): same thread-local message.
spc_status set_error(spc_status st, const std::string& msg) { return fail(st, msg); }

static bool valid_V(int v) { return v == 4 || v == 8 || v == 16; }
static int out_w(const spc_shape& s) { return (s.W + 2 * s.padW - s.R) / s.O + 1; }
static int out_h(const spc_shape& s) { return (s.H + 2 * s.padH - s.S) / s.P + 1; }

// conv_shape::validate (P/src/tensor.cpp:26-36)
static spc_status validate_shape(const spc_shape& s) {
    if (!(s.N > 0 && s.C > 0 && s.K > 0 && s.H > 0 && s.W > 0 && s.R > 0 && s.S > 0))
        return fail(SPC_ERR_SHAPE, "conv_shape: all dimensions must be positive");
    if (!(s.O >= 1 && s.P >= 1)) return fail(SPC_ERR_SHAPE, "conv_shape: strides must be >= 1");
    if (!(s.padW >= 0 && s.padH >= 0 && s.padW < s.R && s.padH < s.S))
        return fail(SPC_ERR_SHAPE, "conv_shape: padding must satisfy 0 <= pad < filter size");
    if (!(s.W + 2 * s.padW >= s.R && s.H + 2 * s.padH >= s.S))
        return fail(SPC_ERR_SHAPE, "conv_shape: filter does not fit the padded image");
    if (!(out_w(s) >= 1 && out_h(s) >= 1)) return fail(SPC_ERR_SHAPE, "conv_shape: output size must be positive");
    return SPC_OK;
}

// kernel_plan::tiled_channels (P/src/planner.cpp:18-23)
static int tiled_channels(const spc_shape& s, int comp, int check) {
    if (comp == SPC_BWI) return s.C;
    if (comp == SPC_BWW && check == SPC_CHECK_OUTPUT_GRAD) return s.C;
    return s.K;
}

// check_common (P/src/kernels.cpp:104-117); max_ring_vectors = 64 (kernel_impl.hpp:19)
static spc_status check_common(const spc_shape& sh, const spc_plan& pl, int comp) {
    spc_status st = validate_shape(sh);
    if (st) return st;
    if (pl.comp != comp) return fail(SPC_ERR_PLAN, "plan was built for another component");
    if (!valid_V(pl.V)) return fail(SPC_ERR_PLAN, "plan has an invalid V");
    if (comp == SPC_BWW && pl.check != SPC_CHECK_INPUT && pl.check != SPC_CHECK_OUTPUT_GRAD)
        return fail(SPC_ERR_PLAN, "plan has an invalid bww check side");
    const int tiled = tiled_channels(sh, comp, pl.check);
    if (!(pl.Q >= pl.V && pl.Q % pl.V == 0 && tiled % pl.Q == 0))
        return fail(SPC_ERR_PLAN, "plan tile Q does not divide the tiled channel dim");
    const int ring_need = (sh.R + (pl.pipelined ? 1 : 0)) * pl.Q / pl.V;
    if (ring_need > 64) return fail(SPC_ERR_PLAN, "plan ring size exceeds the kernel accumulator bound");
    return SPC_OK;
}

// check_act (P/src/kernels.cpp:119-132)
static spc_status check_act(const spc_tensor* t, int want, int V, int n, int ch, int rows, int cols,
                            const char* what) {
    if (!t) return fail(SPC_ERR_ARG, std::string(what) + ": null tensor");
    if (t->layout != want) return fail(SPC_ERR_LAYOUT, std::string(what) + ": wrong layout");
    if (t->V != V) return fail(SPC_ERR_LAYOUT, std::string(what) + ": wrong vector width");
    if (!(t->n == n && t->c == ch && t->h == rows && t->w == cols))
        return fail(SPC_ERR_LAYOUT, std::string(what) + ": dims do not match shape");
    const size_t expect = want == SPC_LAYOUT_ACT_CHWNN ? (size_t)((n + V - 1) / V) * ch * rows * cols * V
                                                       : (size_t)n * ch * rows * cols;
    if (t->numel != expect) return fail(SPC_ERR_LAYOUT, std::string(what) + ": data size mismatch");
    if (!t->data) return fail(SPC_ERR_ARG, std::string(what) + ": null data");
    return SPC_OK;
}

// check_filter (P/src/kernels.cpp:134-142)
static spc_status check_filter(const spc_tensor* t, int V, int k, int c, int s, int r, const char* what) {
    if (!t) return fail(SPC_ERR_ARG, std::string(what) + ": null tensor");
    if (t->layout != SPC_LAYOUT_FILTER_KCRS_BLK) return fail(SPC_ERR_LAYOUT, std::string(what) + ": wrong layout");
    if (t->V != V) return fail(SPC_ERR_LAYOUT, std::string(what) + ": wrong vector width");
    if (!(t->k == k && t->c == c && t->s == s && t->r == r))
        return fail(SPC_ERR_LAYOUT, std::string(what) + ": dims do not match shape");
    if (t->numel != (size_t)k * c * s * r) return fail(SPC_ERR_LAYOUT, std::string(what) + ": data size mismatch");
    if (!t->data) return fail(SPC_ERR_ARG, std::string(what) + ": null data");
    return SPC_OK;
}

static void set_act_desc(spc_tensor* t, int V, int n, int c, int h, int w) {
    t->layout = SPC_LAYOUT_ACT_NCHWC;
    t->V = V;
    t->n = n; t->c = c; t->h = h; t->w = w;
    t->k = t->r = t->s = 0;
}

static void set_filter_desc(spc_tensor* t, int V, int k, int c, int s, int r) {
    t->layout = SPC_LAYOUT_FILTER_KCRS_BLK;
    t->V = V;
    t->k = k; t->c = c; t->s = s; t->r = r;
    t->n = t->h = t->w = 0;
}

static spc_status output_desc(const spc_shape& sh, const spc_plan& pl, spc_tensor* out) {
    const size_t cap = out->numel;
    float* data = out->data;
    if (pl.comp == SPC_FWD) {
        set_act_desc(out, pl.V, sh.N, sh.K, out_h(sh), out_w(sh));
        out->numel = (size_t)sh.N * sh.K * out_h(sh) * out_w(sh);
    } else if (pl.comp == SPC_BWI) {
        set_act_desc(out, pl.V, sh.N, sh.C, sh.H, sh.W);
        out->numel = (size_t)sh.N * sh.C * sh.H * sh.W;
    } else {
        set_filter_desc(out, pl.V, sh.K, sh.C, sh.S, sh.R);
        out->numel = (size_t)sh.K * sh.C * sh.S * sh.R;
    }
    (void)cap;
    out->data = data;
    return SPC_OK;
}

// Output tensor: header is written by the call; the caller supplies data with
// capacity >= the required element count.
static spc_status prepare_dst(const spc_shape& sh, const spc_plan& pl, spc_tensor* dst) {
    if (!dst) return fail(SPC_ERR_ARG, "null output tensor");
    const size_t cap = dst->numel;
    float* data = dst->data;
    output_desc(sh, pl, dst);
    if (!data) return fail(SPC_ERR_ARG, "null output data");
    if (cap < dst->numel) return fail(SPC_ERR_ARG, "output buffer too small");
    return SPC_OK;
}

// ---------------------------------------------------------------- counters
// As-if counters of the reference kernels (P/src/kernel_impl.hpp:129-198,
// 229-325).  checked_vectors and the ring loads/stores depend only on shape
// and plan; dense-mode executed FMAs equal the dense total.
static void analytic_counters(const spc_shape& sh, const spc_plan& pl, int mode, spc_counters* c) {
    std::memset(c, 0, sizeof(*c));
    const int V = pl.V, hp = out_h(sh), wp = out_w(sh);
    const unsigned long long qv = (unsigned long long)(pl.Q / V);
    if (pl.comp == SPC_FWD || pl.comp == SPC_BWI) {
        const bool fwd = pl.comp == SPC_FWD;
        unsigned long long rows = 0;  // valid (output row, filter row) pairs
        const int orows = fwd ? hp : sh.H;
        for (int orow = 0; orow < orows; ++orow)
            for (int v = 0; v < sh.S; ++v) {
                if (fwd) {
                    const int y = orow * sh.P + v - sh.padH;
                    if (y < 0 || y >= sh.H) continue;
                } else {
                    const int num = orow + sh.padH - v;
                    if (num < 0 || num % sh.P != 0 || num / sh.P >= hp) continue;
                }
                ++rows;
            }
        const int scols = fwd ? sh.W : wp;  // swept columns
        const int ocols = fwd ? wp : sh.W;
        std::vector<char> touched(ocols, 0);
        unsigned long long tsum = 0;
        for (int x = 0; x < scols; ++x) {
            for (int u = 0; u < sh.R; ++u) {
                int oc;
                if (fwd) {
                    const int num = x + sh.padW - u;
                    if (num < 0 || num % sh.O != 0) continue;
                    oc = num / sh.O;
                    if (oc >= wp) continue;
                } else {
                    oc = x * sh.O + u - sh.padW;
                    if (oc < 0 || oc >= sh.W) continue;
                }
                touched[oc] = 1;
                ++tsum;
            }
        }
        unsigned long long ntouched = 0;
        for (char t : touched) ntouched += t;
        const int red_blocks = (fwd ? sh.C : sh.K) / V;
        const unsigned long long tiles = (unsigned long long)(fwd ? sh.K : sh.C) / pl.Q;
        const unsigned long long sweeps = rows * red_blocks * (unsigned long long)sh.N * tiles;
        c->output_vector_loads = c->output_vector_stores = sweeps * ntouched * qv;
        if (mode == SPC_SPARSE) {
            c->checked_vectors = tiles * rows * sh.N * (unsigned long long)red_blocks * scols;
        } else {
            c->executed_vector_fmas = rows * sh.N * (unsigned long long)red_blocks * V * tsum * qv * tiles;
        }
    } else {
        const bool on_input = pl.check == SPC_CHECK_INPUT;
        unsigned long long rows = 0;
        for (int v = 0; v < sh.S; ++v)
            for (int yp = 0; yp < hp; ++yp) {
                const int y = yp * sh.P + v - sh.padH;
                if (y >= 0 && y < sh.H) ++rows;
            }
        const int chans = on_input ? sh.C : sh.K;
        const int cols = on_input ? sh.W : wp;
        const unsigned long long tiles = (unsigned long long)(on_input ? sh.K : sh.C) / pl.Q;
        const unsigned long long nb = (unsigned long long)((sh.N + V - 1) / V);
        unsigned long long tsum = 0;
        for (int x = 0; x < cols; ++x)
            for (int u = 0; u < sh.R; ++u) {
                if (on_input) {
                    const int num = x + sh.padW - u;
                    if (num < 0 || num % sh.O != 0 || num / sh.O >= wp) continue;
                } else {
                    const int xx = x * sh.O + u - sh.padW;
                    if (xx < 0 || xx >= sh.W) continue;
                }
                ++tsum;
            }
        c->output_vector_loads = c->output_vector_stores = rows * nb * chans * tiles * sh.R * qv;
        if (mode == SPC_SPARSE) {
            c->checked_vectors = tiles * rows * chans * nb * cols;
        } else {
            c->executed_vector_fmas = rows * chans * (unsigned long long)sh.N * tsum * qv * tiles;
        }
    }
}

__global__ void counters_init_kernel(spc_counters* c, spc_counters v) { *c = v; }

// ---------------------------------------------------------------- device
// bytes of stream-ordered workspace kept cached between calls (SPC_POOL_KEEP_GB)
static unsigned long long pool_keep_bytes() {
    static const unsigned long long v =
        (unsigned long long)(std::getenv("SPC_POOL_KEEP_GB") ? std::atoi(std::getenv("SPC_POOL_KEEP_GB")) : 1) << 30;
    return v;
}

static spc_status check_device() {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(SPC_ERR_NO_DEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
    }
    static int cached_ok[64] = {0};
    if (dev >= 0 && dev < 64 && cached_ok[dev] == 1) return SPC_OK;
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    if (major != 10 || minor != 0)
        return fail(SPC_ERR_NO_DEVICE, "this library is built for sm_100a (B200); device is sm_" +
                                           std::to_string(major) + std::to_string(minor));
    // keep up to 1 GiB of stream-ordered workspace (BWW split partials,
    // tensor-core staging) cached between calls; memory above it returns to
    // the device at synchronisation points, so co-resident allocators
    // (e.g. PyTorch's) can use it
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long thr = pool_keep_bytes();
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    if (dev >= 0 && dev < 64) cached_ok[dev] = 1;
    return SPC_OK;
}

static spc_status cuda_fail(cudaError_t e, const char* where) {
    return fail(SPC_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

static spc_status start_counters(const spc_shape& sh, const spc_plan& pl, int mode, spc_counters* d_counters,
                                 cudaStream_t st) {
    if (!d_counters) return SPC_OK;
    spc_counters init;
    analytic_counters(sh, pl, mode, &init);
    counters_init_kernel<<<1, 1, 0, st>>>(d_counters, init);
    note_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "counters init");
}

static unsigned long long* exec_slot(spc_counters* d_counters, int mode) {
    // dense mode reports the analytic dense total; only sparse mode counts
    if (!d_counters || mode != SPC_SPARSE) return nullptr;
    return reinterpret_cast<unsigned long long*>(&d_counters->executed_vector_fmas);
}

// ---------------------------------------------------------------- passes
static spc_status validate_fwd(const spc_tensor* src, const spc_tensor* filt, const spc_shape& sh,
                               const spc_plan& pl) {
    spc_status st = check_common(sh, pl, SPC_FWD);
    if (st) return st;
    const int V = pl.V;
    if (sh.C % V || sh.K % V) return fail(SPC_ERR_SHAPE, "fwd: C and K must be multiples of V");
    if ((st = check_act(src, SPC_LAYOUT_ACT_NCHWC, V, sh.N, sh.C, sh.H, sh.W, "fwd input"))) return st;
    return check_filter(filt, V, sh.K, sh.C, sh.S, sh.R, "fwd filter");
}

static spc_status validate_bwi(const spc_tensor* dy, const spc_tensor* filt_t, const spc_shape& sh,
                               const spc_plan& pl) {
    spc_status st = check_common(sh, pl, SPC_BWI);
    if (st) return st;
    const int V = pl.V;
    if (sh.C % V || sh.K % V) return fail(SPC_ERR_SHAPE, "bwi: C and K must be multiples of V");
    if ((st = check_act(dy, SPC_LAYOUT_ACT_NCHWC, V, sh.N, sh.K, out_h(sh), out_w(sh), "bwi gradient")))
        return st;
    return check_filter(filt_t, V, sh.C, sh.K, sh.S, sh.R, "bwi transposed filter");
}

static spc_status validate_bww(const spc_tensor* in, const spc_tensor* dy, const spc_shape& sh,
                               const spc_plan& pl) {
    spc_status st = check_common(sh, pl, SPC_BWW);
    if (st) return st;
    const int V = pl.V;
    if (sh.C % V || sh.K % V) return fail(SPC_ERR_SHAPE, "bww: C and K must be multiples of V");
    if (pl.check == SPC_CHECK_INPUT) {
        if ((st = check_act(in, SPC_LAYOUT_ACT_CHWNN, V, sh.N, sh.C, sh.H, sh.W, "bww input"))) return st;
        return check_act(dy, SPC_LAYOUT_ACT_NCHWC, V, sh.N, sh.K, out_h(sh), out_w(sh), "bww gradient");
    }
    if ((st = check_act(dy, SPC_LAYOUT_ACT_CHWNN, V, sh.N, sh.K, out_h(sh), out_w(sh), "bww gradient")))
        return st;
    return check_act(in, SPC_LAYOUT_ACT_NCHWC, V, sh.N, sh.C, sh.H, sh.W, "bww input");
}

static Epi to_epi(const spc_epilogue* e) {
    Epi d;
    if (e) {
        d.alpha = e->alpha;
        d.add = e->add;
        d.mask = e->mask;
        d.relu = e->relu;
        d.beta = e->beta;
    }
    return d;
}

static spc_status run_fwd_bwi(bool fwd, const spc_tensor* src, const spc_tensor* filt, const spc_shape& sh,
                              const spc_plan& pl, int mode, spc_tensor* dst, spc_counters* d_counters,
                              cudaStream_t st, const spc_epilogue* epi = nullptr, const Gate& gate = Gate{}) {
    spc_status s = fwd ? validate_fwd(src, filt, sh, pl) : validate_bwi(src, filt, sh, pl);
    if (s) return s;
    if (mode != SPC_SPARSE && mode != SPC_DENSE) return fail(SPC_ERR_ARG, "bad run mode");
    if ((s = prepare_dst(sh, pl, dst))) return s;
    if ((s = check_device())) return s;
    if ((s = start_counters(sh, pl, mode, d_counters, st))) return s;
    const DevShape ds = make_dev_shape(sh);
    cudaError_t e = launch_conv(fwd, mode == SPC_SPARSE, ds, pl.V, src->data, filt->data, dst->data,
                                exec_slot(d_counters, mode), st, to_epi(epi), gate);
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, fwd ? "fwd launch" : "bwi launch");
}

static spc_status run_bww(const spc_tensor* in, const spc_tensor* dy, const spc_shape& sh, const spc_plan& pl,
                          int mode, spc_tensor* dst, spc_counters* d_counters, cudaStream_t st) {
    spc_status s = validate_bww(in, dy, sh, pl);
    if (s) return s;
    if (mode != SPC_SPARSE && mode != SPC_DENSE) return fail(SPC_ERR_ARG, "bad run mode");
    if ((s = prepare_dst(sh, pl, dst))) return s;
    if ((s = check_device())) return s;
    if ((s = start_counters(sh, pl, mode, d_counters, st))) return s;
    const DevShape ds = make_dev_shape(sh);
    const bool on_input = pl.check == SPC_CHECK_INPUT;
    cudaError_t e = launch_bww(on_input, mode == SPC_SPARSE, ds, pl.V, on_input ? in->data : dy->data,
                               on_input ? dy->data : in->data, dst->data, exec_slot(d_counters, mode), st);
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "bww launch");
}

// ---------------------------------------------------------------- aux kernels
__global__ void relu_kernel(const float* __restrict__ in, float* __restrict__ out, size_t n) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const float x = in[e];
        out[e] = x > 0.0f ? x : 0.0f;  // P/src/sparsity.cpp:13 (-0 and NaN -> +0)
    }
}

__global__ void relu_grad_mask_kernel(const float* __restrict__ pre, const float* __restrict__ up,
                                      float* __restrict__ out, size_t n) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
        out[e] = pre[e] > 0.0f ? up[e] : 0.0f;  // P/src/sparsity.cpp:26: zero where !(pre > 0)
}

// V = 16 fast path: a CTA transposes one (16-image block, 16-channel block,
// 16-pixel run) tile through shared memory: 16 images x 16 px x 16 ch read as
// contiguous 1 KB runs per image, written as contiguous 1 KB runs per channel.
__global__ void __launch_bounds__(256) nchwc_to_chwnn16_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                                               int n, int c, int hw) {
    __shared__ float t[16][16][17];  // [image][pixel][channel] (+1 pad)
    const int cb = blockIdx.y, nb = blockIdx.z, CB = c / 16;
    const int p0 = blockIdx.x * 16;
    // load: 16 images x 16 px x 4 float4
    for (int e = threadIdx.x; e < 16 * 16 * 4; e += 256) {
        const int q = e & 3, p = (e >> 2) & 15, i = e >> 6;
        const int img = nb * 16 + i, px = p0 + p;
        float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (img < n && px < hw) v = __ldg(reinterpret_cast<const float4*>(src + (((size_t)img * CB + cb) * hw + px) * 16) + q);
        t[i][p][q * 4 + 0] = v.x; t[i][p][q * 4 + 1] = v.y; t[i][p][q * 4 + 2] = v.z; t[i][p][q * 4 + 3] = v.w;
    }
    __syncthreads();
    // store: 16 channels x 16 px x 4 float4 (lanes = images)
    for (int e = threadIdx.x; e < 16 * 16 * 4; e += 256) {
        const int q = e & 3, p = (e >> 2) & 15, ch = e >> 6;
        const int px = p0 + p;
        if (px < hw) {
            const float4 v = make_float4(t[q * 4 + 0][p][ch], t[q * 4 + 1][p][ch], t[q * 4 + 2][p][ch], t[q * 4 + 3][p][ch]);
            *(reinterpret_cast<float4*>(dst + (((size_t)nb * c + cb * 16 + ch) * hw + px) * 16) + q) = v;
        }
    }
}

// ActNCHWc -> ActCHWNn with zero-filled ragged tail lanes (P/src/tensor.cpp:94-108).
__global__ void nchwc_to_chwnn_kernel(const float* __restrict__ src, float* __restrict__ dst, int n, int c,
                                      int h, int w, int V) {
    const size_t total = (size_t)((n + V - 1) / V) * c * h * w * V;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        size_t t = e;
        const int lane = (int)(t % V);
        t /= V;
        const int x = (int)(t % w);
        t /= w;
        const int y = (int)(t % h);
        t /= h;
        const int ch = (int)(t % c);
        const int ib = (int)(t / c);
        const int i = ib * V + lane;
        dst[e] = i < n ? src[act_index(c, h, w, V, i, ch, y, x)] : 0.0f;
    }
}

// FFMA peak probe: 16 independent accumulator chains per thread.
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) a[j] = threadIdx.x * 1e-7f + j;
    const float b = 0.999999f, c = 1e-7f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 16; ++j) a[j] = fmaf(a[j], b, c);
    }
    float s = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) s += a[j];
    if (s == 12345.678f) out[0] = s;  // keeps the chains live
}

__global__ void l2_flush_kernel(float* p, size_t n) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
        p[e] = (float)e;
}

static unsigned grid_for(size_t n) {
    size_t b = (n + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    if (b == 0) b = 1;
    return (unsigned)b;
}

}  // namespace spc

using namespace spc;

// ================================================================ C ABI
extern "C" {

int spc_abi_version(void) { return SPC_ABI_VERSION; }
const char* spc_last_error(void) { return g_err.c_str(); }
const char* spc_backend_name(void) { return "cuda-sm100a"; }
uint64_t spc_launch_count(void) { return g_launches.load(); }

int spc_native_backend_available(int V) {
    if (!valid_V(V)) return 0;
    return check_device() == SPC_OK ? 1 : 0;
}

spc_status spc_shape_make_padded(int N, int C, int K, int H, int W, int R, int S, int O, int P, int padW,
                                 int padH, spc_shape* out) {
    if (!out) return fail(SPC_ERR_ARG, "null shape");
    spc_shape s = {N, C, K, H, W, R, S, O, P, padW, padH};
    *out = s;
    return validate_shape(s);
}

spc_status spc_shape_make(int N, int C, int K, int H, int W, int R, int S, int O, int P, spc_shape* out) {
    return spc_shape_make_padded(N, C, K, H, W, R, S, O, P, (R - 1) / 2, (S - 1) / 2, out);
}

spc_status spc_shape_validate(const spc_shape* shape) {
    if (!shape) return fail(SPC_ERR_ARG, "null shape");
    return validate_shape(*shape);
}

// plan() (P/src/planner.cpp:25-73): largest ring under the register budget,
// larger Q on ties, then not pipelining; R=1 tiles capped at 128; bww never
// pipelines; M = 16 (1 for bww).
spc_status spc_plan_make(const spc_shape* shape, int comp, int V, int budget, int check, spc_plan* out) {
    if (!shape || !out) return fail(SPC_ERR_ARG, "null argument");
    spc_status st = validate_shape(*shape);
    if (st) return st;
    if (!valid_V(V)) return fail(SPC_ERR_PLAN, "plan: V must be 4, 8 or 16");
    if (budget < 1) return fail(SPC_ERR_PLAN, "plan: register budget must be >= 1");
    if (comp < SPC_FWD || comp > SPC_BWW) return fail(SPC_ERR_ARG, "plan: bad component");
    spc_plan p;
    std::memset(&p, 0, sizeof(p));
    p.comp = comp;
    p.check = check;
    p.V = V;
    p.register_budget = budget;
    const int ch = tiled_channels(*shape, comp, check);
    if (ch % V) return fail(SPC_ERR_PLAN, "plan: tiled channel dimension must be a multiple of V");
    const int R = shape->R;
    const bool allow_pipe = comp != SPC_BWW;
    int best_q = 0, best_ring = 0;
    bool best_pipe = false;
    for (int q = V; q <= ch; q += V) {
        if (ch % q) continue;
        if (R == 1 && q > 128) continue;
        for (int pipe = 0; pipe <= (allow_pipe ? 1 : 0); ++pipe) {
            const int ring = (R + pipe) * q / V;
            if (ring > budget) continue;
            const bool better =
                ring > best_ring || (ring == best_ring && (q > best_q || (q == best_q && pipe < (int)best_pipe)));
            if (better) {
                best_q = q;
                best_ring = ring;
                best_pipe = pipe != 0;
            }
        }
    }
    if (!best_q) return fail(SPC_ERR_PLAN, "plan: no feasible channel tile fits the register budget");
    p.Q = best_q;
    p.T = R * best_q / V;
    p.pipelined = best_pipe ? 1 : 0;
    p.ring_size = best_ring;
    p.M = comp == SPC_BWW ? 1 : 16;
    p.unroll_hint = best_pipe ? R + 1 : R;
    *out = p;
    return SPC_OK;
}

spc_status spc_output_desc(const spc_shape* shape, const spc_plan* plan, spc_tensor* out) {
    if (!shape || !plan || !out) return fail(SPC_ERR_ARG, "null argument");
    spc_status st = validate_shape(*shape);
    if (st) return st;
    out->data = nullptr;
    return output_desc(*shape, *plan, out);
}

spc_status spc_analytic_counters(const spc_shape* shape, const spc_plan* plan, int mode, spc_counters* out) {
    if (!shape || !plan || !out) return fail(SPC_ERR_ARG, "null argument");
    spc_status st = check_common(*shape, *plan, plan->comp);
    if (st) return st;
    analytic_counters(*shape, *plan, mode, out);
    return SPC_OK;
}

// NVTX ranges around the entry points (tracing): the names show up
// in Nsight Systems / ncu --nvtx timelines; without a tool attached the push
// and pop are a cheap no-op (nvtx3 is header-only, no link dependency).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

spc_status spc_sparse_fwd(const spc_tensor* src, const spc_tensor* filt, const spc_shape* shape,
                          const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters, void* stream) {
    NvtxRange r("spc_sparse_fwd");
    if (!shape || !plan) return fail(SPC_ERR_ARG, "null shape or plan");
    return run_fwd_bwi(true, src, filt, *shape, *plan, mode, dst, d_counters, (cudaStream_t)stream);
}

spc_status spc_sparse_bwi(const spc_tensor* grad_out, const spc_tensor* filt_t, const spc_shape* shape,
                          const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters, void* stream) {
    NvtxRange r("spc_sparse_bwi");
    if (!shape || !plan) return fail(SPC_ERR_ARG, "null shape or plan");
    return run_fwd_bwi(false, grad_out, filt_t, *shape, *plan, mode, dst, d_counters, (cudaStream_t)stream);
}

static spc_status check_epi(const spc_epilogue* epi) {
    if (!epi) return fail(SPC_ERR_ARG, "null epilogue");
    if (!(epi->alpha == epi->alpha)) return fail(SPC_ERR_ARG, "epilogue alpha is NaN");
    return SPC_OK;
}

spc_status spc_sparse_fwd_ex(const spc_tensor* src, const spc_tensor* filt, const spc_shape* shape,
                             const spc_plan* plan, int mode, const spc_epilogue* epi, spc_tensor* dst,
                             spc_counters* d_counters, void* stream) {
    NvtxRange r("spc_sparse_fwd_ex");
    if (!shape || !plan) return fail(SPC_ERR_ARG, "null shape or plan");
    spc_status s = check_epi(epi);
    if (s) return s;
    return run_fwd_bwi(true, src, filt, *shape, *plan, mode, dst, d_counters, (cudaStream_t)stream, epi);
}

spc_status spc_sparse_bwi_ex(const spc_tensor* grad_out, const spc_tensor* filt_t, const spc_shape* shape,
                             const spc_plan* plan, int mode, const spc_epilogue* epi, spc_tensor* dst,
                             spc_counters* d_counters, void* stream) {
    NvtxRange r("spc_sparse_bwi_ex");
    if (!shape || !plan) return fail(SPC_ERR_ARG, "null shape or plan");
    spc_status s = check_epi(epi);
    if (s) return s;
    return run_fwd_bwi(false, grad_out, filt_t, *shape, *plan, mode, dst, d_counters, (cudaStream_t)stream, epi);
}

int spc_set_math(int math) {
    if (math != SPC_MATH_FP32 && math != SPC_MATH_TF32X3) return -1;
    const int prev = math_mode();
    set_math_mode(math);
    return prev;
}
int spc_get_math(void) { return math_mode(); }

spc_status spc_epilogue_apply(const spc_epilogue* epi, float* data, size_t n, void* stream) {
    spc_status s = check_epi(epi);
    if (s) return s;
    if (!data && n) return fail(SPC_ERR_ARG, "null data");
    if ((s = check_device())) return s;
    cudaError_t e = launch_epilogue(to_epi(epi), data, n, (cudaStream_t)stream);
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "epilogue");
}

spc_status spc_sparse_bww(const spc_tensor* input, const spc_tensor* grad_out, const spc_shape* shape,
                          const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters, void* stream) {
    NvtxRange r("spc_sparse_bww");
    if (!shape || !plan) return fail(SPC_ERR_ARG, "null shape or plan");
    return run_bww(input, grad_out, *shape, *plan, mode, dst, d_counters, (cudaStream_t)stream);
}

spc_status spc_run_parallel(const spc_tensor* a, const spc_tensor* b, const spc_shape* shape, const spc_plan* plan,
                            int mode, spc_tensor* dst, spc_counters* d_counters, void* stream) {
    if (!plan) return fail(SPC_ERR_ARG, "null plan");
    switch (plan->comp) {
    case SPC_FWD: return spc_sparse_fwd(a, b, shape, plan, mode, dst, d_counters, stream);
    case SPC_BWI: return spc_sparse_bwi(a, b, shape, plan, mode, dst, d_counters, stream);
    case SPC_BWW: return spc_sparse_bww(a, b, shape, plan, mode, dst, d_counters, stream);
    }
    return fail(SPC_ERR_PLAN, "run_parallel: bad component");
}

// Host-buffer drop-in: validate, copy in, run, copy out, synchronize.
//
// Large calls are pipelined over batch chunks on three streams, so the copy
// of chunk c+1 in, the kernels of chunk c and the copy of chunk c-1 out run
// concurrently (two copy engines + SMs).  FWD/BWI chunks are image ranges
// (per-image independent: results are bitwise those of the device call).
// BWW chunks are whole 16-image blocks of the ActCHWNn tensor; each chunk's
// dG is summed in fixed chunk order by sum_partials_kernel (deterministic;
// the fp32 sum is regrouped relative to a single device call).
__global__ void sum_partials_kernel(const float* __restrict__ part, int nparts, size_t n, float* __restrict__ out) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int c = 0; c < nparts; ++c) s += part[(size_t)c * n + e];
        out[e] = s;
    }
}

namespace {
constexpr int kHostEvents = 64;  // = kMaxHostChunks
struct HostStreams {
    int dev = -1;
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};  // [0] compute, [1] copy-in, [2] copy-out
    cudaEvent_t ready = nullptr;
    cudaEvent_t in_done[kHostEvents] = {};  // chunk c's H2D complete (copy-in -> compute)
    cudaEvent_t k_done[kHostEvents] = {};   // chunk c's kernel complete (compute -> copy-out)
};
thread_local HostStreams g_hs;

spc_status host_streams(HostStreams*& hs) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (g_hs.dev != dev) {
        for (auto& st : g_hs.s) {
            cudaError_t e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "stream create");
        }
        cudaError_t e = cudaEventCreateWithFlags(&g_hs.ready, cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "event create");
        for (int c = 0; c < kHostEvents; ++c) {
            if ((e = cudaEventCreateWithFlags(&g_hs.in_done[c], cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&g_hs.k_done[c], cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "event create");
        }
        g_hs.dev = dev;
    }
    hs = &g_hs;
    return SPC_OK;
}
}  // namespace

static constexpr int kMaxHostChunks = 64;

// chunk count of the per-call host path: ~chunk_mb of traffic per chunk, at most max_chunks
static int host_chunk_count(size_t io_bytes, int units) {
    static const int chunk_mb = std::getenv("SPC_HOST_CHUNK_MB") ? std::atoi(std::getenv("SPC_HOST_CHUNK_MB")) : 48;
    static const int max_chunks =
        std::getenv("SPC_HOST_MAX_CHUNKS") ? std::atoi(std::getenv("SPC_HOST_MAX_CHUNKS")) : 16;
    int nc = (int)((io_bytes + ((size_t)chunk_mb << 20) - 1) / ((size_t)chunk_mb << 20));
    if (nc > max_chunks) nc = max_chunks;
    if (nc > kMaxHostChunks) nc = kMaxHostChunks;
    if (nc > units) nc = units;
    return nc < 1 ? 1 : nc;
}

// FWD / BWI host-buffer drop-in as ONE gated launch: copy-in stream
// (H2D chunk c, then a 4-byte copy raising in_ready[c]), compute stream (the
// kernel; CTAs of image i wait for in_ready[chunk(i)]), copy-out stream (D2H
// chunk c, issued by this host thread as soon as the kernel raises
// out_ready[c] in mapped pinned memory -- stream memory operations are not
// enabled on every driver, host polling is).  Copies overlap compute without
// splitting the kernel into small, inefficient per-chunk launches (Gate,
// common.cuh).
static spc_status run_fwd_bwi_gated(bool fwd, const spc_tensor* a, const spc_tensor* b, const spc_shape& sh,
                                    const spc_plan& pl, int mode, spc_tensor& out, spc_counters* counters,
                                    HostStreams* hs) {
    cudaStream_t s0 = hs->s[0], sin = hs->s[1], sout = hs->s[2];
    const int N = sh.N;
    static const int chunk_mb = std::getenv("SPC_HOST_CHUNK_MB") ? std::atoi(std::getenv("SPC_HOST_CHUNK_MB")) : 64;
    const size_t in_img = a->numel / N, out_img = out.numel / N;
    int ipc = (int)(((size_t)chunk_mb << 20) / ((in_img + out_img) * sizeof(float)));
    if (ipc < 1) ipc = 1;
    if (ipc > N) ipc = N;
    int nc = (N + ipc - 1) / ipc;
    if (nc > kMaxHostChunks) {
        ipc = (N + kMaxHostChunks - 1) / kMaxHostChunks;
        nc = (N + ipc - 1) / ipc;
    }
    // out_ready words live in mapped pinned memory the host polls
    static unsigned* h_out = nullptr;
    static unsigned* d_out = nullptr;
    cudaError_t e;
    if (!h_out) {
        if ((e = cudaHostAlloc((void**)&h_out, kMaxHostChunks * sizeof(unsigned), cudaHostAllocMapped)) != cudaSuccess)
            return cuda_fail(e, "mapped alloc");
        if ((e = cudaHostGetDevicePointer((void**)&d_out, h_out, 0)) != cudaSuccess) return cuda_fail(e, "mapped ptr");
    }
    std::memset(h_out, 0, kMaxHostChunks * sizeof(unsigned));
    float *da = nullptr, *db = nullptr, *dd = nullptr;
    spc_counters* dc = nullptr;
    unsigned* flags = nullptr;  // in_ready[nc], done[nc], (unused)[nc], err
    cudaError_t ce = cudaSuccess;  // first failure of any copy / event call
    auto ck = [&](cudaError_t x) {
        if (x != cudaSuccess && ce == cudaSuccess) ce = x;
    };
    auto release = [&]() {
        if (da) cudaFreeAsync(da, s0);
        if (db) cudaFreeAsync(db, s0);
        if (dd) cudaFreeAsync(dd, s0);
        if (dc) cudaFreeAsync(dc, s0);
        if (flags) cudaFreeAsync(flags, s0);
    };
    ck(cudaMallocAsync((void**)&da, a->numel * sizeof(float), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&db, b->numel * sizeof(float), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&dd, out.numel * sizeof(float), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&dc, sizeof(spc_counters), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&flags, (3 * (size_t)nc + 1) * sizeof(unsigned), s0));
    if (ce != cudaSuccess) {
        release();
        cudaStreamSynchronize(s0);
        return cuda_fail(ce, "alloc");
    }
    ck(cudaMemsetAsync(flags, 0, (3 * (size_t)nc + 1) * sizeof(unsigned), s0));
    ck(cudaMemcpyAsync(db, b->data, b->numel * sizeof(float), cudaMemcpyHostToDevice, s0));
    ck(cudaEventRecord(hs->ready, s0));  // buffers, zeroed flags and the filter visible to the copy streams
    Gate gate;
    gate.in_ready = flags;
    gate.done = flags + nc;
    gate.out_ready = d_out;
    gate.err = flags + 3 * nc;
    gate.ipc = ipc;
    gate.nimg = N;
    // copy-in: chunk c, then its ready word (a 4-byte copy from a pinned
    // constant on the same stream: ordered after the chunk, no SM involved)
    static unsigned* h_one = nullptr;
    if (!h_one) {
        if ((e = cudaMallocHost((void**)&h_one, sizeof(unsigned))) != cudaSuccess) return cuda_fail(e, "pinned alloc");
        *h_one = 1u;
    }
    ck(cudaStreamWaitEvent(sin, hs->ready, 0));
    for (int c = 0; c < nc; ++c) {
        const int i0 = c * ipc, i1 = i0 + ipc < N ? i0 + ipc : N;
        ck(cudaMemcpyAsync(da + (size_t)i0 * in_img, a->data + (size_t)i0 * in_img, (size_t)(i1 - i0) * in_img * sizeof(float),
                        cudaMemcpyHostToDevice, sin));
        ck(cudaMemcpyAsync(const_cast<unsigned*>(gate.in_ready) + c, h_one, sizeof(unsigned), cudaMemcpyHostToDevice, sin));
    }
    // compute: one launch, gated per chunk
    spc_tensor ta = *a, tb = *b, td = out;
    ta.data = da;
    tb.data = db;
    td.data = dd;
    spc_status st = run_fwd_bwi(fwd, &ta, &tb, sh, pl, mode, &td, counters ? dc : nullptr, s0, nullptr, gate);
    if (st == SPC_OK) {
        // copy-out: chunk c once its outputs are written
        // copy-out: poll the mapped words, issue chunk c's D2H as soon as it is written
        ck(cudaStreamWaitEvent(sout, hs->ready, 0));
        for (int c = 0; c < nc; ++c) {
            const int i0 = c * ipc, i1 = i0 + ipc < N ? i0 + ipc : N;
            for (long spin = 0; !*(volatile unsigned*)(h_out + c); ++spin) {
                if ((spin & 4095) == 0 && cudaStreamQuery(s0) != cudaErrorNotReady) {
                    // the kernel has finished (or failed): every word is final
                    if (!*(volatile unsigned*)(h_out + c)) break;
                }
            }
            ck(cudaMemcpyAsync(out.data + (size_t)i0 * out_img, dd + (size_t)i0 * out_img,
                            (size_t)(i1 - i0) * out_img * sizeof(float), cudaMemcpyDeviceToHost, sout));
        }
    }
    spc_counters hc{};
    unsigned herr = 0;
    if (st == SPC_OK) {
        if (counters) ck(cudaMemcpyAsync(&hc, dc, sizeof(hc), cudaMemcpyDeviceToHost, s0));
        ck(cudaMemcpyAsync(&herr, gate.err, sizeof(herr), cudaMemcpyDeviceToHost, s0));
    }
    cudaStreamSynchronize(sin);
    cudaStreamSynchronize(s0);
    cudaStreamSynchronize(sout);
    release();
    e = cudaStreamSynchronize(s0);
    if (st) return st;
    if (ce != cudaSuccess) return cuda_fail(ce, "host run (copy / event)");
    if (e != cudaSuccess) return cuda_fail(e, "host run");
    if (herr) return fail(SPC_ERR_CUDA, "host run: an input chunk never arrived (gated launch timed out)");
    if (counters) *counters = hc;
    return SPC_OK;
}

spc_status spc_run_parallel_host(const spc_tensor* a, const spc_tensor* b, const spc_shape* shape,
                                 const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* counters) {
    NvtxRange r("spc_run_parallel_host");
    if (!a || !b || !shape || !plan || !dst) return fail(SPC_ERR_ARG, "null argument");
    spc_status st;
    switch (plan->comp) {
    case SPC_FWD: st = validate_fwd(a, b, *shape, *plan); break;
    case SPC_BWI: st = validate_bwi(a, b, *shape, *plan); break;
    case SPC_BWW: st = validate_bww(a, b, *shape, *plan); break;
    default: return fail(SPC_ERR_PLAN, "run_parallel: bad component");
    }
    if (st) return st;
    if (mode != SPC_SPARSE && mode != SPC_DENSE) return fail(SPC_ERR_ARG, "bad run mode");
    spc_tensor out = *dst;
    if ((st = prepare_dst(*shape, *plan, &out))) return st;
    if ((st = check_device())) return st;
    HostStreams* hs = nullptr;
    if ((st = host_streams(hs))) return st;
    cudaStream_t s0 = hs->s[0];
    // SPC_HOST_GATE=1 selects the single gated launch for FWD/BWI.  Measured on
    // the VGG16 step it is not faster than the chunked path (0.577 vs 0.562 s:
    // PCIe-bound either way), so the chunked path is the default.  The gated
    // launch is an FFMA tile kernel: the tensor-core arithmetic keeps the
    // chunked path, so the host and device paths compute alike.
    static const bool gate_on = std::getenv("SPC_HOST_GATE") && std::atoi(std::getenv("SPC_HOST_GATE")) == 1;
    if (plan->comp != SPC_BWW && gate_on && math_mode() == SPC_MATH_FP32 && !is_pageable(a->data) &&
        !is_pageable(out.data) &&
        conv_supports_gate(plan->comp == SPC_FWD, make_dev_shape(*shape), plan->V)) {
        st = run_fwd_bwi_gated(plan->comp == SPC_FWD, a, b, *shape, *plan, mode, out, counters, hs);
        if (st == SPC_OK) *dst = out;
        return st;
    }

    const bool bww = plan->comp == SPC_BWW;
    const int V = plan->V;
    const bool on_input = plan->check == SPC_CHECK_INPUT;
    // the batch-sliced operands: FWD/BWI a; BWW both (checked in CHWNn blocks)
    const spc_tensor* chk = bww ? (on_input ? a : b) : a;
    const spc_tensor* oth = bww ? (on_input ? b : a) : nullptr;
    const size_t io_bytes = (a->numel + b->numel + out.numel) * sizeof(float);
    const int units = bww ? (shape->N + V - 1) / V : shape->N;  // chunk granularity
    // chunk count: ~chunk_mb of traffic per chunk, at most max_chunks (the
    // H2D / kernel / D2H of consecutive chunks overlap on 3 streams; the
    // call's exposed tail is one chunk's kernel + D2H)
    const int nc = host_chunk_count(io_bytes, units);

    float *da = nullptr, *db = nullptr, *dd = nullptr, *dpart = nullptr;
    spc_counters* dc = nullptr;
    cudaError_t e;
    // every CUDA call's status is kept (the first failure wins) and checked
    // before the chunk loop goes on; allocations are released on every path
    cudaError_t ce = cudaSuccess;
    auto ck = [&](cudaError_t x) {
        if (x != cudaSuccess && ce == cudaSuccess) ce = x;
    };
    auto release = [&]() {
        if (da) cudaFreeAsync(da, s0);
        if (db) cudaFreeAsync(db, s0);
        if (dd) cudaFreeAsync(dd, s0);
        if (dc) cudaFreeAsync(dc, s0);
        if (dpart) cudaFreeAsync(dpart, s0);
    };
    ck(cudaMallocAsync((void**)&da, a->numel * sizeof(float), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&db, b->numel * sizeof(float), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&dd, out.numel * sizeof(float), s0));
    if (ce == cudaSuccess) ck(cudaMallocAsync((void**)&dc, nc * sizeof(spc_counters), s0));
    if (ce == cudaSuccess && bww && nc > 1) ck(cudaMallocAsync((void**)&dpart, (size_t)nc * out.numel * sizeof(float), s0));
    if (ce != cudaSuccess) {
        release();
        cudaStreamSynchronize(s0);
        return cuda_fail(ce, "alloc");
    }
    // operands that are not batch-sliced go first, on s0
    if (!bww) ck(cudaMemcpyAsync(db, b->data, b->numel * sizeof(float), cudaMemcpyHostToDevice, s0));
    ck(cudaEventRecord(hs->ready, s0));  // allocations (+ filter) visible to the other streams

    const float* hchk = chk->data;
    float* dchk = chk == a ? da : db;
    const float* hoth = oth ? oth->data : nullptr;
    float* doth = oth ? (oth == a ? da : db) : nullptr;
    const size_t chk_unit = chk->numel / units;                // per image (NCHWc) or per block (CHWNn)
    const size_t oth_unit = oth ? oth->numel / shape->N : 0;   // per image (NCHWc)
    const size_t out_unit = bww ? 0 : out.numel / shape->N;    // per image

    // Pageable host buffers (a std::vector caller): the batch-sliced inputs are
    // copied by host threads into two pinned slots and DMA'd from there, the
    // outputs DMA'd into two pinned slots and copied out by the host, so the
    // host copy of chunk c+1 overlaps chunk c's DMA and kernel (host_stage.cu).
    const bool stage_in = is_pageable(hchk) || (oth && is_pageable(hoth));
    const bool stage_out = is_pageable(out.data);
    HostStaging& stg = host_staging();
    size_t in_max = 0, out_max = bww ? out.numel * sizeof(float) : 0;
    for (int c = 0; c < nc; ++c) {
        const int u0 = (int)((long)units * c / nc), u1 = (int)((long)units * (c + 1) / nc);
        const int i0 = bww ? u0 * V : u0;
        const int i1 = bww ? (u1 * V < shape->N ? u1 * V : shape->N) : u1;
        const size_t ib = ((size_t)(u1 - u0) * chk_unit + (size_t)(i1 - i0) * oth_unit) * sizeof(float);
        if (ib > in_max) in_max = ib;
        if (!bww && (size_t)(i1 - i0) * out_unit * sizeof(float) > out_max) out_max = (size_t)(i1 - i0) * out_unit * sizeof(float);
    }
    if (stage_in || stage_out) {
        ck(stg.reserve(stage_in ? in_max : 0, stage_out ? out_max : 0));
        if (ce != cudaSuccess) {
            release();
            cudaStreamSynchronize(s0);
            return cuda_fail(ce, "pinned staging");
        }
    }
    // a finished D2H chunk into a pinned slot -> the caller's pageable output
    auto drain_out = [&](int c) {
        const int u0 = (int)((long)units * c / nc), u1 = (int)((long)units * (c + 1) / nc);
        ck(cudaEventSynchronize(stg.out_ev[c & 1]));
        if (ce == cudaSuccess)
            host_copy(out.data + (size_t)u0 * out_unit, stg.out[c & 1], (size_t)(u1 - u0) * out_unit * sizeof(float));
    };

    // Three engines, three streams: every H2D on the copy-in stream back to
    // back, every kernel on the compute stream, every D2H on the copy-out
    // stream, joined per chunk by events -- so chunk c+1's H2D, chunk c's
    // kernel and chunk c-1's D2H run at once and PCIe carries both directions
    // together (measured duplex 82-91 GB/s vs 55-57 one way).
    cudaStream_t sin = hs->s[1], sout = hs->s[2];
    ck(cudaStreamWaitEvent(sin, hs->ready, 0));
    for (int c = 0; c < nc && st == SPC_OK && ce == cudaSuccess; ++c) {
        const int u0 = (int)((long)units * c / nc), u1 = (int)((long)units * (c + 1) / nc);
        const int i0 = bww ? u0 * V : u0;
        const int i1 = bww ? (u1 * V < shape->N ? u1 * V : shape->N) : u1;
        spc_shape shc = *shape;
        shc.N = i1 - i0;
        // H2D of this chunk's slices
        const size_t cb = (size_t)(u1 - u0) * chk_unit * sizeof(float), ob = (size_t)(i1 - i0) * oth_unit * sizeof(float);
        if (stage_in) {
            float* slot = stg.in[c & 1];
            if (c >= 2) ck(cudaEventSynchronize(stg.in_ev[c & 1]));  // chunk c-2's H2D has read the slot
            if (ce != cudaSuccess) break;
            host_copy(slot, hchk + (size_t)u0 * chk_unit, cb);
            if (oth) host_copy(reinterpret_cast<char*>(slot) + cb, hoth + (size_t)i0 * oth_unit, ob);
            ck(cudaMemcpyAsync(dchk + (size_t)u0 * chk_unit, slot, cb, cudaMemcpyHostToDevice, sin));
            if (oth)
                ck(cudaMemcpyAsync(doth + (size_t)i0 * oth_unit, reinterpret_cast<char*>(slot) + cb, ob,
                                   cudaMemcpyHostToDevice, sin));
            ck(cudaEventRecord(stg.in_ev[c & 1], sin));
        } else {
            ck(cudaMemcpyAsync(dchk + (size_t)u0 * chk_unit, hchk + (size_t)u0 * chk_unit, cb, cudaMemcpyHostToDevice,
                               sin));
            if (oth)
                ck(cudaMemcpyAsync(doth + (size_t)i0 * oth_unit, hoth + (size_t)i0 * oth_unit, ob,
                                   cudaMemcpyHostToDevice, sin));
        }
        ck(cudaEventRecord(hs->in_done[c], sin));
        ck(cudaStreamWaitEvent(s0, hs->in_done[c], 0));
        // chunk tensor descriptors
        spc_tensor tchk = *chk, toth, tb = *b, td = out;
        tchk.data = dchk + (size_t)u0 * chk_unit;
        tchk.n = shc.N;
        tchk.numel = (size_t)(u1 - u0) * chk_unit;
        if (oth) {
            toth = *oth;
            toth.data = doth + (size_t)i0 * oth_unit;
            toth.n = shc.N;
            toth.numel = (size_t)(i1 - i0) * oth_unit;
        }
        if (bww) {
            td.data = nc > 1 ? dpart + (size_t)c * out.numel : dd;
            const spc_tensor* in_t = on_input ? &tchk : &toth;
            const spc_tensor* dy_t = on_input ? &toth : &tchk;
            st = spc_sparse_bww(in_t, dy_t, &shc, plan, mode, &td, counters ? dc + c : nullptr, s0);
        } else {
            tb.data = db;
            td.data = dd + (size_t)i0 * out_unit;
            td.numel = (size_t)(i1 - i0) * out_unit;
            st = plan->comp == SPC_FWD ? spc_sparse_fwd(&tchk, &tb, &shc, plan, mode, &td, counters ? dc + c : nullptr, s0)
                                       : spc_sparse_bwi(&tchk, &tb, &shc, plan, mode, &td, counters ? dc + c : nullptr, s0);
            if (st == SPC_OK) {
                ck(cudaEventRecord(hs->k_done[c], s0));
                ck(cudaStreamWaitEvent(sout, hs->k_done[c], 0));
                if (stage_out) {
                    // the slot was emptied by drain_out(c - 2) in iteration c - 1
                    ck(cudaMemcpyAsync(stg.out[c & 1], td.data, td.numel * sizeof(float), cudaMemcpyDeviceToHost,
                                       sout));
                    ck(cudaEventRecord(stg.out_ev[c & 1], sout));
                    if (c >= 1) drain_out(c - 1);
                } else {
                    ck(cudaMemcpyAsync(out.data + (size_t)i0 * out_unit, td.data, td.numel * sizeof(float),
                                       cudaMemcpyDeviceToHost, sout));
                }
            }
        }
    }
    if (stage_out && !bww && st == SPC_OK && ce == cudaSuccess) drain_out(nc - 1);
    if (st == SPC_OK && ce == cudaSuccess && bww) {
        // reduce the chunks' partial dG in fixed order on the compute stream, copy dG out
        if (nc > 1) {
            sum_partials_kernel<<<grid_for(out.numel), 256, 0, s0>>>(dpart, nc, out.numel, dd);
            note_launch();
            ck(cudaGetLastError());
        }
        if (stage_out) {
            ck(cudaMemcpyAsync(stg.out[0], dd, out.numel * sizeof(float), cudaMemcpyDeviceToHost, s0));
            ck(cudaStreamSynchronize(s0));
            if (ce == cudaSuccess) host_copy(out.data, stg.out[0], out.numel * sizeof(float));
        } else {
            ck(cudaMemcpyAsync(out.data, dd, out.numel * sizeof(float), cudaMemcpyDeviceToHost, s0));
        }
    }
    spc_counters hc[kMaxHostChunks];
    if (st == SPC_OK && counters)
        ck(cudaMemcpyAsync(hc, dc, nc * sizeof(spc_counters), cudaMemcpyDeviceToHost, s0));
    for (int c = 0; c < 3; ++c) cudaStreamSynchronize(hs->s[c]);
    release();
    e = cudaStreamSynchronize(s0);
    if (st) return st;
    if (ce != cudaSuccess) return cuda_fail(ce, "host run (copy / event)");
    if (e != cudaSuccess) return cuda_fail(e, "host run");
    if (counters) {
        std::memset(counters, 0, sizeof(*counters));
        for (int c = 0; c < nc; ++c) {
            counters->checked_vectors += hc[c].checked_vectors;
            counters->executed_vector_fmas += hc[c].executed_vector_fmas;
            counters->output_vector_loads += hc[c].output_vector_loads;
            counters->output_vector_stores += hc[c].output_vector_stores;
        }
    }
    *dst = out;
    return SPC_OK;
}

// ---------------------------------------------------------------- host-buffer batch
// spc_run_parallel_host_batch: a list of host-buffer passes run as if
// spc_run_parallel_host were called on each in order, but pipelined ACROSS
// passes: pass i+1's H2D starts while pass i's kernels and D2H are still in
// flight, so the two copy engines and the SMs stay busy for the whole list
// instead of draining at every call (the per-call form exposes each call's
// first H2D chunk and last kernel + D2H chunk).  Up to batch_slots() (8) passes are
// in flight, each in its own slice of a per-thread device arena (no
// allocation inside the pipeline); every copy runs on the copy-in / copy-out
// streams of the per-call path, every kernel on its compute stream.
namespace {
constexpr int kBatchSlotsMax = 16;
static int batch_slots() {
    static const int v = std::getenv("SPC_BATCH_SLOTS") ? std::atoi(std::getenv("SPC_BATCH_SLOTS")) : 8;
    return v < 1 ? 1 : v > kBatchSlotsMax ? kBatchSlotsMax : v;
}
constexpr int kBatchChunks = 16;
struct BatchSlot {
    cudaEvent_t in_done[kBatchChunks] = {};
    cudaEvent_t k_done[kBatchChunks] = {};
    cudaEvent_t done = nullptr;
    spc_counters* hc = nullptr;  // pinned [kBatchChunks]
    char* mem = nullptr;         // this slot's slice of the arena
    // the pass in flight
    int pass = -1, nc = 0;
    spc_tensor out{};
    // host ranges of the pass (hazard checks) and its uploaded activation operands, which a later
    // pass naming the same host buffer reads in place instead of uploading again (a layer's BWI and
    // BWW both take dY in ActNCHWc); valid until the slot is enqueued again
    const char *h_lo[3] = {nullptr, nullptr, nullptr}, *h_hi[3] = {nullptr, nullptr, nullptr};  // a, b, out
    struct Upload {
        const float* host = nullptr;
        size_t numel = 0;
        float* dev = nullptr;
    } up[2];
    int up_last_chunk = 0;           // in_done[up_last_chunk]: both uploads complete
    cudaEvent_t lent_ev = nullptr;   // recorded after the last kernel of a pass that borrowed from this slot
    bool lent = false;
};
inline bool ranges_overlap(const char* a0, const char* a1, const char* b0, const char* b1) {
    return a0 && b0 && a0 < b1 && b0 < a1;
}
struct BatchState {
    int dev = -1;
    char* arena = nullptr;
    size_t slot_bytes = 0;
    BatchSlot slot[kBatchSlotsMax];
};
thread_local BatchState g_bs;

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// SPC_PASS_CHECKED_NCHWC: the BWW checked operand arrives in ActNCHWc and is packed on the device
bool checked_nchwc(const spc_host_pass& p) {
    return p.plan->comp == SPC_BWW && (p.flags & SPC_PASS_CHECKED_NCHWC) != 0;
}
const spc_tensor* checked_of(const spc_host_pass& p) { return p.plan->check == SPC_CHECK_INPUT ? p.a : p.b; }
// elements of the ActCHWNn form of an N x C x H x W activation
size_t chwnn_numel(const spc_tensor& t, int V) { return (size_t)((t.n + V - 1) / V) * V * t.c * t.h * t.w; }

// device bytes one pass needs in its slot
size_t batch_need(const spc_host_pass& p, const spc_tensor& out, int nc) {
    const bool bww = p.plan->comp == SPC_BWW;
    size_t n = align256(p.a->numel * sizeof(float)) + align256(p.b->numel * sizeof(float)) +
               align256(out.numel * sizeof(float)) + align256(kBatchChunks * sizeof(spc_counters));
    if (bww && nc > 1) n += align256((size_t)nc * out.numel * sizeof(float));
    if (checked_nchwc(p)) n += align256(chwnn_numel(*checked_of(p), p.plan->V) * sizeof(float));
    return n;
}

int batch_chunks(const spc_host_pass& p, const spc_tensor& out) {
    static const int chunk_mb = std::getenv("SPC_BATCH_CHUNK_MB") ? std::atoi(std::getenv("SPC_BATCH_CHUNK_MB")) : 128;
    const bool bww = p.plan->comp == SPC_BWW;
    const int units = bww ? (p.shape->N + p.plan->V - 1) / p.plan->V : p.shape->N;
    const size_t io = (p.a->numel + p.b->numel + out.numel) * sizeof(float);
    // BWW sums its chunks' partial dG, so its chunking is the per-call path's (the two forms then
    // agree bitwise); FWD / BWI chunks are independent image ranges and can be larger here, where
    // the next pass hides a chunk's head and tail
    if (bww) {
        const int n = host_chunk_count(io, units);
        return n > kBatchChunks ? kBatchChunks : n;
    }
    int nc = (int)((io + ((size_t)chunk_mb << 20) - 1) / ((size_t)chunk_mb << 20));
    if (nc > kBatchChunks) nc = kBatchChunks;
    if (nc > units) nc = units;
    return nc < 1 ? 1 : nc;
}

spc_status batch_state(BatchState*& bs, size_t slot_bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e;
    if (g_bs.dev != dev) {
        for (auto& sl : g_bs.slot) {
            for (int c = 0; c < kBatchChunks; ++c)
                if ((e = cudaEventCreateWithFlags(&sl.in_done[c], cudaEventDisableTiming)) != cudaSuccess ||
                    (e = cudaEventCreateWithFlags(&sl.k_done[c], cudaEventDisableTiming)) != cudaSuccess)
                    return cuda_fail(e, "event create");
            if ((e = cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming)) != cudaSuccess ||
                (e = cudaEventCreateWithFlags(&sl.lent_ev, cudaEventDisableTiming)) != cudaSuccess)
                return cuda_fail(e, "event create");
            if ((e = cudaMallocHost((void**)&sl.hc, kBatchChunks * sizeof(spc_counters))) != cudaSuccess)
                return cuda_fail(e, "pinned alloc");
        }
        g_bs.arena = nullptr;
        g_bs.slot_bytes = 0;
        g_bs.dev = dev;
    }
    if (g_bs.slot_bytes < slot_bytes) {  // grow (idle: no pass is in flight between batches)
        if (g_bs.arena) cudaFree(g_bs.arena);
        g_bs.arena = nullptr;
        g_bs.slot_bytes = 0;
        if ((e = cudaMalloc((void**)&g_bs.arena, slot_bytes * batch_slots())) != cudaSuccess)
            return cuda_fail(e, "batch arena");
        g_bs.slot_bytes = slot_bytes;
        for (int i = 0; i < batch_slots(); ++i) {
            g_bs.slot[i].mem = g_bs.arena + (size_t)i * slot_bytes;
            g_bs.slot[i].up[0] = g_bs.slot[i].up[1] = BatchSlot::Upload{};
            g_bs.slot[i].lent = false;
        }
    }
    bs = &g_bs;
    return SPC_OK;
}

// enqueue one pass (pinned host buffers) into `sl`; no host synchronisation
spc_status batch_enqueue(BatchState& bs, BatchSlot& sl, int idx, const spc_host_pass& p, const spc_tensor& out,
                         HostStreams* hs) {
    cudaStream_t s0 = hs->s[0], sin = hs->s[1], sout = hs->s[2];
    const spc_shape* shape = p.shape;
    const spc_plan* plan = p.plan;
    const bool bww = plan->comp == SPC_BWW;
    const int V = plan->V;
    const bool on_input = plan->check == SPC_CHECK_INPUT;
    const spc_tensor *a = p.a, *b = p.b;
    const spc_tensor* chk = bww ? (on_input ? a : b) : a;
    const spc_tensor* oth = bww ? (on_input ? b : a) : nullptr;
    const int units = bww ? (shape->N + V - 1) / V : shape->N;
    const int nc = batch_chunks(p, out);
    char* m = sl.mem;
    float* da = reinterpret_cast<float*>(m);
    m += align256(a->numel * sizeof(float));
    float* db = reinterpret_cast<float*>(m);
    m += align256(b->numel * sizeof(float));
    float* dd = reinterpret_cast<float*>(m);
    m += align256(out.numel * sizeof(float));
    spc_counters* dc = reinterpret_cast<spc_counters*>(m);
    m += align256(kBatchChunks * sizeof(spc_counters));
    float* dpart = reinterpret_cast<float*>(m);
    if (bww && nc > 1) m += align256((size_t)nc * out.numel * sizeof(float));
    float* dconv = reinterpret_cast<float*>(m);  // SPC_PASS_CHECKED_NCHWC: the device-packed ActCHWNn operand
    const bool conv = checked_nchwc(p);
    sl.pass = idx;
    sl.nc = nc;
    sl.out = out;
    sl.up[0] = sl.up[1] = BatchSlot::Upload{};
    sl.h_lo[0] = reinterpret_cast<const char*>(a->data);
    sl.h_hi[0] = sl.h_lo[0] + a->numel * sizeof(float);
    sl.h_lo[1] = reinterpret_cast<const char*>(b->data);
    sl.h_hi[1] = sl.h_lo[1] + b->numel * sizeof(float);
    sl.h_lo[2] = reinterpret_cast<const char*>(out.data);
    sl.h_hi[2] = sl.h_lo[2] + out.numel * sizeof(float);
    cudaError_t ce = cudaSuccess;
    auto ck = [&](cudaError_t x) {
        if (x != cudaSuccess && ce == cudaSuccess) ce = x;
    };
    spc_status st = SPC_OK;
    // a pass that borrowed an operand from this slot may still be reading it
    if (sl.lent) {
        ck(cudaStreamWaitEvent(sin, sl.lent_ev, 0));
        sl.lent = false;
    }
    // device copies of host ranges this pass overwrites are stale from here on
    for (int k = 0; k < batch_slots(); ++k)
        for (auto& u : bs.slot[k].up)
            if (u.host && ranges_overlap(reinterpret_cast<const char*>(u.host),
                                         reinterpret_cast<const char*>(u.host + u.numel), sl.h_lo[2], sl.h_hi[2]))
                u = BatchSlot::Upload{};
    // an activation operand another slot already holds: read it there
    BatchSlot* lender[2] = {nullptr, nullptr};
    auto borrow = [&](const spc_tensor* t, int which) -> float* {
        static const bool off = std::getenv("SPC_BATCH_SHARE") && std::atoi(std::getenv("SPC_BATCH_SHARE")) == 0;
        if (off || !t) return nullptr;
        for (int k = 0; k < batch_slots(); ++k) {
            BatchSlot& o = bs.slot[k];
            if (&o == &sl) continue;
            for (auto& u : o.up)
                if (u.host == t->data && u.numel == t->numel && u.dev) {
                    lender[which] = &o;
                    return u.dev;
                }
        }
        return nullptr;
    };
    if (!bww) ck(cudaMemcpyAsync(db, b->data, b->numel * sizeof(float), cudaMemcpyHostToDevice, sin));
    const float* hchk = chk->data;
    float* dchk = chk == a ? da : db;
    const float* hoth = oth ? oth->data : nullptr;
    float* doth = oth ? (oth == a ? da : db) : nullptr;
    float* bchk = borrow(chk, 0);
    float* both = borrow(oth, 1);
    if (bchk) dchk = bchk;
    if (both) doth = both;
    for (int w = 0; w < 2; ++w)
        if (lender[w]) ck(cudaStreamWaitEvent(s0, lender[w]->in_done[lender[w]->up_last_chunk], 0));
    if (!bchk) sl.up[0] = BatchSlot::Upload{hchk, chk->numel, dchk};
    if (oth && !both) sl.up[1] = BatchSlot::Upload{hoth, oth->numel, doth};
    sl.up_last_chunk = nc - 1;
    // conv: chk is ActNCHWc on the host and in `dchk`; the kernels read its ActCHWNn form in `dconv`
    const size_t img_unit = conv ? chk->numel / shape->N : 0;                 // ActNCHWc, per image
    const size_t chk_unit = conv ? (size_t)V * img_unit : chk->numel / units;  // ActCHWNn per block, or per image
    const size_t oth_unit = oth ? oth->numel / shape->N : 0;
    const size_t out_unit = bww ? 0 : out.numel / shape->N;
    for (int c = 0; c < nc && st == SPC_OK && ce == cudaSuccess; ++c) {
        const int u0 = (int)((long)units * c / nc), u1 = (int)((long)units * (c + 1) / nc);
        const int i0 = bww ? u0 * V : u0;
        const int i1 = bww ? (u1 * V < shape->N ? u1 * V : shape->N) : u1;
        spc_shape shc = *shape;
        shc.N = i1 - i0;
        if (!bchk) {
            if (conv)
                ck(cudaMemcpyAsync(dchk + (size_t)i0 * img_unit, hchk + (size_t)i0 * img_unit,
                                   (size_t)(i1 - i0) * img_unit * sizeof(float), cudaMemcpyHostToDevice, sin));
            else
                ck(cudaMemcpyAsync(dchk + (size_t)u0 * chk_unit, hchk + (size_t)u0 * chk_unit,
                                   (size_t)(u1 - u0) * chk_unit * sizeof(float), cudaMemcpyHostToDevice, sin));
        }
        if (oth && !both)
            ck(cudaMemcpyAsync(doth + (size_t)i0 * oth_unit, hoth + (size_t)i0 * oth_unit,
                               (size_t)(i1 - i0) * oth_unit * sizeof(float), cudaMemcpyHostToDevice, sin));
        ck(cudaEventRecord(sl.in_done[c], sin));
        ck(cudaStreamWaitEvent(s0, sl.in_done[c], 0));
        spc_tensor tchk = *chk, toth, tb = *b, td = out;
        tchk.data = (conv ? dconv : dchk) + (size_t)u0 * chk_unit;
        tchk.n = shc.N;
        tchk.numel = (size_t)(u1 - u0) * chk_unit;
        if (conv) {  // pack this chunk's images into ActCHWNn on the compute stream (pack_act_chwnn's lane rule)
            spc_tensor tsrc = *chk;
            tsrc.data = dchk + (size_t)i0 * img_unit;
            tsrc.n = shc.N;
            tsrc.numel = (size_t)(i1 - i0) * img_unit;
            st = spc_nchwc_to_chwnn(&tsrc, &tchk, s0);
            if (st) break;
        }
        if (oth) {
            toth = *oth;
            toth.data = doth + (size_t)i0 * oth_unit;
            toth.n = shc.N;
            toth.numel = (size_t)(i1 - i0) * oth_unit;
        }
        spc_counters* dcc = p.counters ? dc + c : nullptr;
        if (bww) {
            td.data = nc > 1 ? dpart + (size_t)c * out.numel : dd;
            const spc_tensor* in_t = on_input ? &tchk : &toth;
            const spc_tensor* dy_t = on_input ? &toth : &tchk;
            st = spc_sparse_bww(in_t, dy_t, &shc, plan, p.mode, &td, dcc, s0);
        } else {
            tb.data = db;
            td.data = dd + (size_t)i0 * out_unit;
            td.numel = (size_t)(i1 - i0) * out_unit;
            st = plan->comp == SPC_FWD ? spc_sparse_fwd(&tchk, &tb, &shc, plan, p.mode, &td, dcc, s0)
                                       : spc_sparse_bwi(&tchk, &tb, &shc, plan, p.mode, &td, dcc, s0);
            if (st == SPC_OK) {
                ck(cudaEventRecord(sl.k_done[c], s0));
                ck(cudaStreamWaitEvent(sout, sl.k_done[c], 0));
                ck(cudaMemcpyAsync(out.data + (size_t)i0 * out_unit, td.data, td.numel * sizeof(float),
                                   cudaMemcpyDeviceToHost, sout));
            }
        }
    }
    if (st == SPC_OK && ce == cudaSuccess && bww) {
        if (nc > 1) {
            sum_partials_kernel<<<grid_for(out.numel), 256, 0, s0>>>(dpart, nc, out.numel, dd);
            note_launch();
            ck(cudaGetLastError());
        }
        ck(cudaEventRecord(sl.k_done[nc - 1], s0));
        ck(cudaStreamWaitEvent(sout, sl.k_done[nc - 1], 0));
        ck(cudaMemcpyAsync(out.data, dd, out.numel * sizeof(float), cudaMemcpyDeviceToHost, sout));
    }
    for (int w = 0; w < 2; ++w)
        if (lender[w]) {  // every kernel of this pass is enqueued: the lender's slot may be refilled after them
            ck(cudaEventRecord(lender[w]->lent_ev, s0));
            lender[w]->lent = true;
        }
    if (st == SPC_OK && ce == cudaSuccess && p.counters)
        ck(cudaMemcpyAsync(sl.hc, dc, nc * sizeof(spc_counters), cudaMemcpyDeviceToHost, sout));
    ck(cudaEventRecord(sl.done, sout));
    if (st) return st;
    if (ce != cudaSuccess) return cuda_fail(ce, "host batch (copy / event)");
    return SPC_OK;
}

// wait for the pass in `sl`, deliver its counters and output header
spc_status batch_finish(BatchSlot& sl, spc_host_pass* passes) {
    if (sl.pass < 0) return SPC_OK;
    spc_host_pass& p = passes[sl.pass];
    sl.pass = -1;
    cudaError_t e = cudaEventSynchronize(sl.done);
    if (e != cudaSuccess) return p.status = cuda_fail(e, "host batch");
    if (p.counters) {
        std::memset(p.counters, 0, sizeof(*p.counters));
        for (int c = 0; c < sl.nc; ++c) {
            p.counters->checked_vectors += sl.hc[c].checked_vectors;
            p.counters->executed_vector_fmas += sl.hc[c].executed_vector_fmas;
            p.counters->output_vector_loads += sl.hc[c].output_vector_loads;
            p.counters->output_vector_stores += sl.hc[c].output_vector_stores;
        }
    }
    *p.dst = sl.out;
    return p.status = SPC_OK;
}
}  // namespace

// Frees the calling thread's batch arena (batch_slots() x the largest pass of the last batch; it is
// otherwise kept for the next call).
void spc_host_batch_release(void) {
    if (g_bs.arena) {
        cudaDeviceSynchronize();
        cudaFree(g_bs.arena);
    }
    g_bs.arena = nullptr;
    g_bs.slot_bytes = 0;
}

// SPC_PASS_CHECKED_NCHWC with pageable buffers: a plain synchronous path (upload, pack ActCHWNn on the
// device, one device BWW, download) -- same values as the pipelined form up to the chunking of the sum.
static spc_status run_bww_checked_nchwc_sync(spc_host_pass& p, const spc_tensor& out) {
    const int V = p.plan->V;
    const bool on_input = p.plan->check == SPC_CHECK_INPUT;
    const spc_tensor* chk = on_input ? p.a : p.b;
    const spc_tensor* oth = on_input ? p.b : p.a;
    const size_t cn = chwnn_numel(*chk, V);
    float *dn = nullptr, *dc = nullptr, *dq = nullptr, *dd = nullptr;
    spc_counters* dcnt = nullptr;
    cudaError_t e = cudaMalloc((void**)&dn, chk->numel * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc((void**)&dc, cn * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc((void**)&dq, oth->numel * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc((void**)&dd, out.numel * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc((void**)&dcnt, sizeof(spc_counters));
    spc_status st = SPC_OK;
    if (e == cudaSuccess) e = cudaMemcpy(dn, chk->data, chk->numel * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(dq, oth->data, oth->numel * sizeof(float), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) {
        spc_tensor tn = *chk, tc_ = *chk, tq = *oth, td = out;
        tn.data = dn;
        tc_.data = dc;
        tc_.numel = cn;
        tq.data = dq;
        td.data = dd;
        st = spc_nchwc_to_chwnn(&tn, &tc_, nullptr);
        if (st == SPC_OK)
            st = spc_sparse_bww(on_input ? &tc_ : &tq, on_input ? &tq : &tc_, p.shape, p.plan, p.mode, &td,
                                p.counters ? dcnt : nullptr, nullptr);
        if (st == SPC_OK) e = cudaMemcpy(out.data, dd, out.numel * sizeof(float), cudaMemcpyDeviceToHost);
        if (st == SPC_OK && e == cudaSuccess && p.counters)
            e = cudaMemcpy(p.counters, dcnt, sizeof(spc_counters), cudaMemcpyDeviceToHost);
    }
    cudaFree(dn);
    cudaFree(dc);
    cudaFree(dq);
    cudaFree(dd);
    cudaFree(dcnt);
    if (st) return st;
    if (e != cudaSuccess) return cuda_fail(e, "host batch (checked ActNCHWc, pageable)");
    *p.dst = out;
    return SPC_OK;
}

spc_status spc_run_parallel_host_batch(spc_host_pass* passes, int n) {
    NvtxRange r("spc_run_parallel_host_batch");
    if (n < 0 || (n > 0 && !passes)) return fail(SPC_ERR_ARG, "null pass list");
    if (n == 0) return SPC_OK;
    // validate everything before any device work (like the per-call form)
    std::vector<spc_tensor> outs(n);
    std::vector<char> direct(n);
    size_t slot_bytes = 0;
    for (int i = 0; i < n; ++i) {
        spc_host_pass& p = passes[i];
        p.status = SPC_OK;
        if (!p.a || !p.b || !p.shape || !p.plan || !p.dst) return p.status = fail(SPC_ERR_ARG, "null argument");
        spc_status st;
        switch (p.plan->comp) {
        case SPC_FWD: st = validate_fwd(p.a, p.b, *p.shape, *p.plan); break;
        case SPC_BWI: st = validate_bwi(p.a, p.b, *p.shape, *p.plan); break;
        case SPC_BWW:
            if (p.flags & SPC_PASS_CHECKED_NCHWC) {
                // the checked operand in ActNCHWc: validate the pass as if it were its ActCHWNn form
                const spc_tensor* chk = checked_of(p);
                if (chk->layout != SPC_LAYOUT_ACT_NCHWC || !valid_V(p.plan->V) ||
                    chk->numel != (size_t)chk->n * chk->c * chk->h * chk->w) {
                    st = fail(SPC_ERR_LAYOUT, "bww: SPC_PASS_CHECKED_NCHWC wants the checked tensor in ActNCHWc");
                    break;
                }
                spc_tensor as_chwnn = *chk;
                as_chwnn.layout = SPC_LAYOUT_ACT_CHWNN;
                as_chwnn.numel = chwnn_numel(*chk, p.plan->V);
                st = p.plan->check == SPC_CHECK_INPUT ? validate_bww(&as_chwnn, p.b, *p.shape, *p.plan)
                                                      : validate_bww(p.a, &as_chwnn, *p.shape, *p.plan);
            } else {
                st = validate_bww(p.a, p.b, *p.shape, *p.plan);
            }
            break;
        default: st = fail(SPC_ERR_PLAN, "run_parallel: bad component");
        }
        if (st) return p.status = st;
        if ((p.flags & ~SPC_PASS_CHECKED_NCHWC) || ((p.flags & SPC_PASS_CHECKED_NCHWC) && p.plan->comp != SPC_BWW))
            return p.status = fail(SPC_ERR_ARG, "bad pass flags");
        if (p.mode != SPC_SPARSE && p.mode != SPC_DENSE) return p.status = fail(SPC_ERR_ARG, "bad run mode");
        outs[i] = *p.dst;
        if ((st = prepare_dst(*p.shape, *p.plan, &outs[i]))) return p.status = st;
        // pageable buffers take the per-call path (its pinned staging ring) at their turn
        direct[i] = !(is_pageable(p.a->data) || is_pageable(p.b->data) || is_pageable(outs[i].data));
        if (direct[i]) {
            const size_t need = batch_need(p, outs[i], batch_chunks(p, outs[i]));
            if (need > slot_bytes) slot_bytes = need;
        }
    }
    spc_status st;
    if ((st = check_device())) return st;
    HostStreams* hs = nullptr;
    if ((st = host_streams(hs))) return st;
    BatchState* bs = nullptr;
    if (slot_bytes && (st = batch_state(bs, slot_bytes))) return st;
    // Keep the stream-ordered pool's memory across the call: batch_finish synchronises on events, and at
    // every synchronisation point the pool would otherwise return what exceeds its 1 GiB release threshold
    // (check_device) -- the BWW workspaces (planes, split partials: up to ~0.7 GB per pass) then come back
    // through fresh driver allocations that stall the enqueueing thread (measured: steps of 0.56-0.76 s among
    // 0.26 s ones).  The threshold is restored when the call returns.
    cudaMemPool_t pool = nullptr;
    {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            unsigned long long keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        } else {
            pool = nullptr;
        }
    }
    struct PoolRestore {
        cudaMemPool_t pool;
        ~PoolRestore() {
            if (pool) {
                unsigned long long thr = pool_keep_bytes();
                cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
            }
        }
    } pool_restore{pool};
    auto forget_uploads = [&]() {  // device copies of host buffers are trusted only inside one call
        for (int k = 0; k < kBatchSlotsMax && bs; ++k) bs->slot[k].up[0] = bs->slot[k].up[1] = BatchSlot::Upload{};
    };
    forget_uploads();
    spc_status first = SPC_OK;
    auto drain = [&]() {
        for (int k = 0; k < kBatchSlotsMax && bs; ++k) {
            const spc_status f = batch_finish(bs->slot[k], passes);
            if (f && !first) first = f;
        }
    };
    const int kBatchSlots = batch_slots();
    int next_slot = 0;
    for (int i = 0; i < n && !first; ++i) {
        spc_host_pass& p = passes[i];
        if (!direct[i]) {
            drain();
            if (first) break;
            p.status = checked_nchwc(p) ? run_bww_checked_nchwc_sync(p, outs[i])
                                        : spc_run_parallel_host(p.a, p.b, p.shape, p.plan, p.mode, p.dst, p.counters);
            if (p.status) first = p.status;
            forget_uploads();  // its output may overlap an uploaded range
            continue;
        }
        // host-buffer hazards against the passes in flight: an input an earlier pass writes, or an
        // output an earlier pass reads or writes -> let them finish first (order of a sequential loop)
        {
            const char* lo[3] = {reinterpret_cast<const char*>(p.a->data), reinterpret_cast<const char*>(p.b->data),
                                 reinterpret_cast<const char*>(outs[i].data)};
            const char* hi[3] = {lo[0] + p.a->numel * sizeof(float), lo[1] + p.b->numel * sizeof(float),
                                 lo[2] + outs[i].numel * sizeof(float)};
            bool hazard = false;
            for (int k = 0; k < kBatchSlots && !hazard; ++k) {
                const BatchSlot& o = bs->slot[k];
                if (o.pass < 0) continue;
                hazard = ranges_overlap(lo[0], hi[0], o.h_lo[2], o.h_hi[2]) ||
                         ranges_overlap(lo[1], hi[1], o.h_lo[2], o.h_hi[2]);
                for (int w = 0; w < 3 && !hazard; ++w) hazard = ranges_overlap(lo[2], hi[2], o.h_lo[w], o.h_hi[w]);
            }
            if (hazard) {
                drain();
                if (first) break;
            }
        }
        BatchSlot& sl = bs->slot[next_slot];
        next_slot = (next_slot + 1) % kBatchSlots;
        st = batch_finish(sl, passes);  // the pass that used this slot kBatchSlots passes ago
        if (st) {
            first = st;
            break;
        }
        st = batch_enqueue(*bs, sl, i, p, outs[i], hs);
        if (st) {
            p.status = st;
            first = st;
        }
    }
    // finish in submission order
    for (int k = 0; k < kBatchSlots && bs; ++k) {
        const spc_status f = batch_finish(bs->slot[(next_slot + k) % kBatchSlots], passes);
        if (f && !first) first = f;
    }
    if (first) {
        for (int c = 0; c < 3; ++c) cudaStreamSynchronize(hs->s[c]);
    }
    return first;
}

spc_status spc_relu(const float* in, float* out, size_t n, void* stream) {
    if ((!in || !out) && n) return fail(SPC_ERR_ARG, "null pointer");
    spc_status st = check_device();
    if (st) return st;
    if (!n) return SPC_OK;
    relu_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(in, out, n);
    note_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "relu");
}

spc_status spc_relu_grad_mask(const float* pre, const float* upstream, float* out, size_t n, void* stream) {
    if ((!pre || !upstream || !out) && n) return fail(SPC_ERR_ARG, "null pointer");
    spc_status st = check_device();
    if (st) return st;
    if (!n) return SPC_OK;
    relu_grad_mask_kernel<<<grid_for(n), 256, 0, (cudaStream_t)stream>>>(pre, upstream, out, n);
    note_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "relu_grad_mask");
}

spc_status spc_ffma_peak_kernel(float* out, int blocks, int iters, double* flops, void* stream) {
    if (!out || blocks < 1 || iters < 1) return fail(SPC_ERR_ARG, "bad argument");
    spc_status st = check_device();
    if (st) return st;
    ffma_peak_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(out, iters);
    note_launch();
    if (flops) *flops = 2.0 * 16.0 * (double)iters * 256.0 * (double)blocks;
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "ffma peak");
}

spc_status spc_debug_conv_variant(int variant, const spc_tensor* src, const spc_tensor* filt, const spc_shape* shape,
                                  const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters,
                                  void* stream) {
    if (!shape || !plan) return fail(SPC_ERR_ARG, "null shape or plan");
    if (plan->comp == SPC_BWW) {
        // src = input, filt = grad_out (spc_sparse_bww argument order)
        spc_status s = validate_bww(src, filt, *shape, *plan);
        if (s) return s;
        if ((s = prepare_dst(*shape, *plan, dst))) return s;
        if ((s = check_device())) return s;
        cudaStream_t st = (cudaStream_t)stream;
        if ((s = start_counters(*shape, *plan, mode, d_counters, st))) return s;
#ifdef SPC_DEV
        const bool ci = plan->check == SPC_CHECK_INPUT;
        cudaError_t e = launch_tile_bww_variant(variant, ci, mode == SPC_SPARSE, make_dev_shape(*shape),
                                                ci ? src->data : filt->data, ci ? filt->data : src->data, dst->data,
                                                exec_slot(d_counters, mode), st);
        return e == cudaSuccess ? SPC_OK : cuda_fail(e, "variant launch");
#else
        (void)variant;
        (void)st;
        return fail(SPC_ERR_ARG, "BWW tuning variants need the development build (make DEV=1)");
#endif
    }
    const bool fwd = plan->comp == SPC_FWD;
    spc_status s = fwd ? validate_fwd(src, filt, *shape, *plan) : validate_bwi(src, filt, *shape, *plan);
    if (s) return s;
    if ((s = prepare_dst(*shape, *plan, dst))) return s;
    if ((s = check_device())) return s;
    cudaStream_t st = (cudaStream_t)stream;
    if ((s = start_counters(*shape, *plan, mode, d_counters, st))) return s;
    cudaError_t e = launch_tile_conv_variant(variant, fwd, mode == SPC_SPARSE, make_dev_shape(*shape), src->data,
                                             filt->data, dst->data, exec_slot(d_counters, mode), st);
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "variant launch");
}

// vector_probes (P/include/spconv/kernels.hpp:90-98): the backend's contract
// operations exposed for equivalence tests -- here in the form the kernels
// use them, one warp, lane j = vector lane j: cmp_neq_zero as
// __ballot_sync(v != 0.0f), broadcast_fma as fmaf per lane, add per lane.
__global__ void vector_probe_kernel(int V, int op, const float* __restrict__ a, const float* __restrict__ b, float s,
                                    float* __restrict__ out, unsigned* __restrict__ mask) {
    const int l = threadIdx.x;
    const bool in = l < V;
    const float x = in ? a[l] : 0.0f;
    if (op == SPC_PROBE_CMP_NEQ_ZERO) {
        const unsigned m = __ballot_sync(0xffffffffu, in && x != 0.0f);
        if (l == 0) *mask = m;
    } else if (in) {
        out[l] = op == SPC_PROBE_BROADCAST_FMA ? fmaf(s, b[l], x) : x + b[l];
    }
}

spc_status spc_vector_probe(int V, int op, const float* a, const float* b, float s, float* out, uint32_t* mask) {
    if (!valid_V(V)) return fail(SPC_ERR_ARG, "vector_probe: V must be 4, 8 or 16");
    if (op < SPC_PROBE_CMP_NEQ_ZERO || op > SPC_PROBE_ADD) return fail(SPC_ERR_ARG, "vector_probe: bad op");
    if (!a || (op == SPC_PROBE_CMP_NEQ_ZERO ? !mask : (!b || !out))) return fail(SPC_ERR_ARG, "null argument");
    if (spc_status st = check_device()) return st;
    float* d = nullptr;
    cudaError_t e = cudaMalloc((void**)&d, 3 * 16 * sizeof(float) + sizeof(unsigned));
    if (e != cudaSuccess) return cuda_fail(e, "vector_probe alloc");
    unsigned* dm = reinterpret_cast<unsigned*>(d + 48);
    cudaMemcpy(d, a, V * sizeof(float), cudaMemcpyHostToDevice);
    if (b) cudaMemcpy(d + 16, b, V * sizeof(float), cudaMemcpyHostToDevice);
    vector_probe_kernel<<<1, 32>>>(V, op, d, d + 16, s, d + 32, dm);
    note_launch();
    e = cudaGetLastError();
    if (e == cudaSuccess && op == SPC_PROBE_CMP_NEQ_ZERO) e = cudaMemcpy(mask, dm, sizeof(unsigned), cudaMemcpyDeviceToHost);
    else if (e == cudaSuccess) e = cudaMemcpy(out, d + 32, V * sizeof(float), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "vector_probe");
}

spc_status spc_gen_sparse(float* out, size_t count, double sparsity, uint64_t seed) {
    if (!out && count) return fail(SPC_ERR_ARG, "null output");
    if (!(sparsity >= 0.0 && sparsity <= 1.0)) return fail(SPC_ERR_ARG, "gen_sparse: sparsity must be in [0, 1]");
    std::mt19937_64 rng(seed);
    auto unit = [&] { return double(rng() >> 11) * 0x1p-53; };
    for (size_t e = 0; e < count; ++e) {
        if (unit() < sparsity)
            out[e] = 0.0f;
        else
            out[e] = float(0.1 + 0.9 * unit());
    }
    return SPC_OK;
}

spc_status spc_l2_flush(float* scratch, size_t n, void* stream) {
    if (!scratch) return fail(SPC_ERR_ARG, "null scratch");
    spc_status st = check_device();
    if (st) return st;
    l2_flush_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(scratch, n);
    note_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "l2 flush");
}

spc_status spc_nchwc_to_chwnn(const spc_tensor* src, spc_tensor* dst, void* stream) {
    if (!src || !dst) return fail(SPC_ERR_ARG, "null tensor");
    if (src->layout != SPC_LAYOUT_ACT_NCHWC) return fail(SPC_ERR_LAYOUT, "nchwc_to_chwnn: source must be ActNCHWc");
    if (!valid_V(src->V) || src->c % src->V) return fail(SPC_ERR_LAYOUT, "nchwc_to_chwnn: bad V");
    if (src->numel != (size_t)src->n * src->c * src->h * src->w)
        return fail(SPC_ERR_LAYOUT, "nchwc_to_chwnn: data size mismatch");
    const int V = src->V;
    const size_t need = (size_t)((src->n + V - 1) / V) * src->c * src->h * src->w * V;
    if (!dst->data || dst->numel < need) return fail(SPC_ERR_ARG, "nchwc_to_chwnn: output buffer too small");
    spc_status st = check_device();
    if (st) return st;
    dst->layout = SPC_LAYOUT_ACT_CHWNN;
    dst->V = V;
    dst->n = src->n; dst->c = src->c; dst->h = src->h; dst->w = src->w;
    dst->k = dst->r = dst->s = 0;
    dst->numel = need;
    if (V == 16) {
        const int hw = src->h * src->w;
        dim3 grid((hw + 15) / 16, src->c / 16, (src->n + 15) / 16);
        nchwc_to_chwnn16_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(src->data, dst->data, src->n, src->c, hw);
    } else {
        nchwc_to_chwnn_kernel<<<grid_for(need), 256, 0, (cudaStream_t)stream>>>(src->data, dst->data, src->n,
                                                                               src->c, src->h, src->w, V);
    }
    note_launch();
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? SPC_OK : cuda_fail(e, "nchwc_to_chwnn");
}

}  // extern "C"
