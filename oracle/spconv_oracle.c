/*
 * spconv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's CPU algorithm for the sparse
 * direct-convolution hot path (SparseTrain, arXiv 1911.10175; reference
 * library `spconv` under /root/reference/proj).  It is the *checker* for the
 * CUDA product path: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it.  The product library never links or calls it.
 *
 * Parity of this restatement is pinned in tests/test_oracle.py against
 *   - the reference's own known answers (test_oracle.cpp, test_kernels.cpp,
 *     test_tensor.cpp, test_planner.cpp, test_vec.cpp), and
 *   - the reference library itself compiled from its sources into
 *     oracle/_ref/ (oracle/Makefile), bit-for-bit on dense_* outputs,
 *     generator streams, plans and FMA counts.
 *
 * Every function names the reference file:line it restates.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;

/* conv_shape: P/include/spconv/tensor.hpp:30-48 (field order kept). */
typedef struct {
    int N, C, K, H, W, R, S, O, P, padW, padH;
} orc_shape;

static int out_w(const orc_shape* s) { return (s->W + 2 * s->padW - s->R) / s->O + 1; }
static int out_h(const orc_shape* s) { return (s->H + 2 * s->padH - s->S) / s->P + 1; }

/* conv_shape::validate, P/src/tensor.cpp:26-36.  Returns 0 when valid. */
int orc_shape_validate(const orc_shape* s) {
    if (!(s->N > 0 && s->C > 0 && s->K > 0 && s->H > 0 && s->W > 0 && s->R > 0 && s->S > 0))
        return 1;
    if (!(s->O >= 1 && s->P >= 1)) return 2;
    if (!(s->padW >= 0 && s->padH >= 0 && s->padW < s->R && s->padH < s->S)) return 3;
    if (!(s->W + 2 * s->padW >= s->R && s->H + 2 * s->padH >= s->S)) return 4;
    if (!(out_w(s) >= 1 && out_h(s) >= 1)) return 5;
    return 0;
}

/* conv_shape::make default padding (R-1)/2, P/src/tensor.cpp:11-14. */
int orc_shape_make(int N, int C, int K, int H, int W, int R, int S, int O, int P, orc_shape* out) {
    orc_shape s = {N, C, K, H, W, R, S, O, P, (R - 1) / 2, (S - 1) / 2};
    *out = s;
    return orc_shape_validate(out);
}

/* ------------------------------------------------------------------ */
/* mt19937_64 + the hand-mapped uniform, P/src/sparsity.cpp:32-40.     */
/* (std::mt19937_64 is the published MT19937-64 generator, restated.)  */
typedef struct {
    u64 mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, u64 seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (u64)i;
    g->idx = 312;
}

static u64 mt64_next(mt64* g) {
    if (g->idx >= 312) {
        const u64 UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
        for (int i = 0; i < 312; ++i) {
            u64 x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            u64 xa = x >> 1;
            if (x & 1ULL) xa ^= A;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    u64 x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* value_gen::unit, P/src/sparsity.cpp:37: top 53 bits scaled by 2^-53. */
static double mt64_unit(mt64* g) { return (double)(mt64_next(g) >> 11) * 0x1p-53; }

/* Raw stream, for pinning the generator against std::mt19937_64. */
void orc_mt64_stream(u64 seed, u64* out, size_t n) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

/* gen_sparse, P/src/sparsity.cpp:42-55: zero w.p. s else U[0.1, 1]. */
void orc_gen_sparse(float* out, size_t count, double sparsity, u64 seed) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t e = 0; e < count; ++e) {
        if (mt64_unit(&g) < sparsity)
            out[e] = 0.0f;
        else
            out[e] = (float)(0.1 + 0.9 * mt64_unit(&g));
    }
}

/* gen_gaussian_relu, P/src/sparsity.cpp:57-69: Box-Muller, then ReLU. */
void orc_gen_gaussian_relu(float* out, size_t count, u64 seed) {
    mt64 g;
    mt64_seed(&g, seed);
    for (size_t e = 0; e < count; ++e) {
        double u1 = mt64_unit(&g);
        if (u1 < 1e-300) u1 = 1e-300;
        const double u2 = mt64_unit(&g);
        const double z = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        out[e] = z > 0.0 ? (float)z : 0.0f;
    }
}

/* relu: v > 0 ? v : 0 (P/src/sparsity.cpp:11-15); -0 and NaN map to +0. */
void orc_relu(const float* in, float* out, size_t n) {
    for (size_t e = 0; e < n; ++e) out[e] = in[e] > 0.0f ? in[e] : 0.0f;
}

/* relu_grad_mask: zero where !(pre > 0) (P/src/sparsity.cpp:17-28). */
void orc_relu_grad_mask(const float* pre, const float* up, float* out, size_t n) {
    for (size_t e = 0; e < n; ++e) out[e] = (pre[e] > 0.0f) ? up[e] : 0.0f;
}

/* cmp_neq_zero over V lanes, P/include/spconv/vec.hpp:120-128. */
uint32_t orc_cmp_neq_zero(const float* v, int V) {
    uint32_t m = 0;
    for (int i = 0; i < V; ++i)
        if (v[i] != 0.0f) m |= 1u << i;
    return m;
}

/* ------------------------------------------------------------------ */
/* affected_outputs / bwi_affected_outputs, P/src/tensor.cpp:43-66.    */
/* Writes (u, col) pairs; returns the pair count.                       */
int orc_affected_outputs(const orc_shape* s, int x, int* u_out, int* col_out) {
    int n = 0;
    const int wp = out_w(s);
    for (int u = s->R - 1; u >= 0; --u) {
        const int num = x + s->padW - u;
        if (num < 0 || num % s->O != 0) continue;
        const int xp = num / s->O;
        if (xp < wp) {
            u_out[n] = u;
            col_out[n] = xp;
            ++n;
        }
    }
    return n;
}

int orc_bwi_affected_outputs(const orc_shape* s, int xp, int* u_out, int* col_out) {
    int n = 0;
    for (int u = 0; u < s->R; ++u) {
        const int x = xp * s->O + u - s->padW;
        if (x >= 0 && x < s->W) {
            u_out[n] = u;
            col_out[n] = x;
            ++n;
        }
    }
    return n;
}

/* ------------------------------------------------------------------ */
/* Blocked layouts, P/include/spconv/tensor.hpp:89-119.                */
static size_t act_index(int C, int H, int W, int V, int i, int ch, int y, int x) {
    return ((((size_t)i * (C / V) + ch / V) * H + y) * W + x) * V + ch % V;
}
static size_t chwnn_index(int C, int H, int W, int V, int i, int ch, int y, int x) {
    return ((((size_t)(i / V) * C + ch) * H + y) * W + x) * V + i % V;
}
static size_t filter_index(int Cc, int S, int R, int V, int kk, int cc, int u, int v) {
    return (((((size_t)(kk / V) * (Cc / V) + cc / V) * S + v) * R + u) * V + cc % V) * V + kk % V;
}

/* pack_act_nchwc / pack_act_chwnn / pack_filter / unpack,
 * P/src/tensor.cpp:78-165.  layout: 1 = ActNCHWc, 2 = ActCHWNn,
 * 3 = FilterKCRSblk (swap_kc selects the BWI transpose). */
void orc_pack_act(const float* plain, float* out, int n, int c, int h, int w, int V, int chwnn) {
    if (chwnn) {
        const int nb = (n + V - 1) / V;
        memset(out, 0, sizeof(float) * (size_t)nb * c * h * w * V);
    }
    for (int i = 0; i < n; ++i)
        for (int ch = 0; ch < c; ++ch)
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    const float v = plain[(((size_t)i * c + ch) * h + y) * w + x];
                    const size_t di = chwnn ? chwnn_index(c, h, w, V, i, ch, y, x)
                                            : act_index(c, h, w, V, i, ch, y, x);
                    out[di] = v;
                }
}

void orc_unpack_act(const float* blk, float* plain, int n, int c, int h, int w, int V, int chwnn) {
    for (int i = 0; i < n; ++i)
        for (int ch = 0; ch < c; ++ch)
            for (int y = 0; y < h; ++y)
                for (int x = 0; x < w; ++x) {
                    const size_t si = chwnn ? chwnn_index(c, h, w, V, i, ch, y, x)
                                            : act_index(c, h, w, V, i, ch, y, x);
                    plain[(((size_t)i * c + ch) * h + y) * w + x] = blk[si];
                }
}

/* g is plain (K, C, S, R) indexed at(k, c, v, u). */
void orc_pack_filter(const float* g, float* out, int gn, int gc, int gs, int gr, int V, int swap_kc) {
    const int Cb = swap_kc ? gn : gc; /* blocked "c" dim */
    for (int kk = 0; kk < gn; ++kk)
        for (int cc = 0; cc < gc; ++cc)
            for (int v = 0; v < gs; ++v)
                for (int u = 0; u < gr; ++u) {
                    const int dk = swap_kc ? cc : kk;
                    const int dc = swap_kc ? kk : cc;
                    out[filter_index(Cb, gs, gr, V, dk, dc, u, v)] =
                        g[(((size_t)kk * gc + cc) * gs + v) * gr + u];
                }
}

/* blocked filter with dims (k, c, s, r) -> plain (k, c, s, r). */
void orc_unpack_filter(const float* blk, float* g, int k, int c, int s, int r, int V) {
    for (int kk = 0; kk < k; ++kk)
        for (int cc = 0; cc < c; ++cc)
            for (int v = 0; v < s; ++v)
                for (int u = 0; u < r; ++u)
                    g[(((size_t)kk * c + cc) * s + v) * r + u] = blk[filter_index(c, s, r, V, kk, cc, u, v)];
}

/* ------------------------------------------------------------------ */
/* Dense 64-bit oracles, P/src/oracle.cpp:39-148.  Per-output summation */
/* order is the reference's (FWD: c,v,u; BWI: k,v,u; BWW: i,y',x'), so   */
/* results are bitwise equal to the reference's dense_*.                */
typedef struct {
    int lo, hi;
} span;

static int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

/* valid_out_span, P/src/oracle.cpp:20-28 */
static span valid_out_span(int u, int pad, int stride, int in_limit, int out_limit) {
    int lo = -floor_div(u - pad, stride);
    if (lo < 0) lo = 0;
    int hi = floor_div(in_limit - 1 + pad - u, stride) + 1;
    if (hi > out_limit) hi = out_limit;
    span s = {lo, hi > lo ? hi : lo};
    return s;
}

typedef struct {
    int comp; /* 0 fwd, 1 bwi, 2 bww */
    const orc_shape* sh;
    const float* a;
    const float* b;
    float* out;
    int t, nt;
} dense_job;

static void dense_fwd_range(const dense_job* j) {
    const orc_shape* sh = j->sh;
    const int wp = out_w(sh), hp = out_h(sh);
    double* acc = (double*)malloc(sizeof(double) * (size_t)hp * wp);
    const float* D = j->a;
    const float* G = j->b;
    for (long ik = j->t; ik < (long)sh->N * sh->K; ik += j->nt) {
        const int i = (int)(ik / sh->K), k = (int)(ik % sh->K);
        for (size_t e = 0; e < (size_t)hp * wp; ++e) acc[e] = 0.0;
        for (int c = 0; c < sh->C; ++c)
            for (int v = 0; v < sh->S; ++v) {
                const span ys = valid_out_span(v, sh->padH, sh->P, sh->H, hp);
                for (int u = 0; u < sh->R; ++u) {
                    const double g = G[(((size_t)k * sh->C + c) * sh->S + v) * sh->R + u];
                    const span xs = valid_out_span(u, sh->padW, sh->O, sh->W, wp);
                    for (int yp = ys.lo; yp < ys.hi; ++yp) {
                        const int y = yp * sh->P + v - sh->padH;
                        const float* drow = D + (((size_t)i * sh->C + c) * sh->H + y) * sh->W;
                        double* arow = acc + (size_t)yp * wp;
                        for (int xp = xs.lo; xp < xs.hi; ++xp)
                            arow[xp] += g * drow[xp * sh->O + u - sh->padW];
                    }
                }
            }
        float* o = j->out + ((size_t)i * sh->K + k) * hp * wp;
        for (size_t e = 0; e < (size_t)hp * wp; ++e) o[e] = (float)acc[e];
    }
    free(acc);
}

static void dense_bwi_range(const dense_job* j) {
    const orc_shape* sh = j->sh;
    const int wp = out_w(sh), hp = out_h(sh);
    double* acc = (double*)malloc(sizeof(double) * (size_t)sh->H * sh->W);
    const float* dY = j->a;
    const float* G = j->b;
    for (long ic = j->t; ic < (long)sh->N * sh->C; ic += j->nt) {
        const int i = (int)(ic / sh->C), c = (int)(ic % sh->C);
        for (size_t e = 0; e < (size_t)sh->H * sh->W; ++e) acc[e] = 0.0;
        for (int k = 0; k < sh->K; ++k)
            for (int v = 0; v < sh->S; ++v) {
                const span ys = valid_out_span(v, sh->padH, sh->P, sh->H, hp);
                for (int u = 0; u < sh->R; ++u) {
                    const double g = G[(((size_t)k * sh->C + c) * sh->S + v) * sh->R + u];
                    const span xs = valid_out_span(u, sh->padW, sh->O, sh->W, wp);
                    for (int yp = ys.lo; yp < ys.hi; ++yp) {
                        const int y = yp * sh->P + v - sh->padH;
                        const float* grow = dY + (((size_t)i * sh->K + k) * hp + yp) * wp;
                        double* arow = acc + (size_t)y * sh->W;
                        for (int xp = xs.lo; xp < xs.hi; ++xp)
                            arow[xp * sh->O + u - sh->padW] += g * grow[xp];
                    }
                }
            }
        float* o = j->out + ((size_t)i * sh->C + c) * sh->H * sh->W;
        for (size_t e = 0; e < (size_t)sh->H * sh->W; ++e) o[e] = (float)acc[e];
    }
    free(acc);
}

static void dense_bww_range(const dense_job* j) {
    const orc_shape* sh = j->sh;
    const int wp = out_w(sh), hp = out_h(sh);
    const float* D = j->a;
    const float* dY = j->b;
    for (long kc = j->t; kc < (long)sh->K * sh->C; kc += j->nt) {
        const int k = (int)(kc / sh->C), c = (int)(kc % sh->C);
        for (int v = 0; v < sh->S; ++v) {
            const span ys = valid_out_span(v, sh->padH, sh->P, sh->H, hp);
            for (int u = 0; u < sh->R; ++u) {
                const span xs = valid_out_span(u, sh->padW, sh->O, sh->W, wp);
                double acc = 0.0;
                for (int i = 0; i < sh->N; ++i)
                    for (int yp = ys.lo; yp < ys.hi; ++yp) {
                        const int y = yp * sh->P + v - sh->padH;
                        const float* drow = D + (((size_t)i * sh->C + c) * sh->H + y) * sh->W;
                        const float* grow = dY + (((size_t)i * sh->K + k) * hp + yp) * wp;
                        for (int xp = xs.lo; xp < xs.hi; ++xp)
                            acc += (double)grow[xp] * drow[xp * sh->O + u - sh->padW];
                    }
                j->out[(((size_t)k * sh->C + c) * sh->S + v) * sh->R + u] = (float)acc;
            }
        }
    }
}

static void* dense_thread(void* p) {
    const dense_job* j = (const dense_job*)p;
    if (j->comp == 0) dense_fwd_range(j);
    else if (j->comp == 1) dense_bwi_range(j);
    else dense_bww_range(j);
    return NULL;
}

/* comp: 0 = dense_fwd(D, G) -> Y; 1 = dense_bwi(dY, G) -> dD;
 * 2 = dense_bww(D, dY) -> dG.  All tensors plain row-major.  Threads only
 * split independent outputs, so results do not depend on `threads`. */
int orc_dense(int comp, const orc_shape* sh, const float* a, const float* b, float* out, int threads) {
    if (orc_shape_validate(sh)) return 1;
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    dense_job jobs[256];
    for (int t = 0; t < threads; ++t) {
        dense_job j = {comp, sh, a, b, out, t, threads};
        jobs[t] = j;
    }
    if (threads == 1) {
        dense_thread(&jobs[0]);
        return 0;
    }
    for (int t = 0; t < threads; ++t) pthread_create(&tid[t], NULL, dense_thread, &jobs[t]);
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Planner, P/src/planner.cpp:18-111.                                   */
typedef struct {
    int comp, check, V, Q, T, pipelined, ring_size, M, register_budget, unroll_hint, prefetch_hints;
} orc_plan;

/* kernel_plan::tiled_channels, P/src/planner.cpp:18-23 */
int orc_tiled_channels(const orc_shape* s, int comp, int check) {
    if (comp == 1) return s->C;
    if (comp == 2 && check == 1) return s->C;
    return s->K;
}

/* plan(), P/src/planner.cpp:25-73.  Returns 0 on success. */
int orc_plan_make(const orc_shape* s, int comp, int V, int budget, int check, orc_plan* p) {
    if (orc_shape_validate(s)) return 1;
    if (!(V == 4 || V == 8 || V == 16)) return 2;
    if (budget < 1) return 3;
    memset(p, 0, sizeof(*p));
    p->comp = comp;
    p->check = check;
    p->V = V;
    p->register_budget = budget;
    const int ch = orc_tiled_channels(s, comp, check);
    if (ch % V != 0) return 4;
    const int allow_pipe = comp != 2;
    int best_q = 0, best_ring = 0, best_pipe = 0;
    for (int q = V; q <= ch; q += V) {
        if (ch % q) continue;
        if (s->R == 1 && q > 128) continue;
        for (int pipe = 0; pipe <= allow_pipe; ++pipe) {
            const int ring = (s->R + pipe) * q / V;
            if (ring > budget) continue;
            const int better = ring > best_ring ||
                               (ring == best_ring && (q > best_q || (q == best_q && pipe < best_pipe)));
            if (better) {
                best_q = q;
                best_ring = ring;
                best_pipe = pipe;
            }
        }
    }
    if (!best_q) return 5;
    p->Q = best_q;
    p->T = s->R * best_q / V;
    p->pipelined = best_pipe;
    p->ring_size = best_ring;
    p->M = comp == 2 ? 1 : 16;
    p->unroll_hint = best_pipe ? s->R + 1 : s->R;
    return 0;
}

/* decompose(), P/src/planner.cpp:81-111: task axis counts. */
void orc_decompose(const orc_shape* s, const orc_plan* p, int counts[3]) {
    const int m = p->M < s->N ? p->M : s->N;
    const int tiles = (s->N + m - 1) / m;
    if (p->comp == 0) {
        counts[0] = tiles; counts[1] = out_h(s); counts[2] = s->K / p->Q;
    } else if (p->comp == 1) {
        counts[0] = tiles; counts[1] = s->H; counts[2] = s->C / p->Q;
    } else if (p->check == 0) {
        counts[0] = s->S; counts[1] = s->C; counts[2] = s->K / p->Q;
    } else {
        counts[0] = s->S; counts[1] = s->K; counts[2] = s->C / p->Q;
    }
}

/* ------------------------------------------------------------------ */
/* expected_fma_counts, P/src/oracle.cpp:150-284: walks the kernel's    */
/* loop structure over the zeros of the plain mask source.              */
/* rep = {checked_vectors, nonzero_elements, executed, skipped}.        */
int orc_expected_counts(const orc_shape* sh, const orc_plan* pl, const float* mask, u64 rep[4]) {
    if (orc_shape_validate(sh)) return 1;
    const int V = pl->V;
    const int wp = out_w(sh), hp = out_h(sh);
    const u64 qv = (u64)pl->Q / V;
    u64 checked = 0, nnz_total = 0, exec = 0, dense_exec = 0;
    int ubuf[64], cbuf[64];
    if (pl->comp == 0) {
        const u64 tiles = (u64)sh->K / pl->Q;
        int* tsize = (int*)malloc(sizeof(int) * sh->W);
        for (int x = 0; x < sh->W; ++x) tsize[x] = orc_affected_outputs(sh, x, ubuf, cbuf);
        for (int yp = 0; yp < hp; ++yp)
            for (int v = 0; v < sh->S; ++v) {
                const int yin = yp * sh->P + v - sh->padH;
                if (yin < 0 || yin >= sh->H) continue;
                for (int i = 0; i < sh->N; ++i)
                    for (int cb = 0; cb < sh->C / V; ++cb)
                        for (int x = 0; x < sh->W; ++x) {
                            int nnz = 0;
                            for (int l = 0; l < V; ++l)
                                if (mask[(((size_t)i * sh->C + cb * V + l) * sh->H + yin) * sh->W + x] != 0.0f) ++nnz;
                            checked += tiles;
                            nnz_total += tiles * nnz;
                            exec += tiles * (u64)nnz * tsize[x] * qv;
                            dense_exec += tiles * (u64)V * tsize[x] * qv;
                        }
            }
        free(tsize);
    } else if (pl->comp == 1) {
        const u64 tiles = (u64)sh->C / pl->Q;
        int* tsize = (int*)malloc(sizeof(int) * wp);
        for (int xp = 0; xp < wp; ++xp) tsize[xp] = orc_bwi_affected_outputs(sh, xp, ubuf, cbuf);
        for (int y = 0; y < sh->H; ++y)
            for (int v = 0; v < sh->S; ++v) {
                const int num = y + sh->padH - v;
                if (num < 0 || num % sh->P != 0) continue;
                const int yp = num / sh->P;
                if (yp >= hp) continue;
                for (int i = 0; i < sh->N; ++i)
                    for (int kb = 0; kb < sh->K / V; ++kb)
                        for (int xp = 0; xp < wp; ++xp) {
                            int nnz = 0;
                            for (int l = 0; l < V; ++l)
                                if (mask[(((size_t)i * sh->K + kb * V + l) * hp + yp) * wp + xp] != 0.0f) ++nnz;
                            checked += tiles;
                            nnz_total += tiles * nnz;
                            exec += tiles * (u64)nnz * tsize[xp] * qv;
                            dense_exec += tiles * (u64)V * tsize[xp] * qv;
                        }
            }
        free(tsize);
    } else {
        const int on_input = pl->check == 0;
        const u64 tiles = (u64)(on_input ? sh->K : sh->C) / pl->Q;
        const int chans = on_input ? sh->C : sh->K;
        const int cols = on_input ? sh->W : wp;
        const int mh = on_input ? sh->H : hp;
        const int mw = cols;
        int* tsize = (int*)malloc(sizeof(int) * cols);
        for (int x = 0; x < cols; ++x)
            tsize[x] = on_input ? orc_affected_outputs(sh, x, ubuf, cbuf) : orc_bwi_affected_outputs(sh, x, ubuf, cbuf);
        const int nb = (sh->N + V - 1) / V;
        for (int v = 0; v < sh->S; ++v)
            for (int ch = 0; ch < chans; ++ch)
                for (int ib = 0; ib < nb; ++ib) {
                    const int lanes = V < sh->N - ib * V ? V : sh->N - ib * V;
                    for (int yp = 0; yp < hp; ++yp) {
                        const int yin = yp * sh->P + v - sh->padH;
                        if (yin < 0 || yin >= sh->H) continue;
                        const int row = on_input ? yin : yp;
                        for (int x = 0; x < cols; ++x) {
                            int nnz = 0;
                            for (int l = 0; l < lanes; ++l)
                                if (mask[(((size_t)(ib * V + l) * chans + ch) * mh + row) * mw + x] != 0.0f) ++nnz;
                            checked += tiles;
                            nnz_total += tiles * nnz;
                            exec += tiles * (u64)nnz * tsize[x] * qv;
                            dense_exec += tiles * (u64)lanes * tsize[x] * qv;
                        }
                    }
                }
        free(tsize);
    }
    rep[0] = checked;
    rep[1] = nnz_total;
    rep[2] = exec;
    rep[3] = dense_exec - exec;
    return 0;
}

/* ------------------------------------------------------------------ */
/* 64-bit inner product and the reference's elementwise error metric,  */
/* P/src/oracle.cpp:409-425; plus the north-star max-abs metric.        */
double orc_dot(const float* a, const float* b, size_t n) {
    double acc = 0.0;
    for (size_t e = 0; e < n; ++e) acc += (double)a[e] * b[e];
    return acc;
}

double orc_max_rel_error(const float* a, const float* ref, size_t n) {
    double worst = 0.0;
    for (size_t e = 0; e < n; ++e) {
        const double d = fabs((double)a[e] - ref[e]);
        const double r = d / (fabs((double)ref[e]) + 1e-6);
        if (r > worst) worst = r;
    }
    return worst;
}

/* max|a - ref| / max|ref| (north-star parity metric; not in the reference). */
double orc_max_abs_rel(const float* a, const float* ref, size_t n) {
    double md = 0.0, mr = 0.0;
    for (size_t e = 0; e < n; ++e) {
        const double d = fabs((double)a[e] - ref[e]);
        if (d > md || d != d) md = d != d ? INFINITY : d;
        const double r = fabs((double)ref[e]);
        if (r > mr) mr = r;
    }
    if (mr == 0.0) return md;
    return md / mr;
}
