// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C ABI over the *unmodified* reference library (`spconv`, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests and bench.py's cpu_baseline / --impl reference arms call the
// reference's own public API: plan() (P/src/planner.cpp:25), pack_*
// (P/src/tensor.cpp:78-130), run_parallel (P/src/kernels.cpp:304),
// dense_* and expected_fma_counts (P/src/oracle.cpp:39-284), gen_sparse
// (P/src/sparsity.cpp:42).  Nothing here re-implements reference arithmetic.
#include <cstdint>
#include <cstring>
#include <sstream>
#include <vector>
#include <exception>
#include <memory>
#include <random>
#include <string>
#include <thread>

#include "spconv/bench.hpp"
#include "spconv/kernels.hpp"
#include "spconv/projector.hpp"
#include "spconv/oracle.hpp"
#include "spconv/planner.hpp"
#include "spconv/sparsity.hpp"
#include "spconv/tensor.hpp"

using namespace spconv;

namespace {

thread_local std::string g_err;

conv_shape to_shape(const int* s) {
    conv_shape sh;
    sh.N = s[0]; sh.C = s[1]; sh.K = s[2]; sh.H = s[3]; sh.W = s[4];
    sh.R = s[5]; sh.S = s[6]; sh.O = s[7]; sh.P = s[8];
    sh.padW = s[9]; sh.padH = s[10];
    return sh;
}

plain_tensor plain_from(const float* p, int n, int c, int h, int w) {
    plain_tensor t(n, c, h, w);
    std::memcpy(t.data.data(), p, t.size() * sizeof(float));
    return t;
}

// A prepared reference run: packed operands + plan, ready for timed calls.
struct prepared {
    conv_shape sh;
    kernel_plan pl;
    blocked_tensor a, b;
    conv_result res;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

// plan(): fields out = {Q, T, pipelined, ring_size, M, unroll_hint}
int ref_plan(const int* shape, int comp, int V, int budget, int check, int* out) {
    try {
        const kernel_plan p = plan(to_shape(shape), component(comp), V, budget, bww_check(check));
        out[0] = p.Q; out[1] = p.T; out[2] = p.pipelined; out[3] = p.ring_size;
        out[4] = p.M; out[5] = p.unroll_hint;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// conv_shape::make -> 11 ints; returns nonzero on spconv::error.
int ref_shape_make(int N, int C, int K, int H, int W, int R, int S, int O, int P, int* out) {
    try {
        const conv_shape sh = conv_shape::make(N, C, K, H, W, R, S, O, P);
        const int v[11] = {sh.N, sh.C, sh.K, sh.H, sh.W, sh.R, sh.S, sh.O, sh.P, sh.padW, sh.padH};
        std::memcpy(out, v, sizeof(v));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

void ref_gen_sparse(int n, int c, int h, int w, double s, uint64_t seed, float* out) {
    const plain_tensor t = gen_sparse(n, c, h, w, s, seed);
    std::memcpy(out, t.data.data(), t.size() * sizeof(float));
}

void ref_gen_gaussian_relu(int n, int c, int h, int w, uint64_t seed, float* out) {
    const plain_tensor t = gen_gaussian_relu(n, c, h, w, seed);
    std::memcpy(out, t.data.data(), t.size() * sizeof(float));
}

void ref_mt64_stream(uint64_t seed, uint64_t* out, size_t n) {
    std::mt19937_64 g(seed);
    for (size_t i = 0; i < n; ++i) out[i] = g();
}

// comp 0: dense_fwd(a=D, b=G); 1: dense_bwi(a=dY, b=G); 2: dense_bww(a=D, b=dY)
int ref_dense(int comp, const int* shape, const float* a, const float* b, float* out) {
    try {
        const conv_shape sh = to_shape(shape);
        const int hp = sh.out_h(), wp = sh.out_w();
        plain_tensor r;
        if (comp == 0)
            r = dense_fwd(plain_from(a, sh.N, sh.C, sh.H, sh.W), plain_from(b, sh.K, sh.C, sh.S, sh.R), sh);
        else if (comp == 1)
            r = dense_bwi(plain_from(a, sh.N, sh.K, hp, wp), plain_from(b, sh.K, sh.C, sh.S, sh.R), sh);
        else
            r = dense_bww(plain_from(a, sh.N, sh.C, sh.H, sh.W), plain_from(b, sh.N, sh.K, hp, wp), sh);
        std::memcpy(out, r.data.data(), r.size() * sizeof(float));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// expected_fma_counts with the default plan for (comp, V, check).
// rep = {checked, nonzero, executed, skipped}
int ref_expected_counts(int comp, int check, const int* shape, int V, const float* mask, uint64_t* rep) {
    try {
        const conv_shape sh = to_shape(shape);
        const kernel_plan pl = plan(sh, component(comp), V, 30, bww_check(check));
        const bool on_out = comp == 1 || (comp == 2 && check == 1);
        const plain_tensor m = on_out ? plain_from(mask, sh.N, sh.K, sh.out_h(), sh.out_w())
                                      : plain_from(mask, sh.N, sh.C, sh.H, sh.W);
        const fma_count_report r = expected_fma_counts(sh, pl, m);
        rep[0] = r.checked_vectors; rep[1] = r.nonzero_elements;
        rep[2] = r.executed_vector_fmas; rep[3] = r.skipped_vector_fmas;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Prepare a reference run on plain operands, packed exactly as the
// reference harness does (P/src/bench.cpp:106-159 / tests/testutil.hpp:43-78):
//   fwd: a = D -> ActNCHWc, b = G -> FilterKCRSblk
//   bwi: a = dY -> ActNCHWc, b = G -> FilterKCRSblk(swap_kc)
//   bww: a = D, b = dY; the tensor named by `check` goes ActCHWNn.
void* ref_prepare(int comp, int check, const int* shape, int V, int budget, const float* a, const float* b) {
    try {
        auto p = std::make_unique<prepared>();
        p->sh = to_shape(shape);
        const conv_shape& sh = p->sh;
        const int hp = sh.out_h(), wp = sh.out_w();
        p->pl = plan(sh, component(comp), V, budget, bww_check(check));
        if (comp == 0) {
            p->a = pack_act_nchwc(plain_from(a, sh.N, sh.C, sh.H, sh.W), V);
            p->b = pack_filter(plain_from(b, sh.K, sh.C, sh.S, sh.R), V);
        } else if (comp == 1) {
            p->a = pack_act_nchwc(plain_from(a, sh.N, sh.K, hp, wp), V);
            p->b = pack_filter(plain_from(b, sh.K, sh.C, sh.S, sh.R), V, true);
        } else {
            const plain_tensor D = plain_from(a, sh.N, sh.C, sh.H, sh.W);
            const plain_tensor dY = plain_from(b, sh.N, sh.K, hp, wp);
            if (check == 0) {
                p->a = pack_act_chwnn(D, V);
                p->b = pack_act_nchwc(dY, V);
            } else {
                p->a = pack_act_nchwc(D, V);
                p->b = pack_act_chwnn(dY, V);
            }
        }
        return p.release();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// The timed call: run_parallel on the prepared blocked operands
// (P/src/kernels.cpp:304-313).  pref: 0 automatic, 1 scalar, 2 native.
int ref_exec(void* h, int mode, int workers, int pref) {
    try {
        auto* p = static_cast<prepared*>(h);
        p->res = run_parallel(p->a, p->b, p->sh, p->pl, run_mode(mode), workers, backend_pref(pref));
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Result of the last ref_exec: plain output + counters + backend name.
int ref_result(void* h, float* out_plain, uint64_t* counters, char* backend, int backend_len) {
    auto* p = static_cast<prepared*>(h);
    const plain_tensor o = unpack(p->res.out);
    if (out_plain) std::memcpy(out_plain, o.data.data(), o.size() * sizeof(float));
    if (counters) {
        counters[0] = p->res.counters.checked_vectors;
        counters[1] = p->res.counters.executed_vector_fmas;
        counters[2] = p->res.counters.output_vector_loads;
        counters[3] = p->res.counters.output_vector_stores;
    }
    if (backend && backend_len > 0) {
        std::strncpy(backend, p->res.backend.c_str(), backend_len - 1);
        backend[backend_len - 1] = 0;
    }
    return 0;
}

// The prepared (blocked) operands, for feeding identical bytes to the GPU.
size_t ref_operand(void* h, int which, float* out) {
    auto* p = static_cast<prepared*>(h);
    const blocked_tensor& t = which == 0 ? p->a : p->b;
    if (out) std::memcpy(out, t.data.data(), t.data.size() * sizeof(float));
    return t.data.size();
}

// Raw blocked output of the last ref_exec (FilterKCRSblk for bww).
size_t ref_blocked_output(void* h, float* out) {
    auto* p = static_cast<prepared*>(h);
    if (out) std::memcpy(out, p->res.out.data.data(), p->res.out.data.size() * sizeof(float));
    return p->res.out.data.size();
}

void ref_free(void* h) { delete static_cast<prepared*>(h); }

int ref_native_backend_available(int V) { return native_backend_available(V) ? 1 : 0; }


// ---- harness (P/src/bench.cpp, P/src/projector.cpp) ----

static int put_str(const std::string& s, char* out, size_t len) {
    if (s.size() + 1 > len) { g_err = "buffer too small"; return 1; }
    std::memcpy(out, s.c_str(), s.size() + 1);
    return 0;
}

// layer_registry()/find_layer(): shape of the named layer (11 ints), -1 if unknown
int ref_find_layer(const char* name, int* shape_out) {
    const layer_config* lc = find_layer(name);
    if (!lc) return -1;
    const conv_shape& sh = lc->shape;
    const int v[11] = {sh.N, sh.C, sh.K, sh.H, sh.W, sh.R, sh.S, sh.O, sh.P, sh.padW, sh.padH};
    std::memcpy(shape_out, v, sizeof v);
    return 0;
}

int ref_registry_size() { return int(layer_registry().size()); }

int ref_registry_name(int i, char* out, size_t len) {
    const auto& reg = layer_registry();
    if (i < 0 || i >= int(reg.size())) return -1;
    return put_str(reg[i].name, out, len);
}

int ref_scaled_shape(const int* base, int minibatch, int scale, int* out) {
    try {
        const conv_shape sh = scaled_shape(to_shape(base), minibatch, scale);
        const int v[11] = {sh.N, sh.C, sh.K, sh.H, sh.W, sh.R, sh.S, sh.O, sh.P, sh.padW, sh.padH};
        std::memcpy(out, v, sizeof v);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// run_sweep() with workers = 1 and the given request; both CSVs returned
int ref_run_sweep(const char* layers_nl, int comps_mask, const double* grid, int ngrid, int minibatch, int scale,
                  uint64_t seed, int repeats, char* sweep_csv, size_t sweep_len, char* curves_csv,
                  size_t curves_len) {
    try {
        sweep_request req;
        req.layers.clear();
        std::istringstream ls(layers_nl);
        for (std::string l; std::getline(ls, l);)
            if (!l.empty()) req.layers.push_back(l);
        req.comps.clear();
        for (int c = 0; c < 3; ++c)
            if (comps_mask >> c & 1) req.comps.push_back(component(c));
        req.grid.assign(grid, grid + ngrid);
        req.minibatch = minibatch;
        req.scale = scale;
        req.seed = seed;
        req.repeats = repeats;
        const auto recs = run_sweep(req);
        std::ostringstream a, b;
        write_sweep_csv(recs, a);
        write_curves_csv(recs, b);
        return put_str(a.str(), sweep_csv, sweep_len) || put_str(b.str(), curves_csv, curves_len);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// write_sweep_csv / write_curves_csv of caller-supplied records
int ref_format_csv(int n, const char* layers_nl, const int* comps, const double* sparsity, const int* modes,
                   const int* workers, const double* median_ns, const uint64_t* exec_fmas, const double* speedups,
                   char* sweep_csv, size_t sweep_len, char* curves_csv, size_t curves_len) {
    try {
        std::vector<bench_record> recs(n);
        std::istringstream ls(layers_nl);
        for (int i = 0; i < n; ++i) {
            std::getline(ls, recs[i].layer);
            recs[i].comp = component(comps[i]);
            recs[i].sparsity = sparsity[i];
            recs[i].mode = run_mode(modes[i]);
            recs[i].workers = workers[i];
            recs[i].median_ns = median_ns[i];
            recs[i].exec_fmas = exec_fmas[i];
            recs[i].speedup_vs_dense = speedups[i];
        }
        std::ostringstream a, b;
        write_sweep_csv(recs, a);
        write_curves_csv(recs, b);
        return put_str(a.str(), sweep_csv, sweep_len) || put_str(b.str(), curves_csv, curves_len);
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// load_curves(): number of (layer, component) curves parsed, -1 on error
int ref_load_curves(const char* path) {
    try {
        return int(load_curves(path).curves.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

}  // extern "C"
