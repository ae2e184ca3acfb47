// test_dropin.cpp -- the C++ drop-in, tested the way the reference tests its
// kernels (P/tests/test_kernels.cpp): every case runs the UNMODIFIED reference
// (spconv::run_parallel, CPU, linked from oracle/_ref as the checker) and the
// B200 path (spconv::cuda::run_parallel) on the same blocked tensors.
// Exit status = number of failed checks.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <limits>
#include <random>

#include "spconv/kernels.hpp"
#include "spconv/oracle.hpp"
#include "spconv/sparsity.hpp"
#include "spconv_cuda.hpp"

using namespace spconv;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                                         \
    do {                                                         \
        if (cond) {                                              \
            ++g_pass;                                            \
        } else {                                                 \
            ++g_fail;                                            \
            std::printf("FAIL %s:%d: %s | ", __FILE__, __LINE__, #cond); \
            std::printf(__VA_ARGS__);                            \
            std::printf("\n");                                   \
        }                                                        \
    } while (0)

static double max_abs_rel(const plain_tensor& a, const plain_tensor& ref) {
    double md = 0, mr = 0;
    for (size_t e = 0; e < a.size(); ++e) {
        md = std::max(md, std::fabs(double(a.data[e]) - ref.data[e]));
        mr = std::max(mr, std::fabs(double(ref.data[e])));
    }
    return mr > 0 ? md / mr : md;
}

struct inputs {
    plain_tensor a_plain, b_plain;
    blocked_tensor a, b;
};

// testutil::make_inputs (P/tests/testutil.hpp:43-78)
static inputs make_inputs(const conv_shape& sh, component comp, bww_check check, double s, int V, u64 seed) {
    inputs in;
    const int hp = sh.out_h(), wp = sh.out_w();
    if (comp == component::fwd) {
        in.a_plain = gen_sparse(sh.N, sh.C, sh.H, sh.W, s, seed);
        in.b_plain = gen_sparse(sh.K, sh.C, sh.S, sh.R, 0.0, seed + 1);
        in.a = pack_act_nchwc(in.a_plain, V);
        in.b = pack_filter(in.b_plain, V);
    } else if (comp == component::bwi) {
        in.a_plain = gen_sparse(sh.N, sh.K, hp, wp, s, seed);
        in.b_plain = gen_sparse(sh.K, sh.C, sh.S, sh.R, 0.0, seed + 1);
        in.a = pack_act_nchwc(in.a_plain, V);
        in.b = pack_filter(in.b_plain, V, true);
    } else if (check == bww_check::input) {
        in.a_plain = gen_sparse(sh.N, sh.C, sh.H, sh.W, s, seed);
        in.b_plain = gen_sparse(sh.N, sh.K, hp, wp, 0.0, seed + 2);
        in.a = pack_act_chwnn(in.a_plain, V);
        in.b = pack_act_nchwc(in.b_plain, V);
    } else {
        in.a_plain = gen_sparse(sh.N, sh.C, sh.H, sh.W, 0.0, seed);
        in.b_plain = gen_sparse(sh.N, sh.K, hp, wp, s, seed + 2);
        in.a = pack_act_nchwc(in.a_plain, V);
        in.b = pack_act_chwnn(in.b_plain, V);
    }
    return in;
}

static void compare(const conv_shape& sh, component comp, bww_check check, int V, double s, u64 seed,
                    const char* what) {
    const kernel_plan pl = plan(sh, comp, V, 30, check);
    const kernel_plan pg = cuda::plan(sh, comp, V, 30, check);
    CHECK(pl.Q == pg.Q && pl.T == pg.T && pl.pipelined == pg.pipelined && pl.ring_size == pg.ring_size &&
              pl.M == pg.M,
          "%s plan mismatch", what);
    const inputs in = make_inputs(sh, comp, check, s, V, seed);
    for (run_mode mode : {run_mode::sparse, run_mode::dense}) {
        const conv_result ref = run_parallel(in.a, in.b, sh, pl, mode, 4);
        const conv_result got = cuda::run_parallel(in.a, in.b, sh, pg, mode, 1);
        CHECK(got.out.layout == ref.out.layout && got.out.data.size() == ref.out.data.size(), "%s header", what);
        const double err = max_abs_rel(unpack(got.out), unpack(ref.out));
        CHECK(err <= 1e-5, "%s comp=%s mode=%d s=%.1f err=%.3g", what, component_name(comp), int(mode), s, err);
        CHECK(got.counters == ref.counters,
              "%s comp=%s mode=%d counters checked %llu/%llu exec %llu/%llu loads %llu/%llu", what,
              component_name(comp), int(mode), (unsigned long long)got.counters.checked_vectors,
              (unsigned long long)ref.counters.checked_vectors,
              (unsigned long long)got.counters.executed_vector_fmas,
              (unsigned long long)ref.counters.executed_vector_fmas,
              (unsigned long long)got.counters.output_vector_loads,
              (unsigned long long)ref.counters.output_vector_loads);
        CHECK(got.backend == "cuda-sm100a", "backend name %s", got.backend.c_str());
    }
}

int main() {
    if (!cuda::native_backend_available(16)) {
        std::printf("no sm_100a device\n");
        return 2;
    }
    // kernels match the reference across random tiny shapes (test_kernels.cpp:26-47)
    std::mt19937_64 rng(101);
    auto pick = [&](std::initializer_list<int> xs) { return *(xs.begin() + rng() % xs.size()); };
    for (int trial = 0; trial < 24; ++trial) {
        const int V = pick({4, 8, 16});
        const int C = V * pick({1, 2, 4}), K = V * pick({1, 2, 4}), R = pick({1, 3, 3, 5});
        const int O = R == 1 ? 1 : pick({1, 1, 2});
        const conv_shape sh =
            conv_shape::make(int(rng() % 5) + 1, C, K, int(rng() % 6) + R, int(rng() % 6) + R, R, R, O, O);
        const double s = std::vector<double>{0.0, 0.3, 0.5, 0.8, 0.9, 1.0}[rng() % 6];
        for (component comp : {component::fwd, component::bwi, component::bww})
            for (bww_check chk : {bww_check::input, bww_check::output_grad}) {
                if (comp != component::bww && chk == bww_check::output_grad) continue;
                compare(sh, comp, chk, V, s, trial * 7 + 1, "random");
            }
    }
    // the tuned V=16 tile path (C,K multiples of 64), strides 1 and 2
    for (int R : {1, 3})
        for (int O : {1, 2}) {
            const conv_shape sh = conv_shape::make(3, 64, 128, 13, 11, R, R, O, O);
            for (component comp : {component::fwd, component::bwi, component::bww})
                for (bww_check chk : {bww_check::input, bww_check::output_grad}) {
                    if (comp != component::bww && chk == bww_check::output_grad) continue;
                    compare(sh, comp, chk, 16, 0.6, 5, "tile");
                }
        }
    // run_batch: three passes in one call equal the reference and the per-call results
    {
        const auto sh = conv_shape::make(3, 64, 128, 13, 11, 3, 3, 1, 1);
        std::vector<inputs> ins;
        std::vector<cuda::pass_request> reqs;
        std::vector<kernel_plan> pls;
        for (component comp : {component::fwd, component::bwi, component::bww}) {
            ins.push_back(make_inputs(sh, comp, bww_check::input, 0.6, 16, 77));
            pls.push_back(cuda::plan(sh, comp, 16, 30, bww_check::input));
        }
        for (size_t i = 0; i < ins.size(); ++i)
            reqs.push_back(cuda::pass_request{&ins[i].a, &ins[i].b, sh, pls[i], run_mode::sparse});
        const std::vector<conv_result> got = cuda::run_batch(reqs);
        CHECK(got.size() == 3, "run_batch size");
        for (size_t i = 0; i < got.size(); ++i) {
            const conv_result one = cuda::run_parallel(ins[i].a, ins[i].b, sh, pls[i], run_mode::sparse, 1);
            const conv_result ref = run_parallel(ins[i].a, ins[i].b, sh, plan(sh, pls[i].comp, 16, 30, bww_check::input),
                                                 run_mode::sparse, 4);
            CHECK(got[i].out.data == one.out.data, "run_batch pass %zu differs from the per-call result", i);
            CHECK(got[i].counters == ref.counters, "run_batch pass %zu counters", i);
            CHECK(max_abs_rel(unpack(got[i].out), unpack(ref.out)) <= 1e-5, "run_batch pass %zu value", i);
        }
    }
    // single interior non-zero: exactly 36 vector FMAs (test_kernels.cpp:97-110)
    {
        const int V = 8;
        const auto sh = conv_shape::make(1, 32, 32, 8, 8, 3, 3, 1, 1);
        plain_tensor D(1, 32, 8, 8);
        D.at(0, 5, 4, 4) = 0.7f;
        const plain_tensor G = gen_sparse(32, 32, 3, 3, 0.0, 2);
        const conv_result r = cuda::sparse_fwd(pack_act_nchwc(D, V), pack_filter(G, V), sh,
                                               cuda::plan(sh, component::fwd, V), run_mode::sparse);
        CHECK(r.counters.executed_vector_fmas == 36u, "36 FMAs: %llu",
              (unsigned long long)r.counters.executed_vector_fmas);
        CHECK(max_rel_error(unpack(r.out), dense_fwd(D, G, sh)) <= 1e-4, "single nonzero value");
    }
    // layout and plan mismatches throw spconv::error (test_kernels.cpp:328-352)
    {
        const int V = 8;
        const auto sh = conv_shape::make(2, 16, 16, 6, 6, 3, 3, 1, 1);
        const kernel_plan pl = cuda::plan(sh, component::fwd, V);
        const inputs in = make_inputs(sh, component::fwd, bww_check::input, 0.5, V, 1);
        auto throws = [&](auto fn) {
            try {
                fn();
            } catch (const error&) {
                return true;
            }
            return false;
        };
        blocked_tensor bad = in.b;
        bad.layout = tensor_layout::act_nchwc;
        CHECK(throws([&] { cuda::sparse_fwd(in.a, bad, sh, pl, run_mode::sparse); }), "bad filter layout");
        blocked_tensor wv = in.a;
        wv.V = 4;
        CHECK(throws([&] { cuda::sparse_fwd(wv, in.b, sh, pl, run_mode::sparse); }), "wrong V");
        CHECK(throws([&] { cuda::sparse_fwd(in.a, in.b, sh, cuda::plan(sh, component::bwi, V), run_mode::sparse); }),
              "plan for another component");
        CHECK(throws([&] { cuda::plan(conv_shape::make(2, 16, 12, 6, 6, 3, 3, 1, 1), component::fwd, 8); }),
              "K not a multiple of V");
        CHECK(throws([&] { cuda::sparse_fwd(in.a, in.b, sh, pl, run_mode::sparse, 0); }), "workers = 0");
    }
    // vector_probes (kernels.hpp:90-98): the device backend's contract ops vs
    // the reference's native backend on the same vectors (test_vec.cpp:38-57)
    for (int V : {4, 8, 16}) {
        const auto ours = cuda::vector_probes(V);
        const auto refs = vector_probes(V);
        CHECK(ours.size() == 1 && ours[0].width == V && ours[0].native, "vector_probes(%d) shape", V);
        const vec_probe* rp = nullptr;
        for (const auto& p : refs)
            if (p.native) rp = &p;
        if (!rp && !refs.empty()) rp = &refs.front();
        std::mt19937_64 rng(V);
        std::normal_distribution<float> nd(0.0f, 1.0f);
        for (int t = 0; t < 20; ++t) {
            float v[16], a[16], w[16], a2[16], b2[16];
            for (int j = 0; j < V; ++j) {
                v[j] = (rng() % 3 == 0) ? 0.0f : nd(rng);
                a[j] = nd(rng);
                w[j] = nd(rng);
            }
            v[0] = -0.0f;
            if (V >= 8) { v[2] = std::numeric_limits<float>::quiet_NaN(); v[3] = std::numeric_limits<float>::infinity(); }
            CHECK(ours[0].cmp_neq_zero(v) == rp->cmp_neq_zero(v), "cmp_neq_zero V=%d", V);
            const float s = nd(rng);
            std::memcpy(a2, a, sizeof(a));
            ours[0].broadcast_fma(a, s, w);
            rp->broadcast_fma(a2, s, w);
            CHECK(std::memcmp(a, a2, V * sizeof(float)) == 0 || !rp->native, "broadcast_fma V=%d", V);
            std::memcpy(b2, a, sizeof(a));
            ours[0].add(a, w);
            rp->add(b2, w);
            CHECK(std::memcmp(a, b2, V * sizeof(float)) == 0, "add V=%d", V);
        }
    }
    std::printf("%d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
