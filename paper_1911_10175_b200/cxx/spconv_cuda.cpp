// spconv_cuda.cpp -- spconv::cuda::* over the C ABI (see spconv_cuda.hpp).
#include "spconv_cuda.hpp"

#include <cstring>

#include "../../include/spconv_b200.h"

namespace spconv::cuda {

namespace {

spc_shape to_c(const conv_shape& s) {
    return spc_shape{s.N, s.C, s.K, s.H, s.W, s.R, s.S, s.O, s.P, s.padW, s.padH};
}

spc_plan to_c(const kernel_plan& p) {
    return spc_plan{int(p.comp), int(p.check), p.V, p.Q, p.T, p.pipelined ? 1 : 0, p.ring_size, p.M,
                    p.register_budget, p.unroll_hint, p.prefetch_hints ? 1 : 0};
}

int layout_to_c(tensor_layout l) {
    switch (l) {
    case tensor_layout::plain: return SPC_LAYOUT_PLAIN;
    case tensor_layout::act_nchwc: return SPC_LAYOUT_ACT_NCHWC;
    case tensor_layout::filter_kcrs_blk: return SPC_LAYOUT_FILTER_KCRS_BLK;
    case tensor_layout::act_chwnn: return SPC_LAYOUT_ACT_CHWNN;
    }
    return -1;
}

spc_tensor to_c(const blocked_tensor& t) {
    spc_tensor c;
    c.layout = layout_to_c(t.layout);
    c.V = t.V;
    c.n = t.n; c.c = t.c; c.h = t.h; c.w = t.w;
    c.k = t.k; c.r = t.r; c.s = t.s;
    c.data = const_cast<float*>(t.data.data());  // read-only on the input side
    c.numel = t.data.size();
    return c;
}

void check(spc_status st) {
    if (st != SPC_OK) throw error(std::string(spc_last_error()));
}

conv_result run(component comp, const blocked_tensor& a, const blocked_tensor& b, const conv_shape& shape,
                const kernel_plan& pl, run_mode mode, int workers, backend_pref pref) {
    SPCONV_REQUIRE(workers >= 1, "workers must be >= 1");                       // kernels.cpp:109
    SPCONV_REQUIRE(pl.comp == comp, "plan was built for another component");    // kernels.cpp:107
    SPCONV_REQUIRE(pref != backend_pref::force_scalar,
                   "force_scalar: the CUDA backend has no scalar emulation");
    const spc_shape cs = to_c(shape);
    const spc_plan cp = to_c(pl);
    spc_tensor od;
    std::memset(&od, 0, sizeof(od));
    check(spc_output_desc(&cs, &cp, &od));

    conv_result res;
    res.out.layout = od.layout == SPC_LAYOUT_FILTER_KCRS_BLK ? tensor_layout::filter_kcrs_blk
                                                             : tensor_layout::act_nchwc;
    res.out.V = od.V;
    res.out.n = od.n; res.out.c = od.c; res.out.h = od.h; res.out.w = od.w;
    res.out.k = od.k; res.out.r = od.r; res.out.s = od.s;
    res.out.data.assign(od.numel, 0.0f);

    const spc_tensor ca = to_c(a), cb = to_c(b);
    spc_tensor cd = od;
    cd.data = res.out.data.data();
    cd.numel = res.out.data.size();
    spc_counters cnt;
    std::memset(&cnt, 0, sizeof(cnt));
    check(spc_run_parallel_host(&ca, &cb, &cs, &cp, mode == run_mode::sparse ? SPC_SPARSE : SPC_DENSE, &cd, &cnt));
    res.counters.checked_vectors = cnt.checked_vectors;
    res.counters.executed_vector_fmas = cnt.executed_vector_fmas;
    res.counters.output_vector_loads = cnt.output_vector_loads;
    res.counters.output_vector_stores = cnt.output_vector_stores;
    res.backend = spc_backend_name();
    return res;
}

}  // namespace

std::vector<conv_result> run_batch(const std::vector<pass_request>& passes) {
    const size_t n = passes.size();
    std::vector<conv_result> res(n);
    std::vector<spc_shape> cs(n);
    std::vector<spc_plan> cp(n);
    std::vector<spc_tensor> ca(n), cb(n), cd(n);
    std::vector<spc_counters> cnt(n);
    std::vector<spc_host_pass> hp(n);
    for (size_t i = 0; i < n; ++i) {
        const pass_request& p = passes[i];
        SPCONV_REQUIRE(p.a != nullptr && p.b != nullptr, "run_batch: null operand");
        cs[i] = to_c(p.shape);
        cp[i] = to_c(p.plan);
        spc_tensor od;
        std::memset(&od, 0, sizeof(od));
        check(spc_output_desc(&cs[i], &cp[i], &od));
        conv_result& r = res[i];
        r.out.layout = od.layout == SPC_LAYOUT_FILTER_KCRS_BLK ? tensor_layout::filter_kcrs_blk
                                                               : tensor_layout::act_nchwc;
        r.out.V = od.V;
        r.out.n = od.n; r.out.c = od.c; r.out.h = od.h; r.out.w = od.w;
        r.out.k = od.k; r.out.r = od.r; r.out.s = od.s;
        r.out.data.assign(od.numel, 0.0f);
        ca[i] = to_c(*p.a);
        cb[i] = to_c(*p.b);
        cd[i] = od;
        cd[i].data = r.out.data.data();
        cd[i].numel = r.out.data.size();
        std::memset(&cnt[i], 0, sizeof(spc_counters));
        // a BWW checked operand given in act_nchwc is packed into act_chwnn on the device
        const blocked_tensor& chk = p.plan.check == bww_check::input ? *p.a : *p.b;
        const int flags =
            p.plan.comp == component::bww && chk.layout == tensor_layout::act_nchwc ? SPC_PASS_CHECKED_NCHWC : 0;
        hp[i] = spc_host_pass{&ca[i], &cb[i], &cs[i], &cp[i], p.mode == run_mode::sparse ? SPC_SPARSE : SPC_DENSE,
                              &cd[i], &cnt[i], SPC_OK, flags};
    }
    check(spc_run_parallel_host_batch(hp.data(), (int)n));
    for (size_t i = 0; i < n; ++i) {
        res[i].counters.checked_vectors = cnt[i].checked_vectors;
        res[i].counters.executed_vector_fmas = cnt[i].executed_vector_fmas;
        res[i].counters.output_vector_loads = cnt[i].output_vector_loads;
        res[i].counters.output_vector_stores = cnt[i].output_vector_stores;
        res[i].backend = spc_backend_name();
    }
    return res;
}

kernel_plan plan(const conv_shape& shape, component comp, int V, int register_budget, bww_check chk) {
    const spc_shape cs = to_c(shape);
    spc_plan p;
    check(spc_plan_make(&cs, int(comp), V, register_budget, int(chk), &p));
    kernel_plan out;
    out.comp = component(p.comp);
    out.check = bww_check(p.check);
    out.V = p.V;
    out.Q = p.Q;
    out.T = p.T;
    out.pipelined = p.pipelined != 0;
    out.ring_size = p.ring_size;
    out.M = p.M;
    out.register_budget = p.register_budget;
    out.unroll_hint = p.unroll_hint;
    out.prefetch_hints = p.prefetch_hints != 0;
    return out;
}

bool native_backend_available(int V) { return spc_native_backend_available(V) != 0; }

std::vector<std::string> backend_names() { return {spc_backend_name()}; }

namespace {
// vec_probe holds plain function pointers without a width: one set per V.
template <int V>
lane_mask probe_cmp(const float* v) {
    uint32_t m = 0;
    check(spc_vector_probe(V, SPC_PROBE_CMP_NEQ_ZERO, v, nullptr, 0.0f, nullptr, &m));
    return m;
}
template <int V>
void probe_fma(float* acc, float s, const float* w) {
    check(spc_vector_probe(V, SPC_PROBE_BROADCAST_FMA, acc, w, s, acc, nullptr));
}
template <int V>
void probe_add(float* a, const float* b) {
    check(spc_vector_probe(V, SPC_PROBE_ADD, a, b, 0.0f, a, nullptr));
}
template <int V>
vec_probe make_probe() {
    vec_probe p;
    p.name = spc_backend_name();
    p.width = V;
    p.native = true;
    p.cmp_neq_zero = &probe_cmp<V>;
    p.broadcast_fma = &probe_fma<V>;
    p.add = &probe_add<V>;
    return p;
}
}  // namespace

std::vector<vec_probe> vector_probes(int V) {
    switch (V) {
    case 4: return {make_probe<4>()};
    case 8: return {make_probe<8>()};
    case 16: return {make_probe<16>()};
    default: throw error("vector_probes: V must be 4, 8 or 16");
    }
}

conv_result sparse_fwd(const blocked_tensor& src, const blocked_tensor& filt, const conv_shape& shape,
                       const kernel_plan& pl, run_mode mode, int workers, backend_pref pref) {
    return run(component::fwd, src, filt, shape, pl, mode, workers, pref);
}

conv_result sparse_bwi(const blocked_tensor& grad_out, const blocked_tensor& filt_t, const conv_shape& shape,
                       const kernel_plan& pl, run_mode mode, int workers, backend_pref pref) {
    return run(component::bwi, grad_out, filt_t, shape, pl, mode, workers, pref);
}

conv_result sparse_bww(const blocked_tensor& input, const blocked_tensor& grad_out, const conv_shape& shape,
                       const kernel_plan& pl, run_mode mode, int workers, backend_pref pref) {
    return run(component::bww, input, grad_out, shape, pl, mode, workers, pref);
}

conv_result run_parallel(const blocked_tensor& a, const blocked_tensor& b, const conv_shape& shape,
                         const kernel_plan& pl, run_mode mode, int workers, backend_pref pref) {
    switch (pl.comp) {
    case component::fwd: return cuda::sparse_fwd(a, b, shape, pl, mode, workers, pref);
    case component::bwi: return cuda::sparse_bwi(a, b, shape, pl, mode, workers, pref);
    case component::bww: return cuda::sparse_bww(a, b, shape, pl, mode, workers, pref);
    }
    throw error("run_parallel: bad component");
}

}  // namespace spconv::cuda
