// spconv_cuda.hpp -- C++ drop-in for the reference's hot-path API on B200.
//
// Same signatures, types and error behaviour as the reference's layer API
// (P/include/spconv/kernels.hpp:53-98, planner.hpp:44-46), in namespace
// spconv::cuda.  The reference's own headers define the types (included by
// path, -I $SPCONV_REF/include); no reference code is linked.  Every call
// goes through the C ABI of libspconv_b200.so (include/spconv_b200.h) with
// host buffers: copy in, sm_100a kernels, copy out -- synchronous and
// reentrant like the reference.  Contract violations throw spconv::error
// before any device work.
#pragma once

#include <string>
#include <vector>

#include "spconv/kernels.hpp"
#include "spconv/planner.hpp"
#include "spconv/tensor.hpp"

namespace spconv::cuda {

// spconv::plan (P/src/planner.cpp:25-73), computed by spc_plan_make.
kernel_plan plan(const conv_shape& shape, component comp, int V, int register_budget = 30,
                 bww_check check = bww_check::input);

bool native_backend_available(int V);
std::vector<std::string> backend_names();
// vector_probes (P/include/spconv/kernels.hpp:90-98): the device backend's
// contract operations (spc_vector_probe), one warp, lane j = vector lane j.
std::vector<vec_probe> vector_probes(int V);

conv_result sparse_fwd(const blocked_tensor& src, const blocked_tensor& filt, const conv_shape& shape,
                       const kernel_plan& plan, run_mode mode, int workers = 1,
                       backend_pref pref = backend_pref::automatic);
conv_result sparse_bwi(const blocked_tensor& grad_out, const blocked_tensor& filt_t, const conv_shape& shape,
                       const kernel_plan& plan, run_mode mode, int workers = 1,
                       backend_pref pref = backend_pref::automatic);
conv_result sparse_bww(const blocked_tensor& input, const blocked_tensor& grad_out, const conv_shape& shape,
                       const kernel_plan& plan, run_mode mode, int workers = 1,
                       backend_pref pref = backend_pref::automatic);
conv_result run_parallel(const blocked_tensor& a, const blocked_tensor& b, const conv_shape& shape,
                         const kernel_plan& plan, run_mode mode, int workers,
                         backend_pref pref = backend_pref::automatic);

// A list of passes in one call (spc_run_parallel_host_batch): the reference's bench loop over
// layers and components (P/src/bench.cpp:216-288) with the copies and kernels of consecutive
// passes pipelined.  Same results, counters and errors per pass as run_parallel; every pass is
// validated before any device work.  blocked_tensor keeps its data in a std::vector (pageable
// memory), which the library moves through its pinned staging ring pass by pass; buffers
// registered with cudaHostRegister are pipelined across passes.
struct pass_request {
    const blocked_tensor* a;
    const blocked_tensor* b;
    conv_shape shape;
    kernel_plan plan;
    run_mode mode = run_mode::sparse;
};
std::vector<conv_result> run_batch(const std::vector<pass_request>& passes);

}  // namespace spconv::cuda
