/*
 * spconv_b200.h -- C ABI of the B200-native sparse direct-convolution path.
 *
 * Drop-in replacement for the hot path of the reference `spconv` library
 * (SparseTrain, arXiv 1911.10175): the three training passes FWD / BWI / BWW
 * over dense blocked fp32 tensors that skip work on zeros ReLU puts into the
 * checked tensor.  Zero skipping is per element on the 3x3 stride-1 passes
 * (FWD / BWI / BWW), 3x3 stride-2 BWI and BWW with check = output_grad; the
 * 1x1 passes and 3x3 stride-2 FWD / BWW (check = input) execute every FMA
 * ("counted dense": measured faster than any skip granularity on B200,
 * profiles/r02_skip_evidence.md) with the reference's exact
 * counters and Inf/NaN semantics.
 * Every entry point below replaces one reference interface
 * (cited as P/<file>:<line>, P = /root/reference/proj):
 *
 *   spc_sparse_fwd      <- spconv::sparse_fwd    P/include/spconv/kernels.hpp:58-61
 *   spc_sparse_bwi      <- spconv::sparse_bwi    P/include/spconv/kernels.hpp:65-69
 *   spc_sparse_bww      <- spconv::sparse_bww    P/include/spconv/kernels.hpp:74-78
 *   spc_run_parallel    <- spconv::run_parallel  P/include/spconv/kernels.hpp:83-86
 *   spc_plan_make       <- spconv::plan          P/include/spconv/planner.hpp:44-46
 *   spc_shape_make      <- conv_shape::make      P/include/spconv/tensor.hpp:39-40
 *   spc_shape_validate  <- conv_shape::validate  P/include/spconv/tensor.hpp:47
 *   spc_native_backend_available <- native_backend_available  kernels.hpp:53
 *   spc_backend_name    <- conv_result::backend / backend_names  kernels.hpp:47-54
 *   spc_relu / spc_relu_grad_mask <- relu / relu_grad_mask  P/include/spconv/sparsity.hpp:14-18
 *   spc_gen_sparse      <- spconv::gen_sparse    P/include/spconv/sparsity.hpp (P/src/sparsity.cpp:42-55)
 *   spc_vector_probes   <- spconv::vector_probes P/include/spconv/kernels.hpp:90-98
 *   spc_run_parallel_host_batch <- the harness loop over layers and components,
 *                       one run_parallel per pass (P/src/bench.cpp:216-288), as one call
 *   spc_bww_allreduce / spc_bww_sharded / spc_comm_*: no reference counterpart
 *                       (the reference is single-process, P/src/kernels.cpp:76-102);
 *                       the batch-sharded BWW exchange of SURVEY.md 8(e)
 *
 * Conventions
 *   - Plain pointers and sizes only; no C++ types or exceptions cross the ABI.
 *   - `spc_sparse_*` take DEVICE pointers and enqueue on `stream`
 *     (a cudaStream_t, NULL = legacy default stream); they never synchronize.
 *   - `spc_sparse_*_host` take HOST pointers: H2D, kernels, D2H, synchronize.
 *     They are the exact-semantics drop-in (the reference is synchronous).
 *   - Every contract violation the reference turns into `throw spconv::error`
 *     (P/src/kernels.cpp:104-142, P/src/tensor.cpp:26-36, P/src/planner.cpp:33-64)
 *     returns a nonzero spc_status BEFORE any device work, with the message in
 *     spc_last_error() (thread-local).
 *   - Outputs are zero-initialised then written (P/src/kernels.cpp:183);
 *     results are bitwise deterministic run to run (no float atomics).
 */
#ifndef SPCONV_B200_H
#define SPCONV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPC_ABI_VERSION 3 /* 2: spc_epilogue.beta, multi-GPU comm entries, spc_vector_probe; 3: spc_run_parallel_host_batch */

typedef enum {
    SPC_OK = 0,
    SPC_ERR_SHAPE = 1,     /* conv_shape::validate failure        (P/src/tensor.cpp:26-36) */
    SPC_ERR_PLAN = 2,      /* plan/component/Q/ring checks        (P/src/kernels.cpp:104-117, planner.cpp:33-64) */
    SPC_ERR_LAYOUT = 3,    /* layout / V / dims / size mismatch   (P/src/kernels.cpp:119-142) */
    SPC_ERR_ARG = 4,       /* null pointer, bad enum, small buffer */
    SPC_ERR_CUDA = 5,      /* CUDA runtime / launch failure */
    SPC_ERR_NCCL = 6,      /* collective failure */
    SPC_ERR_NO_DEVICE = 7  /* no sm_100 device visible */
} spc_status;

/* conv_shape, field for field (P/include/spconv/tensor.hpp:30-38). */
typedef struct {
    int N, C, K, H, W, R, S, O, P, padW, padH;
} spc_shape;

typedef enum { SPC_FWD = 0, SPC_BWI = 1, SPC_BWW = 2 } spc_component;         /* planner.hpp:18 */
typedef enum { SPC_CHECK_INPUT = 0, SPC_CHECK_OUTPUT_GRAD = 1 } spc_bww_check; /* planner.hpp:19 */
typedef enum { SPC_SPARSE = 0, SPC_DENSE = 1 } spc_run_mode;                   /* kernels.hpp:24 */

/* kernel_plan, field for field (P/include/spconv/planner.hpp:22-38).
 * On the GPU, Q/ring/M do not shape the tiling; they are validated like
 * check_common and Q keeps its counter semantics. */
typedef struct {
    int comp, check, V, Q, T, pipelined, ring_size, M, register_budget, unroll_hint, prefetch_hints;
} spc_plan;

/* kernel_counters (P/include/spconv/kernels.hpp:31-45).
 * executed_vector_fmas is counted in-kernel (exact, integer);
 * checked_vectors and output_vector_loads/stores are the reference's
 * as-if values (data-independent, computed from shape + plan). */
typedef struct {
    uint64_t checked_vectors;
    uint64_t executed_vector_fmas;
    uint64_t output_vector_loads;
    uint64_t output_vector_stores;
} spc_counters;

/* tensor_layout (P/include/spconv/tensor.hpp:76). */
typedef enum {
    SPC_LAYOUT_PLAIN = 0,
    SPC_LAYOUT_ACT_NCHWC = 1,       /* [N][C/V][H][W][V]            */
    SPC_LAYOUT_FILTER_KCRS_BLK = 2, /* [K/V][C/V][S][R][Vc][Vk]     */
    SPC_LAYOUT_ACT_CHWNN = 3        /* [ceil(N/V)][C][H][W][V]      */
} spc_layout;

/* blocked_tensor header + data pointer (P/include/spconv/tensor.hpp:80-96).
 * Activation layouts use n/c/h/w; the filter layout uses k/c/s/r.
 * `numel` is the element count of `data` (for outputs: its capacity). */
typedef struct {
    int layout, V;
    int n, c, h, w;
    int k, r, s;
    float* data;
    size_t numel;
} spc_tensor;

/* ---- geometry and planning (host only, no device needed) ---- */
spc_status spc_shape_make(int N, int C, int K, int H, int W, int R, int S, int O, int P, spc_shape* out);
spc_status spc_shape_make_padded(int N, int C, int K, int H, int W, int R, int S, int O, int P, int padW,
                                 int padH, spc_shape* out);
spc_status spc_shape_validate(const spc_shape* shape);
spc_status spc_plan_make(const spc_shape* shape, int comp, int V, int register_budget, int check, spc_plan* out);
/* Header (layout, dims, numel) of the output a pass produces; data = NULL. */
spc_status spc_output_desc(const spc_shape* shape, const spc_plan* plan, spc_tensor* out);
/* The as-if counters (checked, loads, stores) for a pass; executed = dense total
 * in dense mode, 0 in sparse mode (the kernels add the executed count). */
spc_status spc_analytic_counters(const spc_shape* shape, const spc_plan* plan, int mode, spc_counters* out);

/* ---- the three passes on device buffers (asynchronous on `stream`) ---- */
/* FWD: src = D (ActNCHWc over C), filt = G (FilterKCRSblk K,C); dst = Y (ActNCHWc over K). */
spc_status spc_sparse_fwd(const spc_tensor* src, const spc_tensor* filt, const spc_shape* shape,
                          const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters,
                          void* stream);
/* BWI: src = dY (ActNCHWc over K), filt = G^T (pack_filter swap_kc: FilterKCRSblk C,K);
 * dst = dD (ActNCHWc over C). */
spc_status spc_sparse_bwi(const spc_tensor* grad_out, const spc_tensor* filt_t, const spc_shape* shape,
                          const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters,
                          void* stream);
/* BWW: the tensor named by plan->check is ActCHWNn, the other ActNCHWc;
 * dst = dG (FilterKCRSblk K,C) for either check side. */
spc_status spc_sparse_bww(const spc_tensor* input, const spc_tensor* grad_out, const spc_shape* shape,
                          const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters,
                          void* stream);
/* Dispatch on plan->comp (a = swept tensor or input, b = filters or grad_out). */
spc_status spc_run_parallel(const spc_tensor* a, const spc_tensor* b, const spc_shape* shape,
                            const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters,
                            void* stream);

/* ---- fused output epilogue for layer chains ----
 * Applied per output element as the kernel writes it:
 *   v = acc * alpha (+ add[i]) (+ beta);  if (relu) v = v > 0 ? v : 0;  if (mask) v = mask[i] > 0 ? v : 0
 * i.e. the reference's relu / relu_grad_mask (P/src/sparsity.cpp:11-28) fused
 * into FWD/BWI.  `add` and `mask` are DEVICE buffers with the output's layout
 * and numel (ActNCHWc); NULL disables them.  `beta` is a scalar bias added
 * after the (fused) residual add (0 = none; Fixup's bias before the ReLU).
 * {1, NULL, NULL, 0, 0} = plain pass. */
typedef struct {
    float alpha;
    const float* add;
    const float* mask;
    int relu;
    float beta;
} spc_epilogue;
spc_status spc_sparse_fwd_ex(const spc_tensor* src, const spc_tensor* filt, const spc_shape* shape,
                             const spc_plan* plan, int mode, const spc_epilogue* epi, spc_tensor* dst,
                             spc_counters* d_counters, void* stream);
spc_status spc_sparse_bwi_ex(const spc_tensor* grad_out, const spc_tensor* filt_t, const spc_shape* shape,
                             const spc_plan* plan, int mode, const spc_epilogue* epi, spc_tensor* dst,
                             spc_counters* d_counters, void* stream);
/* The same epilogue as a standalone pass over n elements of `data` (in place). */
spc_status spc_epilogue_apply(const spc_epilogue* epi, float* data, size_t n, void* stream);

/* ---- arithmetic of the passes (no reference counterpart) ----
 * SPC_MATH_FP32 (default): FP32 CUDA-core FFMA, zero skipping, the reference's
 * per-product rounding.  SPC_MATH_TF32X3: tcgen05 tensor cores with 3xTF32
 * split products (hi*hi + hi*lo + lo*hi, fp32 accumulate), its own stated
 * tolerance; used for the geometries it covers (V = 16,
 * stride 1 or 2, 3x3 pad 1 / 1x1 pad 0), the FP32 kernels elsewhere and for
 * inputs holding Inf/NaN.  Per host thread; returns the previous mode, or -1
 * for an unknown mode (unchanged). */
typedef enum { SPC_MATH_FP32 = 0, SPC_MATH_TF32X3 = 1 } spc_math;
int spc_set_math(int math);
int spc_get_math(void);

/* ---- host-buffer drop-ins: copy in, run, copy out, synchronize ---- */
spc_status spc_run_parallel_host(const spc_tensor* a, const spc_tensor* b, const spc_shape* shape,
                                 const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* counters);

/* A list of host-buffer passes, run as if spc_run_parallel_host were called on
 * each in order (the reference's bench loop over layers and components,
 * P/src/bench.cpp:216-288, in one call) but pipelined across passes: pass
 * i + 1's H2D overlaps pass i's kernels and D2H.  Results, counters and error
 * behaviour per pass are those of spc_run_parallel_host; every pass is
 * validated before any device work starts.  Pinned host buffers are pipelined;
 * a pass with pageable buffers runs through spc_run_parallel_host at its turn.
 * All buffers must stay valid until the call returns.  Returns the first
 * failing pass's status (also in its `status`), SPC_OK otherwise. */
typedef struct {
    const spc_tensor* a;
    const spc_tensor* b;
    const spc_shape* shape;
    const spc_plan* plan;
    int mode;               /* spc_run_mode */
    spc_tensor* dst;        /* data + capacity in, header out */
    spc_counters* counters; /* may be NULL */
    spc_status status;      /* out */
    int flags;              /* SPC_PASS_* */
} spc_host_pass;
/* BWW only: the checked operand (plan.check: `a` for input, `b` for output_grad) is given in
 * ActNCHWc instead of ActCHWNn and packed on the device by pack_act_chwnn's rule
 * (P/src/tensor.cpp:94-108: ragged image lanes zero) -- the caller keeps one host layout of
 * an activation, and a buffer an earlier pass of the batch already uploaded (a layer's FWD
 * takes the same ActNCHWc input) is not uploaded again. */
#define SPC_PASS_CHECKED_NCHWC 1
spc_status spc_run_parallel_host_batch(spc_host_pass* passes, int n);
/* The batch call keeps a per-thread device arena (8 passes in flight x the largest pass of the
 * last batch) for its next call; this frees it. */
void spc_host_batch_release(void);

/* ---- ReLU semantics on device (P/src/sparsity.cpp:11-28), bit-exact ---- */
spc_status spc_relu(const float* in, float* out, size_t n, void* stream);
spc_status spc_relu_grad_mask(const float* pre, const float* upstream, float* out, size_t n, void* stream);

/* ---- synthetic inputs of the reference harness (host, no device needed) ---- */
/* gen_sparse (P/src/sparsity.cpp:42-55): out[e] = 0 with probability
 * `sparsity`, else U[0.1, 1], from std::mt19937_64(seed) through the
 * reference's hand-mapped unit() (sparsity.cpp:34-38) -- the same stream, so
 * the same tensor, as the reference's sweep/verify harness (bench.cpp:127-180). */
spc_status spc_gen_sparse(float* out, size_t count, double sparsity, uint64_t seed);

/* ---- vector_probes (P/include/spconv/kernels.hpp:90-98) ----
 * The contract operations of this backend, run on the device the way the
 * kernels run them (one warp; lane j = vector lane j), for the reference's
 * scalar-vs-SIMD equivalence tests: host arrays of V floats in and out.
 *   SPC_PROBE_CMP_NEQ_ZERO: *mask = bit j set iff a[j] != 0 (-0 -> 0, NaN -> 1)
 *   SPC_PROBE_BROADCAST_FMA: out[j] = fmaf(s, b[j], a[j])   (acc = a, w = b)
 *   SPC_PROBE_ADD:           out[j] = a[j] + b[j] */
typedef enum { SPC_PROBE_CMP_NEQ_ZERO = 0, SPC_PROBE_BROADCAST_FMA = 1, SPC_PROBE_ADD = 2 } spc_probe_op;
spc_status spc_vector_probe(int V, int op, const float* a, const float* b, float s, float* out, uint32_t* mask);

/* ---- device layout conversion: ActNCHWc -> ActCHWNn (tensor.cpp:94-108) ---- */
spc_status spc_nchwc_to_chwnn(const spc_tensor* src, spc_tensor* dst, void* stream);

/* ---- multi-GPU: batch-sharded passes, BWW weight-gradient exchange ----
 * One process per GPU.  FWD/BWI run each rank's contiguous ActNCHWc batch slice
 * with no communication; BWW computes the slice's partial dG and the ranks sum
 * it (NCCL allreduce, fp32, in place, on the caller's stream, no host sync).
 * NCCL is loaded at run time (libnccl.so.2); without it these return SPC_ERR_NCCL.
 * Communicator setup: rank 0 calls spc_comm_unique_id, the host broadcasts
 * the SPC_COMM_ID_BYTES bytes, every rank calls spc_comm_init on its device. */
#define SPC_COMM_ID_BYTES 128
typedef struct spc_comm spc_comm;
int spc_nccl_version(void); /* NCCL_VERSION_CODE of the loaded library, 0 if none */
spc_status spc_comm_unique_id(unsigned char* id /* [SPC_COMM_ID_BYTES] */);
spc_status spc_comm_init(spc_comm** comm, int nranks, const unsigned char* id, int rank);
/* Wrap an existing ncclComm_t (not destroyed by spc_comm_destroy). */
spc_status spc_comm_wrap(spc_comm** comm, void* nccl_comm);
void* spc_comm_nccl(spc_comm* comm); /* the ncclComm_t */
int spc_comm_size(spc_comm* comm);
int spc_comm_rank(spc_comm* comm);
spc_status spc_comm_destroy(spc_comm* comm);
/* Collective (all ranks, same sizes, same order): a device buffer in
 * ncclMemAlloc memory registered as an NCCL symmetric window
 * (NCCL_WIN_COLL_SYMMETRIC) when the library supports it (*symmetric = 1).
 * BWW dG buffers placed here are reduced by NCCL's symmetric kernels. */
spc_status spc_comm_window_alloc(spc_comm* comm, size_t bytes, void** ptr, int* symmetric);
spc_status spc_comm_window_free(spc_comm* comm, void* ptr);
/* In-place fp32 sum of n floats across the ranks of `nccl_comm` (an ncclComm_t). */
spc_status spc_bww_allreduce(void* nccl_comm, float* dG, size_t n, void* stream);
/* spc_sparse_bww over this rank's shard (shard_shape->N = local images), then
 * the dG allreduce and a u64 sum of d_counters, all on `stream`. */
spc_status spc_bww_sharded(spc_comm* comm, const spc_tensor* input, const spc_tensor* grad_out,
                           const spc_shape* shard_shape, const spc_plan* plan, int mode, spc_tensor* dst,
                           spc_counters* d_counters, void* stream);

/* ---- introspection ---- */
const char* spc_last_error(void);
const char* spc_backend_name(void);
int spc_native_backend_available(int V);
int spc_abi_version(void);
/* Count of device kernels this library has launched in this process. */
uint64_t spc_launch_count(void);

/* ---- measurement support (not part of the reference interface) ---- */
/* FP32 FFMA-pipe peak probe: launches `blocks` CTAs of 256 threads, each
 * thread running `iters` x 16 independent FFMAs; out[0] receives a checksum.
 * Returns the kernel's FLOP count in *flops (time it with events). */
spc_status spc_ffma_peak_kernel(float* out, int blocks, int iters, double* flops, void* stream);
/* Write `n` floats of scratch (an L2 flush between timed steps). */
spc_status spc_l2_flush(float* scratch, size_t n, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPCONV_B200_H */
