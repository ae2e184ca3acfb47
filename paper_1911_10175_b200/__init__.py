"""B200-native sparse direct convolution (SparseTrain, arXiv 1911.10175).

FWD / BWI / BWW passes over dense blocked fp32 tensors that skip the work fed
by ReLU zeros, as hand-written sm_100a CUDA kernels behind a C ABI
(``include/spconv_b200.h``).  :mod:`.api` mirrors the reference's C++ layer API
(``spconv::sparse_fwd`` etc.); :mod:`.workloads` holds the BASELINE configs and
their seeded synthetic inputs; :mod:`.dist` the batch-sharded multi-GPU path; :mod:`.sweep` the reference
harness's timed sweeps and CSVs; :mod:`.chain` layer chains (ResNet-50 /
Fixup) with fused ReLU epilogues.
"""
from .api import (BackendPref, BlockedTensor, BwwCheck, Component, ConvResult, ConvShape, Epilogue,  # noqa: F401
                  HostBatch, KernelCounters, KernelPlan, Math, get_math, math_mode, set_math, epilogue_apply, Layout, PreparedPass, RunMode, SpconvError, analytic_counters, backend_name,
                  backend_names, launch_count, native_backend_available, nchwc_to_chwnn, output_shape,
                  VecProbe, vector_probes,
                  pack_act_chwnn, pack_act_nchwc, pack_filter, plan, relu_, relu_grad_mask, run_parallel,
                  sparse_bwi, sparse_bww, sparse_fwd, unpack)

__all__ = [n for n in dir() if not n.startswith("_")]
