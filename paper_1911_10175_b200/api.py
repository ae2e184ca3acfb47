"""Python mirror of the reference's public C++ interface for the hot path.

Same names, argument meaning and error behaviour as ``spconv`` (reference
headers P/include/spconv/{tensor,planner,kernels}.hpp), executed by the
sm_100a CUDA library through its C ABI (include/spconv_b200.h):

=========================  ==========================================  =======================
this module                 reference                                   C ABI
=========================  ==========================================  =======================
``ConvShape.make``          ``conv_shape::make``  tensor.hpp:39          ``spc_shape_make``
``plan``                    ``spconv::plan``      planner.hpp:44         ``spc_plan_make``
``pack_act_nchwc`` etc.     ``pack_*`` / ``unpack`` tensor.hpp:124-130   (host numpy / torch)
``sparse_fwd``              ``sparse_fwd``        kernels.hpp:58         ``spc_sparse_fwd``
``sparse_bwi``              ``sparse_bwi``        kernels.hpp:65         ``spc_sparse_bwi``
``sparse_bww``              ``sparse_bww``        kernels.hpp:74         ``spc_sparse_bww``
``run_parallel``            ``run_parallel``      kernels.hpp:83         ``spc_run_parallel``
=========================  ==========================================  =======================

Blocked tensors carry either a host ``numpy`` array (the call then copies in,
runs and copies out: ``spc_run_parallel_host``) or a CUDA ``torch`` tensor
(device-resident; the call is enqueued on the current torch stream).
Contract violations raise :class:`SpconvError` (the analogue of
``spconv::error``, common.hpp:11) before any device work.
"""
from __future__ import annotations

import ctypes as C
import contextlib
import dataclasses
import enum
from typing import Any

import numpy as np

from . import _lib
from ._lib import spc_counters, spc_plan, spc_shape, spc_tensor


class SpconvError(RuntimeError):
    """Raised on a nonzero spc_status (mirror of spconv::error)."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Component(enum.IntEnum):
    fwd = 0
    bwi = 1
    bww = 2


class BwwCheck(enum.IntEnum):
    input = 0
    output_grad = 1


class RunMode(enum.IntEnum):
    sparse = 0
    dense = 1


class BackendPref(enum.IntEnum):
    automatic = 0
    force_scalar = 1
    force_native = 2


class Layout(enum.IntEnum):
    plain = 0
    act_nchwc = 1
    filter_kcrs_blk = 2
    act_chwnn = 3


LAYOUT_NAMES = {Layout.plain: "Plain", Layout.act_nchwc: "ActNCHWc", Layout.filter_kcrs_blk: "FilterKCRSblk",
                Layout.act_chwnn: "ActCHWNn"}


def _check(status: int) -> None:
    if status:
        raise SpconvError(status, _lib.last_error())


# ------------------------------------------------------------------ shape
@dataclasses.dataclass(frozen=True)
class ConvShape:
    """conv_shape (P/include/spconv/tensor.hpp:30-48)."""
    N: int
    C: int
    K: int
    H: int
    W: int
    R: int
    S: int
    O: int = 1
    P: int = 1
    padW: int = 0
    padH: int = 0

    @classmethod
    def make(cls, N, C_, K, H, W, R, S, O=1, P=1) -> "ConvShape":
        s = spc_shape()
        _check(_lib.load().spc_shape_make(N, C_, K, H, W, R, S, O, P, C.byref(s)))
        return cls._from_c(s)

    @classmethod
    def make_padded(cls, N, C_, K, H, W, R, S, O, P, padW, padH) -> "ConvShape":
        s = spc_shape()
        _check(_lib.load().spc_shape_make_padded(N, C_, K, H, W, R, S, O, P, padW, padH, C.byref(s)))
        return cls._from_c(s)

    @classmethod
    def _from_c(cls, s: spc_shape) -> "ConvShape":
        return cls(*[getattr(s, f) for f, _ in spc_shape._fields_])

    def to_c(self) -> spc_shape:
        return spc_shape(*dataclasses.astuple(self))

    def out_w(self) -> int:
        return (self.W + 2 * self.padW - self.R) // self.O + 1

    def out_h(self) -> int:
        return (self.H + 2 * self.padH - self.S) // self.P + 1

    def validate(self) -> None:
        _check(_lib.load().spc_shape_validate(C.byref(self.to_c())))

    def astuple(self) -> tuple:
        return dataclasses.astuple(self)

    def dense_flops(self) -> int:
        """Dense-equivalent FLOPs of one pass: 2*N*K*C*R*S*H'*W'."""
        return 2 * self.N * self.K * self.C * self.R * self.S * self.out_h() * self.out_w()

    def with_batch(self, n: int) -> "ConvShape":
        return dataclasses.replace(self, N=n)


def output_shape(shape: ConvShape) -> tuple[int, int]:
    """(W', H') after validation (P/include/spconv/tensor.hpp:51)."""
    shape.validate()
    return shape.out_w(), shape.out_h()


# ------------------------------------------------------------------ plan
@dataclasses.dataclass
class KernelPlan:
    """kernel_plan (P/include/spconv/planner.hpp:22-38)."""
    comp: Component = Component.fwd
    check: BwwCheck = BwwCheck.input
    V: int = 0
    Q: int = 0
    T: int = 0
    pipelined: bool = False
    ring_size: int = 0
    M: int = 1
    register_budget: int = 30
    unroll_hint: int = 0
    prefetch_hints: bool = False

    def tiled_channels(self, shape: ConvShape) -> int:
        if self.comp == Component.bwi:
            return shape.C
        if self.comp == Component.bww and self.check == BwwCheck.output_grad:
            return shape.C
        return shape.K

    def to_c(self) -> spc_plan:
        return spc_plan(int(self.comp), int(self.check), self.V, self.Q, self.T, int(bool(self.pipelined)),
                        self.ring_size, self.M, self.register_budget, self.unroll_hint,
                        int(bool(self.prefetch_hints)))

    @classmethod
    def _from_c(cls, p: spc_plan) -> "KernelPlan":
        return cls(Component(p.comp), BwwCheck(p.check), p.V, p.Q, p.T, bool(p.pipelined), p.ring_size, p.M,
                   p.register_budget, p.unroll_hint, bool(p.prefetch_hints))


def plan(shape: ConvShape, comp: Component, V: int, register_budget: int = 30,
         check: BwwCheck = BwwCheck.input) -> KernelPlan:
    """spconv::plan (P/src/planner.cpp:25-73)."""
    p = spc_plan()
    _check(_lib.load().spc_plan_make(C.byref(shape.to_c()), int(comp), V, register_budget, int(check),
                                     C.byref(p)))
    return KernelPlan._from_c(p)


# ------------------------------------------------------------------ tensors
@dataclasses.dataclass
class BlockedTensor:
    """blocked_tensor (P/include/spconv/tensor.hpp:80-120).  ``data`` is a
    1-D float32 numpy array (host) or torch tensor (CUDA, device-resident)."""
    layout: Layout = Layout.act_nchwc
    V: int = 0
    n: int = 0
    c: int = 0
    h: int = 0
    w: int = 0
    k: int = 0
    r: int = 0
    s: int = 0
    data: Any = None

    def c_blocks(self) -> int:
        return self.c // self.V

    def k_blocks(self) -> int:
        return self.k // self.V

    def n_blocks(self) -> int:
        return (self.n + self.V - 1) // self.V

    def act_index(self, i, ch, y, x) -> int:
        return (((i * self.c_blocks() + ch // self.V) * self.h + y) * self.w + x) * self.V + ch % self.V

    def chwnn_index(self, i, ch, y, x) -> int:
        return (((i // self.V * self.c + ch) * self.h + y) * self.w + x) * self.V + i % self.V

    def filter_index(self, kk, cc, u, v) -> int:
        return ((((kk // self.V * self.c_blocks() + cc // self.V) * self.s + v) * self.r + u) * self.V
                + cc % self.V) * self.V + kk % self.V

    @property
    def on_device(self) -> bool:
        return _is_torch_cuda(self.data)

    def numel(self) -> int:
        return int(self.data.numel() if _is_torch(self.data) else self.data.size)

    def to_c(self) -> spc_tensor:
        return spc_tensor(int(self.layout), self.V, self.n, self.c, self.h, self.w, self.k, self.r, self.s,
                          _data_ptr(self.data), self.numel())

    def header(self) -> dict:
        return {f.name: getattr(self, f.name) for f in dataclasses.fields(self) if f.name != "data"}

    def to(self, device) -> "BlockedTensor":
        """Copy to a torch device ('cuda') or to host numpy (device=None/'cpu')."""
        import torch
        if device in (None, "cpu", "numpy"):
            d = self.data.detach().cpu().numpy() if _is_torch(self.data) else self.data
        else:
            d = torch.as_tensor(np.ascontiguousarray(self.data)) if not _is_torch(self.data) else self.data
            d = d.to(device)
        return dataclasses.replace(self, data=d)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def _is_torch_cuda(x) -> bool:
    return _is_torch(x) and x.is_cuda


def _data_ptr(x) -> int | None:
    if x is None:
        return None
    if _is_torch(x):
        assert x.is_contiguous() and str(x.dtype) == "torch.float32", "blocked data must be contiguous float32"
        return x.data_ptr()
    assert isinstance(x, np.ndarray) and x.dtype == np.float32 and x.flags["C_CONTIGUOUS"], \
        "blocked data must be a contiguous float32 array"
    return x.ctypes.data


def _xp(x):
    if _is_torch(x):
        import torch
        return torch
    return np


def _perm(xp, a, axes):
    return a.permute(*axes) if xp is not np else a.transpose(axes)


def _contig(xp, a):
    return a.contiguous().reshape(-1) if xp is not np else np.ascontiguousarray(a).reshape(-1)


def pack_act_nchwc(t, V: int) -> BlockedTensor:
    """pack_act_nchwc (P/src/tensor.cpp:78-92): plain (n,c,h,w) -> [n][c/V][h][w][V]."""
    if V not in (4, 8, 16):
        raise SpconvError(_lib.SPC_ERR_LAYOUT, "pack: V must be 4, 8 or 16")
    n, c, h, w = t.shape
    if c % V:
        raise SpconvError(_lib.SPC_ERR_LAYOUT, "pack_act_nchwc: channels not divisible by V")
    xp = _xp(t)
    b = _perm(xp, t.reshape(n, c // V, V, h, w), (0, 1, 3, 4, 2))
    return BlockedTensor(Layout.act_nchwc, V, n, c, h, w, data=_contig(xp, b))


def pack_act_chwnn(t, V: int) -> BlockedTensor:
    """pack_act_chwnn (P/src/tensor.cpp:94-108): [ceil(n/V)][c][h][w][V], ragged lanes zero."""
    if V not in (4, 8, 16):
        raise SpconvError(_lib.SPC_ERR_LAYOUT, "pack: V must be 4, 8 or 16")
    n, c, h, w = t.shape
    nb = (n + V - 1) // V
    xp = _xp(t)
    if xp is np:
        full = np.zeros((nb * V, c, h, w), np.float32)
    else:
        full = xp.zeros((nb * V, c, h, w), dtype=t.dtype, device=t.device)
    full[:n] = t
    b = _perm(xp, full.reshape(nb, V, c, h, w), (0, 2, 3, 4, 1))
    return BlockedTensor(Layout.act_chwnn, V, n, c, h, w, data=_contig(xp, b))


def pack_filter(g, V: int, swap_kc: bool = False) -> BlockedTensor:
    """pack_filter (P/src/tensor.cpp:110-130): plain (K,C,S,R) -> [K/V][C/V][S][R][Vc][Vk];
    swap_kc packs the transpose BWI wants (k' = c, c' = k)."""
    if V not in (4, 8, 16):
        raise SpconvError(_lib.SPC_ERR_LAYOUT, "pack: V must be 4, 8 or 16")
    xp = _xp(g)
    if swap_kc:
        g = _perm(xp, g, (1, 0, 2, 3))
    K, Cc, S, R = g.shape
    if K % V or Cc % V:
        raise SpconvError(_lib.SPC_ERR_LAYOUT, "pack_filter: K and C must be divisible by V")
    b = _perm(xp, g.reshape(K // V, V, Cc // V, V, S, R), (0, 2, 4, 5, 3, 1))
    return BlockedTensor(Layout.filter_kcrs_blk, V, k=K, c=Cc, s=S, r=R, data=_contig(xp, b))


def unpack(b: BlockedTensor):
    """unpack (P/src/tensor.cpp:132-165) -> plain array of the data's kind."""
    xp = _xp(b.data)
    V = b.V
    if b.layout == Layout.act_nchwc:
        t = _perm(xp, b.data.reshape(b.n, b.c // V, b.h, b.w, V), (0, 1, 4, 2, 3))
        return t.reshape(b.n, b.c, b.h, b.w) if xp is not np else np.ascontiguousarray(t).reshape(b.n, b.c, b.h, b.w)
    if b.layout == Layout.act_chwnn:
        nb = b.n_blocks()
        t = _perm(xp, b.data.reshape(nb, b.c, b.h, b.w, V), (0, 4, 1, 2, 3)).reshape(nb * V, b.c, b.h, b.w)
        t = t[: b.n]
        return t.contiguous() if xp is not np else np.ascontiguousarray(t)
    if b.layout == Layout.filter_kcrs_blk:
        t = _perm(xp, b.data.reshape(b.k // V, b.c // V, b.s, b.r, V, V), (0, 5, 1, 4, 2, 3))
        t = t.reshape(b.k, b.c, b.s, b.r)
        return t.contiguous() if xp is not np else np.ascontiguousarray(t)
    raise SpconvError(_lib.SPC_ERR_LAYOUT, "unpack: unsupported layout")


# ------------------------------------------------------------------ passes
@dataclasses.dataclass
class KernelCounters:
    """kernel_counters (P/include/spconv/kernels.hpp:31-45)."""
    checked_vectors: int = 0
    executed_vector_fmas: int = 0
    output_vector_loads: int = 0
    output_vector_stores: int = 0

    @classmethod
    def _from_c(cls, c: spc_counters) -> "KernelCounters":
        return cls(int(c.checked_vectors), int(c.executed_vector_fmas), int(c.output_vector_loads),
                   int(c.output_vector_stores))

    def __iadd__(self, o: "KernelCounters") -> "KernelCounters":
        for f in dataclasses.fields(self):
            setattr(self, f.name, getattr(self, f.name) + getattr(o, f.name))
        return self


@dataclasses.dataclass
class ConvResult:
    """conv_result (P/include/spconv/kernels.hpp:47-51)."""
    out: BlockedTensor
    counters: KernelCounters
    backend: str


def output_desc(shape: ConvShape, pl: KernelPlan) -> BlockedTensor:
    t = spc_tensor()
    _check(_lib.load().spc_output_desc(C.byref(shape.to_c()), C.byref(pl.to_c()), C.byref(t)))
    return BlockedTensor(Layout(t.layout), t.V, t.n, t.c, t.h, t.w, t.k, t.r, t.s, None), int(t.numel)


def analytic_counters(shape: ConvShape, pl: KernelPlan, mode: RunMode) -> KernelCounters:
    c = spc_counters()
    _check(_lib.load().spc_analytic_counters(C.byref(shape.to_c()), C.byref(pl.to_c()), int(mode), C.byref(c)))
    return KernelCounters._from_c(c)


def backend_name() -> str:
    return _lib.load().spc_backend_name().decode()


def native_backend_available(V: int) -> bool:
    return bool(_lib.load().spc_native_backend_available(V))


def backend_names() -> list[str]:
    return [backend_name()]


@dataclasses.dataclass
class VecProbe:
    """vec_probe (P/include/spconv/kernels.hpp:90-97): this backend's contract
    operations, executed on the device as the kernels execute them."""
    name: str
    width: int
    native: bool

    def cmp_neq_zero(self, v) -> int:
        a = np.ascontiguousarray(v, np.float32)
        m = C.c_uint32()
        _check(_lib.load().spc_vector_probe(self.width, 0, a.ctypes.data, None, 0.0, None, C.byref(m)))
        return int(m.value)

    def broadcast_fma(self, acc, s: float, w):
        a, b = np.ascontiguousarray(acc, np.float32), np.ascontiguousarray(w, np.float32)
        out = np.empty(self.width, np.float32)
        _check(_lib.load().spc_vector_probe(self.width, 1, a.ctypes.data, b.ctypes.data, float(s), out.ctypes.data,
                                            None))
        return out

    def add(self, a, b):
        a, b = np.ascontiguousarray(a, np.float32), np.ascontiguousarray(b, np.float32)
        out = np.empty(self.width, np.float32)
        _check(_lib.load().spc_vector_probe(self.width, 2, a.ctypes.data, b.ctypes.data, 0.0, out.ctypes.data, None))
        return out


def vector_probes(V: int) -> list[VecProbe]:
    """vector_probes(V) (P/include/spconv/kernels.hpp:98): the one device backend."""
    if V not in (4, 8, 16):
        raise SpconvError(_lib.SPC_ERR_ARG, "vector_probes: V must be 4, 8 or 16")
    return [VecProbe(backend_name(), V, True)]


def launch_count() -> int:
    return int(_lib.load().spc_launch_count())


class Math(enum.IntEnum):
    """Arithmetic of FWD/BWI (``spc_set_math``): ``fp32`` = FP32 FFMA with
    zero skipping (default, the reference's per-product rounding); ``tf32x3``
    = tcgen05 tensor cores with 3xTF32 split products (its own tolerance,
    DESIGN.md 4.7).  Per host thread."""
    fp32 = 0
    tf32x3 = 1


def set_math(m: Math) -> Math:
    prev = _lib.load().spc_set_math(int(m))
    if prev < 0:
        raise SpconvError(_lib.SPC_ERR_ARG, f"unknown math mode {m!r}")
    return Math(prev)


def get_math() -> Math:
    return Math(_lib.load().spc_get_math())


@contextlib.contextmanager
def math_mode(m: Math):
    """``with math_mode(Math.tf32x3): ...`` -- restores the previous mode."""
    prev = set_math(m)
    try:
        yield
    finally:
        set_math(prev)


@dataclasses.dataclass
class Epilogue:
    """Fused FWD/BWI output epilogue (include/spconv_b200.h spc_epilogue):
    v = acc*alpha (+ add) (+ beta); relu -> v > 0 ? v : 0; mask -> mask > 0 ? v : 0.
    `add` / `mask` are device tensors with the output's ActNCHWc layout;
    `beta` a scalar bias (Fixup's bias before the ReLU)."""
    alpha: float = 1.0
    add: object = None
    mask: object = None
    relu: bool = False
    beta: float = 0.0

    def to_c(self) -> "_lib.spc_epilogue":
        def ptr(t):
            if t is None:
                return None
            if isinstance(t, BlockedTensor):
                t = t.data
            if not _is_torch_cuda(t):
                raise SpconvError(_lib.SPC_ERR_ARG, "epilogue tensors must be CUDA tensors")
            return t.data_ptr()
        return _lib.spc_epilogue(float(self.alpha), ptr(self.add), ptr(self.mask), 1 if self.relu else 0,
                                 float(self.beta))


def epilogue_apply(epi: Epilogue, t) -> None:
    """The epilogue as a standalone in-place pass over a device tensor."""
    ce = epi.to_c()
    _check(_lib.load().spc_epilogue_apply(C.byref(ce), C.c_void_p(t.data_ptr()), t.numel(),
                                          C.c_void_p(_current_stream_ptr())))


def _current_stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


def _run(comp: Component, a: BlockedTensor, b: BlockedTensor, shape: ConvShape, pl: KernelPlan,
         mode: RunMode, workers: int, pref: BackendPref) -> ConvResult:
    L = _lib.load()
    if workers < 1:  # check_common (P/src/kernels.cpp:109)
        raise SpconvError(_lib.SPC_ERR_ARG, "workers must be >= 1")
    if pref == BackendPref.force_scalar:
        raise SpconvError(_lib.SPC_ERR_ARG, "no scalar backend: this library runs only on sm_100a")
    desc, numel = output_desc(shape, pl)
    ca, cb = a.to_c(), b.to_c()
    cshape, cplan = shape.to_c(), pl.to_c()
    fn = {Component.fwd: L.spc_sparse_fwd, Component.bwi: L.spc_sparse_bwi,
          Component.bww: L.spc_sparse_bww}[comp]
    if a.on_device and b.on_device:
        import torch
        dev = a.data.device
        out = torch.empty(numel, dtype=torch.float32, device=dev)
        cnt = torch.zeros(4, dtype=torch.int64, device=dev)
        cd = spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.data_ptr(), numel)
        with torch.cuda.device(dev):
            _check(fn(C.byref(ca), C.byref(cb), C.byref(cshape), C.byref(cplan), int(mode), C.byref(cd),
                      C.c_void_p(cnt.data_ptr()), C.c_void_p(_current_stream_ptr())))
        host_cnt = cnt.cpu().numpy().view(np.uint64)
        counters = KernelCounters(*[int(v) for v in host_cnt])
        desc.data = out
        return ConvResult(desc, counters, L.spc_backend_name().decode())
    if a.on_device or b.on_device:
        raise SpconvError(_lib.SPC_ERR_ARG, "operands must both be host or both be device tensors")
    out = np.empty(numel, np.float32)
    cd = spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.ctypes.data, numel)
    cnt = spc_counters()
    # validation happens inside before any device work; comp mismatches are
    # caught by the plan check exactly as the reference does
    if pl.comp != comp:
        raise SpconvError(_lib.SPC_ERR_PLAN, "plan was built for another component")
    _check(L.spc_run_parallel_host(C.byref(ca), C.byref(cb), C.byref(cshape), C.byref(cplan), int(mode),
                                   C.byref(cd), C.byref(cnt)))
    desc.data = out
    return ConvResult(desc, KernelCounters._from_c(cnt), L.spc_backend_name().decode())


def sparse_fwd(src: BlockedTensor, filt: BlockedTensor, shape: ConvShape, pl: KernelPlan,
               mode: RunMode = RunMode.sparse, workers: int = 1,
               pref: BackendPref = BackendPref.automatic) -> ConvResult:
    """FWD: src = D in ActNCHWc, filt = FilterKCRSblk; returns Y (kernels.hpp:56-61)."""
    return _run(Component.fwd, src, filt, shape, pl, mode, workers, pref)


def sparse_bwi(grad_out: BlockedTensor, filt_t: BlockedTensor, shape: ConvShape, pl: KernelPlan,
               mode: RunMode = RunMode.sparse, workers: int = 1,
               pref: BackendPref = BackendPref.automatic) -> ConvResult:
    """BWI: grad_out = dY in ActNCHWc over K, filt_t = pack_filter(swap_kc); returns dD."""
    return _run(Component.bwi, grad_out, filt_t, shape, pl, mode, workers, pref)


def sparse_bww(input: BlockedTensor, grad_out: BlockedTensor, shape: ConvShape, pl: KernelPlan,
               mode: RunMode = RunMode.sparse, workers: int = 1,
               pref: BackendPref = BackendPref.automatic) -> ConvResult:
    """BWW: the plan.check tensor must be ActCHWNn, the other ActNCHWc; returns dG (K, C)."""
    return _run(Component.bww, input, grad_out, shape, pl, mode, workers, pref)


def run_parallel(a: BlockedTensor, b: BlockedTensor, shape: ConvShape, pl: KernelPlan, mode: RunMode,
                 workers: int = 1, pref: BackendPref = BackendPref.automatic) -> ConvResult:
    """Dispatch on plan.comp (P/src/kernels.cpp:304-313)."""
    if pl.comp not in (Component.fwd, Component.bwi, Component.bww):
        raise SpconvError(_lib.SPC_ERR_PLAN, "run_parallel: bad component")
    return _run(Component(pl.comp), a, b, shape, pl, mode, workers, pref)


class HostBatch:
    """A prepared list of host-buffer passes for ``spc_run_parallel_host_batch``
    (include/spconv_b200.h): the reference's bench loop over layers and
    components (P/src/bench.cpp:216-288) as one call whose H2D copies, kernels
    and D2H copies are pipelined across passes.  ``add`` takes host (numpy)
    operands and an optional preallocated output; ``run`` executes every pass
    and returns one ConvResult per pass (counters included).  Buffers in
    pinned memory are pipelined; pageable ones go through the per-call path.
    A BWW pass may give its checked operand in ActNCHWc (the layout FWD takes):
    the library packs ActCHWNn on the device (``SPC_PASS_CHECKED_NCHWC``), and a
    buffer an earlier pass already uploaded is not uploaded again."""

    def __init__(self):
        self._keep = []
        self._items = []

    def add(self, a: BlockedTensor, b: BlockedTensor, shape: ConvShape, pl: KernelPlan,
            mode: RunMode = RunMode.sparse, out=None) -> int:
        if a.on_device or b.on_device:
            raise SpconvError(_lib.SPC_ERR_ARG, "HostBatch takes host operands")
        desc, numel = output_desc(shape, pl)
        o = out if out is not None else np.empty(numel, np.float32)
        flags = 0
        if Component(pl.comp) == Component.bww:
            checked = a if BwwCheck(pl.check) == BwwCheck.input else b
            if checked.layout == Layout.act_nchwc:
                flags = _lib.SPC_PASS_CHECKED_NCHWC
        item = dict(ca=a.to_c(), cb=b.to_c(), cs=shape.to_c(), cp=pl.to_c(), mode=int(mode),
                    cd=spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, o.ctypes.data, o.size), cnt=spc_counters(),
                    out=o, desc=desc, flags=flags)
        self._keep.append((a, b))
        self._items.append(item)
        return len(self._items) - 1

    def __len__(self):
        return len(self._items)

    @staticmethod
    def release():
        """Free the calling thread's device arena (kept between runs otherwise)."""
        _lib.load().spc_host_batch_release()

    def run(self):
        L = _lib.load()
        n = len(self._items)
        arr = (_lib.spc_host_pass * n)()
        for i, it in enumerate(self._items):
            it["cd"].data = it["out"].ctypes.data
            it["cd"].numel = it["out"].size
            arr[i].a = C.pointer(it["ca"])
            arr[i].b = C.pointer(it["cb"])
            arr[i].shape = C.pointer(it["cs"])
            arr[i].plan = C.pointer(it["cp"])
            arr[i].mode = it["mode"]
            arr[i].dst = C.pointer(it["cd"])
            arr[i].counters = C.pointer(it["cnt"])
            arr[i].status = 0
            arr[i].flags = it["flags"]
        _check(L.spc_run_parallel_host_batch(arr, n))
        res = []
        for it in self._items:
            d = dataclasses.replace(it["desc"]) if dataclasses.is_dataclass(it["desc"]) else it["desc"]
            d.data = it["out"]
            res.append(ConvResult(d, KernelCounters._from_c(it["cnt"]), L.spc_backend_name().decode()))
        return res


class PreparedPass:
    """A validated, device-resident pass with a preallocated output, for
    repeated asynchronous launches (bench / training loops).  ``launch`` does
    one C-ABI call on the given stream and no host synchronisation."""

    def __init__(self, a: BlockedTensor, b: BlockedTensor, shape: ConvShape, pl: KernelPlan,
                 mode: RunMode = RunMode.sparse, out=None, counters=None, epilogue: Epilogue | None = None):
        import torch
        L = _lib.load()
        self.L = L
        desc, numel = output_desc(shape, pl)
        dev = a.data.device
        self.out = out if out is not None else torch.empty(numel, dtype=torch.float32, device=dev)
        desc.data = self.out
        self.desc = desc
        self.counters = counters  # optional torch int64[4] device tensor
        self._a, self._b = a, b  # keep operands alive
        self._ca, self._cb = a.to_c(), b.to_c()
        self._cd = spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, self.out.data_ptr(), numel)
        self._shape, self._plan = shape.to_c(), pl.to_c()
        self.shape_obj, self.plan_obj = shape, pl
        self._mode = int(mode)
        if epilogue is not None and Component(pl.comp) == Component.bww:
            raise SpconvError(_lib.SPC_ERR_ARG, "BWW has no output epilogue")
        self._epi = epilogue.to_c() if epilogue is not None else None
        self._epi_keep = epilogue  # keep add/mask tensors alive
        if self._epi is None:
            self._fn = {Component.fwd: L.spc_sparse_fwd, Component.bwi: L.spc_sparse_bwi,
                        Component.bww: L.spc_sparse_bww}[Component(pl.comp)]
            self._args = (C.byref(self._ca), C.byref(self._cb), C.byref(self._shape), C.byref(self._plan),
                          self._mode, C.byref(self._cd))
        else:
            self._fn = {Component.fwd: L.spc_sparse_fwd_ex, Component.bwi: L.spc_sparse_bwi_ex}[Component(pl.comp)]
            self._args = (C.byref(self._ca), C.byref(self._cb), C.byref(self._shape), C.byref(self._plan),
                          self._mode, C.byref(self._epi), C.byref(self._cd))
        self._cnt_ptr = C.c_void_p(counters.data_ptr()) if counters is not None else C.c_void_p(None)

    def launch(self, stream_ptr: int) -> None:
        st = self._fn(*self._args, self._cnt_ptr, C.c_void_p(stream_ptr))
        if st:
            raise SpconvError(st, _lib.last_error())

    def read_counters(self) -> KernelCounters:
        v = self.counters.cpu().numpy().view(np.uint64)
        return KernelCounters(*[int(x) for x in v])


def relu_(x_in, x_out=None):
    """Device ReLU with the reference's semantics (P/src/sparsity.cpp:11-15)."""
    import torch
    out = x_out if x_out is not None else torch.empty_like(x_in)
    _check(_lib.load().spc_relu(C.c_void_p(x_in.data_ptr()), C.c_void_p(out.data_ptr()), x_in.numel(),
                                C.c_void_p(_current_stream_ptr())))
    return out


def relu_grad_mask(pre, upstream, out=None):
    """Device ReLU-gradient mask (P/src/sparsity.cpp:17-28)."""
    import torch
    o = out if out is not None else torch.empty_like(upstream)
    _check(_lib.load().spc_relu_grad_mask(C.c_void_p(pre.data_ptr()), C.c_void_p(upstream.data_ptr()),
                                          C.c_void_p(o.data_ptr()), upstream.numel(),
                                          C.c_void_p(_current_stream_ptr())))
    return o


def nchwc_to_chwnn(src: BlockedTensor) -> BlockedTensor:
    """Device ActNCHWc -> ActCHWNn (P/src/tensor.cpp:94-108)."""
    import torch
    V = src.V
    need = ((src.n + V - 1) // V) * src.c * src.h * src.w * V
    out = torch.empty(need, dtype=torch.float32, device=src.data.device)
    cs = src.to_c()
    cd = spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.data_ptr(), need)
    _check(_lib.load().spc_nchwc_to_chwnn(C.byref(cs), C.byref(cd), C.c_void_p(_current_stream_ptr())))
    return BlockedTensor(Layout.act_chwnn, V, src.n, src.c, src.h, src.w, data=out)
