"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.

Two CPU implementations of the reference's sparse direct-conv path:

* ``liboracle.so``  -- this repo's plain-C restatement (``spconv_oracle.c``),
  each function citing the reference file:line it follows;
* ``_ref/libspconv_ref.so`` -- the unmodified reference library compiled from
  its own sources (``oracle/Makefile``) behind ``ref_shim.cpp``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
and ``--impl reference`` legs may import this package.

Shapes are 11-tuples in ``conv_shape`` field order
``(N, C, K, H, W, R, S, O, P, padW, padH)`` (P/include/spconv/tensor.hpp:30-38).
Components: 0 = fwd, 1 = bwi, 2 = bww; bww check: 0 = input, 1 = output_grad.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libspconv_ref.so")
REF_SRC = os.environ.get("SPCONV_REF", "/root/reference/proj")

FWD, BWI, BWW = 0, 1, 2
CHECK_INPUT, CHECK_OUTPUT_GRAD = 0, 1

_f32p = C.POINTER(C.c_float)
_u64p = C.POINTER(C.c_uint64)
_i32p = C.POINTER(C.c_int)


class _Shape(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "C", "K", "H", "W", "R", "S", "O", "P", "padW", "padH")]


class _Plan(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("comp", "check", "V", "Q", "T", "pipelined", "ring_size", "M",
                                        "register_budget", "unroll_hint", "prefetch_hints")]


def build(with_ref: bool | None = None) -> None:
    """Compile the C restatement (and the reference when its sources exist)."""
    targets = ["all"]
    if with_ref is None:
        with_ref = os.path.isdir(os.path.join(REF_SRC, "src"))
    if with_ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE, f"-j{os.cpu_count() or 4}", *targets,
                    f"SPCONV_REF={REF_SRC}"], check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build(with_ref=False)
        L = C.CDLL(LIB_PATH)
        L.orc_dense.argtypes = [C.c_int, C.POINTER(_Shape), _f32p, _f32p, _f32p, C.c_int]
        L.orc_expected_counts.argtypes = [C.POINTER(_Shape), C.POINTER(_Plan), _f32p, _u64p]
        L.orc_plan_make.argtypes = [C.POINTER(_Shape), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(_Plan)]
        L.orc_shape_make.argtypes = [C.c_int] * 9 + [C.POINTER(_Shape)]
        L.orc_shape_validate.argtypes = [C.POINTER(_Shape)]
        L.orc_decompose.argtypes = [C.POINTER(_Shape), C.POINTER(_Plan), _i32p]
        L.orc_gen_sparse.argtypes = [_f32p, C.c_size_t, C.c_double, C.c_uint64]
        L.orc_gen_gaussian_relu.argtypes = [_f32p, C.c_size_t, C.c_uint64]
        L.orc_mt64_stream.argtypes = [C.c_uint64, _u64p, C.c_size_t]
        L.orc_relu.argtypes = [_f32p, _f32p, C.c_size_t]
        L.orc_relu_grad_mask.argtypes = [_f32p, _f32p, _f32p, C.c_size_t]
        L.orc_cmp_neq_zero.argtypes = [_f32p, C.c_int]
        L.orc_cmp_neq_zero.restype = C.c_uint32
        L.orc_affected_outputs.argtypes = [C.POINTER(_Shape), C.c_int, _i32p, _i32p]
        L.orc_bwi_affected_outputs.argtypes = [C.POINTER(_Shape), C.c_int, _i32p, _i32p]
        L.orc_pack_act.argtypes = [_f32p, _f32p] + [C.c_int] * 6
        L.orc_unpack_act.argtypes = [_f32p, _f32p] + [C.c_int] * 6
        L.orc_pack_filter.argtypes = [_f32p, _f32p] + [C.c_int] * 6
        L.orc_unpack_filter.argtypes = [_f32p, _f32p] + [C.c_int] * 5
        L.orc_dot.argtypes = [_f32p, _f32p, C.c_size_t]
        L.orc_dot.restype = C.c_double
        L.orc_max_rel_error.argtypes = [_f32p, _f32p, C.c_size_t]
        L.orc_max_rel_error.restype = C.c_double
        L.orc_max_abs_rel.argtypes = [_f32p, _f32p, C.c_size_t]
        L.orc_max_abs_rel.restype = C.c_double
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The compiled reference library, or None when it was never built."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            return None
        L = C.CDLL(REF_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_plan.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.c_int, _i32p]
        L.ref_shape_make.argtypes = [C.c_int] * 9 + [_i32p]
        L.ref_gen_sparse.argtypes = [C.c_int] * 4 + [C.c_double, C.c_uint64, _f32p]
        L.ref_gen_gaussian_relu.argtypes = [C.c_int] * 4 + [C.c_uint64, _f32p]
        L.ref_mt64_stream.argtypes = [C.c_uint64, _u64p, C.c_size_t]
        L.ref_dense.argtypes = [C.c_int, _i32p, _f32p, _f32p, _f32p]
        L.ref_expected_counts.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, _f32p, _u64p]
        L.ref_prepare.argtypes = [C.c_int, C.c_int, _i32p, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_prepare.restype = C.c_void_p
        L.ref_exec.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.ref_result.argtypes = [C.c_void_p, _f32p, _u64p, C.c_char_p, C.c_int]
        L.ref_operand.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.ref_operand.restype = C.c_size_t
        L.ref_blocked_output.argtypes = [C.c_void_p, _f32p]
        L.ref_blocked_output.restype = C.c_size_t
        L.ref_free.argtypes = [C.c_void_p]
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_find_layer.argtypes = [C.c_char_p, _i32p]
        L.ref_registry_name.argtypes = [C.c_int, C.c_char_p, C.c_size_t]
        L.ref_scaled_shape.argtypes = [_i32p, C.c_int, C.c_int, _i32p]
        L.ref_run_sweep.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int,
                                    C.c_uint64, C.c_int, C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]
        L.ref_format_csv.argtypes = [C.c_int, C.c_char_p, _i32p, C.POINTER(C.c_double), _i32p, _i32p,
                                     C.POINTER(C.c_double), _u64p, C.POINTER(C.c_double),
                                     C.c_char_p, C.c_size_t, C.c_char_p, C.c_size_t]
        L.ref_load_curves.argtypes = [C.c_char_p]
        _ref = L
    return _ref


# ---------------------------------------------------------------- helpers
def _fp(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_f32p)


def _shape(sh) -> _Shape:
    return _Shape(*[int(v) for v in sh])


def out_hw(sh):
    N, Cc, K, H, W, R, S, O, P, pw, ph = sh
    return (H + 2 * ph - S) // P + 1, (W + 2 * pw - R) // O + 1


def shape_make(N, Cc, K, H, W, R, S, O=1, P=1):
    """conv_shape::make (P/src/tensor.cpp:11-14); raises ValueError when invalid."""
    s = _Shape()
    if lib().orc_shape_make(N, Cc, K, H, W, R, S, O, P, C.byref(s)):
        raise ValueError("invalid conv_shape")
    return tuple(getattr(s, f) for f, _ in _Shape._fields_)


def shape_valid(sh) -> bool:
    return lib().orc_shape_validate(C.byref(_shape(sh))) == 0


def plan(sh, comp, V, budget=30, check=0) -> dict:
    p = _Plan()
    rc = lib().orc_plan_make(C.byref(_shape(sh)), comp, V, budget, check, C.byref(p))
    if rc:
        raise ValueError(f"plan failed ({rc})")
    return {f: getattr(p, f) for f, _ in _Plan._fields_}


def decompose(sh, pl) -> tuple:
    out = (C.c_int * 3)()
    lib().orc_decompose(C.byref(_shape(sh)), C.byref(_Plan(**pl)), out)
    return tuple(out)


def dense(comp, sh, a, b, threads=None) -> np.ndarray:
    """64-bit dense oracle (P/src/oracle.cpp:39-148) on plain tensors."""
    N, Cc, K, H, W, R, S = sh[:7]
    hp, wp = out_hw(sh)
    shape = {FWD: (N, K, hp, wp), BWI: (N, Cc, H, W), BWW: (K, Cc, S, R)}[comp]
    out = np.empty(shape, np.float32)
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    if threads is None:
        threads = os.cpu_count() or 1
    if lib().orc_dense(comp, C.byref(_shape(sh)), _fp(a), _fp(b), _fp(out), int(threads)):
        raise ValueError("dense: invalid shape")
    return out


def expected_counts(sh, pl, mask) -> dict:
    """expected_fma_counts (P/src/oracle.cpp:150-284)."""
    rep = (C.c_uint64 * 4)()
    mask = np.ascontiguousarray(mask, np.float32)
    lib().orc_expected_counts(C.byref(_shape(sh)), C.byref(_Plan(**pl)), _fp(mask), rep)
    return {"checked_vectors": rep[0], "nonzero_elements": rep[1],
            "executed_vector_fmas": rep[2], "skipped_vector_fmas": rep[3],
            "dense_total": rep[2] + rep[3]}


def gen_sparse(n, c, h, w, s, seed) -> np.ndarray:
    out = np.empty((n, c, h, w), np.float32)
    lib().orc_gen_sparse(_fp(out), out.size, float(s), int(seed))
    return out


def gen_gaussian_relu(n, c, h, w, seed) -> np.ndarray:
    out = np.empty((n, c, h, w), np.float32)
    lib().orc_gen_gaussian_relu(_fp(out), out.size, int(seed))
    return out


def mt64_stream(seed, n) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().orc_mt64_stream(int(seed), out.ctypes.data_as(_u64p), n)
    return out


def relu(x):
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(x)
    lib().orc_relu(_fp(x), _fp(out), x.size)
    return out


def relu_grad_mask(pre, up):
    pre = np.ascontiguousarray(pre, np.float32)
    up = np.ascontiguousarray(up, np.float32)
    out = np.empty_like(up)
    lib().orc_relu_grad_mask(_fp(pre), _fp(up), _fp(out), up.size)
    return out


def cmp_neq_zero(v) -> int:
    v = np.ascontiguousarray(v, np.float32)
    return int(lib().orc_cmp_neq_zero(_fp(v), v.size))


def affected_outputs(sh, x, bwi=False):
    u = (C.c_int * 64)()
    col = (C.c_int * 64)()
    f = lib().orc_bwi_affected_outputs if bwi else lib().orc_affected_outputs
    n = f(C.byref(_shape(sh)), x, u, col)
    return [(u[i], col[i]) for i in range(n)]


def pack_act(plain, V, chwnn=False) -> np.ndarray:
    plain = np.ascontiguousarray(plain, np.float32)
    n, c, h, w = plain.shape
    size = ((n + V - 1) // V) * c * h * w * V if chwnn else plain.size
    out = np.zeros(size, np.float32)
    lib().orc_pack_act(_fp(plain), _fp(out), n, c, h, w, V, int(chwnn))
    return out


def unpack_act(blk, n, c, h, w, V, chwnn=False) -> np.ndarray:
    blk = np.ascontiguousarray(blk, np.float32).ravel()
    out = np.empty((n, c, h, w), np.float32)
    lib().orc_unpack_act(_fp(blk), _fp(out), n, c, h, w, V, int(chwnn))
    return out


def pack_filter(g, V, swap_kc=False) -> np.ndarray:
    g = np.ascontiguousarray(g, np.float32)
    gn, gc, gs, gr = g.shape
    out = np.zeros(g.size, np.float32)
    lib().orc_pack_filter(_fp(g), _fp(out), gn, gc, gs, gr, V, int(swap_kc))
    return out


def unpack_filter(blk, k, c, s, r, V) -> np.ndarray:
    blk = np.ascontiguousarray(blk, np.float32).ravel()
    out = np.empty((k, c, s, r), np.float32)
    lib().orc_unpack_filter(_fp(blk), _fp(out), k, c, s, r, V)
    return out


def dot(a, b) -> float:
    a = np.ascontiguousarray(a, np.float32).ravel()
    b = np.ascontiguousarray(b, np.float32).ravel()
    return lib().orc_dot(_fp(a), _fp(b), a.size)


def max_rel_error(a, refv) -> float:
    """The reference's elementwise metric (P/src/oracle.cpp:417-425)."""
    a = np.ascontiguousarray(a, np.float32).ravel()
    refv = np.ascontiguousarray(refv, np.float32).ravel()
    return lib().orc_max_rel_error(_fp(a), _fp(refv), a.size)


def max_abs_rel(a, refv) -> float:
    """North-star parity metric: max|a-ref| / max|ref|."""
    a = np.ascontiguousarray(a, np.float32).ravel()
    refv = np.ascontiguousarray(refv, np.float32).ravel()
    return lib().orc_max_abs_rel(_fp(a), _fp(refv), a.size)


# ------------------------------------------------ the compiled reference
class RefRun:
    """One prepared reference call: packed operands + plan (ref_prepare),
    timed run_parallel (exec), and its result."""

    def __init__(self, comp, check, sh, V, a_plain, b_plain, budget=30):
        L = ref()
        if L is None:
            raise RuntimeError("reference library not built (oracle/_ref)")
        self.L, self.comp, self.sh = L, comp, tuple(sh)
        self._a = np.ascontiguousarray(a_plain, np.float32)
        self._b = np.ascontiguousarray(b_plain, np.float32)
        self._shape = (C.c_int * 11)(*self.sh)
        self.h = L.ref_prepare(comp, check, self._shape, V, budget, _fp(self._a), _fp(self._b))
        if not self.h:
            raise ValueError(L.ref_last_error().decode())

    def exec(self, mode=0, workers=1, pref=0):
        if self.L.ref_exec(self.h, mode, workers, pref):
            raise ValueError(self.L.ref_last_error().decode())

    def operand(self, which) -> np.ndarray:
        n = self.L.ref_operand(self.h, which, None)
        out = np.empty(n, np.float32)
        self.L.ref_operand(self.h, which, _fp(out))
        return out

    def blocked_output(self) -> np.ndarray:
        n = self.L.ref_blocked_output(self.h, None)
        out = np.empty(n, np.float32)
        self.L.ref_blocked_output(self.h, _fp(out))
        return out

    def result(self):
        N, Cc, K, H, W, R, S = self.sh[:7]
        hp, wp = out_hw(self.sh)
        shape = {FWD: (N, K, hp, wp), BWI: (N, Cc, H, W), BWW: (K, Cc, S, R)}[self.comp]
        out = np.empty(shape, np.float32)
        cnt = (C.c_uint64 * 4)()
        name = C.create_string_buffer(64)
        self.L.ref_result(self.h, _fp(out), cnt, name, 64)
        counters = {"checked_vectors": cnt[0], "executed_vector_fmas": cnt[1],
                    "output_vector_loads": cnt[2], "output_vector_stores": cnt[3]}
        return out, counters, name.value.decode()

    def close(self):
        if self.h:
            self.L.ref_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_dense(comp, sh, a, b) -> np.ndarray:
    N, Cc, K, H, W, R, S = sh[:7]
    hp, wp = out_hw(sh)
    shape = {FWD: (N, K, hp, wp), BWI: (N, Cc, H, W), BWW: (K, Cc, S, R)}[comp]
    out = np.empty(shape, np.float32)
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    if ref().ref_dense(comp, (C.c_int * 11)(*sh), _fp(a), _fp(b), _fp(out)):
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_plan(sh, comp, V, budget=30, check=0) -> dict:
    out = (C.c_int * 6)()
    if ref().ref_plan((C.c_int * 11)(*sh), comp, V, budget, check, out):
        raise ValueError(ref().ref_last_error().decode())
    return dict(zip(("Q", "T", "pipelined", "ring_size", "M", "unroll_hint"), list(out)))


def ref_expected_counts(comp, check, sh, V, mask) -> dict:
    rep = (C.c_uint64 * 4)()
    mask = np.ascontiguousarray(mask, np.float32)
    if ref().ref_expected_counts(comp, check, (C.c_int * 11)(*sh), V, _fp(mask), rep):
        raise ValueError(ref().ref_last_error().decode())
    return {"checked_vectors": rep[0], "nonzero_elements": rep[1],
            "executed_vector_fmas": rep[2], "skipped_vector_fmas": rep[3]}


def ref_gen_sparse(n, c, h, w, s, seed) -> np.ndarray:
    out = np.empty((n, c, h, w), np.float32)
    ref().ref_gen_sparse(n, c, h, w, float(s), int(seed), _fp(out))
    return out


def ref_mt64_stream(seed, n) -> np.ndarray:
    out = np.empty(n, np.uint64)
    ref().ref_mt64_stream(int(seed), out.ctypes.data_as(_u64p), n)
    return out


def ref_shape_make(N, Cc, K, H, W, R, S, O=1, P=1):
    out = (C.c_int * 11)()
    if ref().ref_shape_make(N, Cc, K, H, W, R, S, O, P, out):
        raise ValueError(ref().ref_last_error().decode())
    return tuple(out)


# ---------------------------------------------------------------- harness (bench.cpp / projector.cpp)
def ref_registry() -> dict:
    """name -> 11-int shape of the reference's layer registry (bench.cpp:21-52)."""
    L = ref()
    out = {}
    for i in range(L.ref_registry_size()):
        buf = C.create_string_buffer(64)
        L.ref_registry_name(i, buf, 64)
        sh = (C.c_int * 11)()
        L.ref_find_layer(buf.value, sh)
        out[buf.value.decode()] = tuple(sh)
    return out


def ref_scaled_shape(base, minibatch, scale):
    out = (C.c_int * 11)()
    if ref().ref_scaled_shape((C.c_int * 11)(*base), minibatch, scale, out):
        raise ValueError(ref().ref_last_error().decode())
    return tuple(out)


def ref_run_sweep(layers, comps, grid, minibatch, scale, seed, repeats=1):
    """The reference's run_sweep -> (sweep CSV, curves CSV) strings."""
    mask = sum(1 << int(c) for c in comps)
    g = (C.c_double * len(grid))(*grid)
    a, b = C.create_string_buffer(1 << 20), C.create_string_buffer(1 << 20)
    if ref().ref_run_sweep("\n".join(layers).encode(), mask, g, len(grid), minibatch, scale, int(seed), repeats,
                           a, 1 << 20, b, 1 << 20):
        raise ValueError(ref().ref_last_error().decode())
    return a.value.decode(), b.value.decode()


def ref_format_csv(records):
    """write_sweep_csv / write_curves_csv of the given records (objects with
    layer, comp, sparsity, mode, workers, median_ns, exec_fmas, speedup_vs_dense)."""
    n = len(records)
    comps = (C.c_int * n)(*[int(r.comp) for r in records])
    sp = (C.c_double * n)(*[float(r.sparsity) for r in records])
    modes = (C.c_int * n)(*[int(r.mode) for r in records])
    wk = (C.c_int * n)(*[int(r.workers) for r in records])
    ns = (C.c_double * n)(*[float(r.median_ns) for r in records])
    fm = (C.c_uint64 * n)(*[int(r.exec_fmas) for r in records])
    su = (C.c_double * n)(*[float(r.speedup_vs_dense) for r in records])
    a, b = C.create_string_buffer(1 << 20), C.create_string_buffer(1 << 20)
    if ref().ref_format_csv(n, "\n".join(r.layer for r in records).encode(), comps, sp, modes, wk, ns, fm, su,
                            a, 1 << 20, b, 1 << 20):
        raise ValueError(ref().ref_last_error().decode())
    return a.value.decode(), b.value.decode()


def ref_load_curves(path) -> int:
    n = ref().ref_load_curves(str(path).encode())
    if n < 0:
        raise ValueError(ref().ref_last_error().decode())
    return n
