"""Timed sparsity sweeps on the GPU with the reference harness's records and CSVs.

The reference's harness (P/src/bench.cpp, P = /root/reference/proj) times
`run_parallel` per (layer, component, sparsity) against a dense-mode
baseline, adds geo-mean summary rows, and writes two CSVs that its projector
consumes (P/src/projector.cpp:51-103).  This module is the same harness over
the sm_100a kernels, so GPU curves drop into the reference's tooling:

* `layer_registry` / `find_layer` / `scaled_shape`   bench.cpp:21-78
* `prepare` (synthetic operands, same seeds)          bench.cpp:127-180
* `run_sweep`                                          bench.cpp:215-292
* `geo_mean`, `write_sweep_csv`, `write_curves_csv`   bench.cpp:294-327
* `time_median_ns`                                     bench.cpp:80-98

Inputs come from `spc_gen_sparse`, the reference's generator stream
(sparsity.cpp:42-55), so `exec_fmas` equals the reference sweep's value on
the same request.  `median_ns` is measured on the device with CUDA events
around the C-ABI call (`timing="device"`, inputs resident in HBM), or around
the host-buffer drop-in with the reference's wall-clock method
(`timing="host"`: H2D + kernels + D2H + output allocation, like the
reference's timed `run_parallel` call).
"""
from __future__ import annotations

import argparse
import ctypes as C
import dataclasses
import math
import sys
import time

import numpy as np

from . import _lib
from .api import (BlockedTensor, BwwCheck, Component, ConvShape, PreparedPass, RunMode, SpconvError,
                  pack_act_chwnn, pack_act_nchwc, pack_filter, plan, run_parallel)

COMPONENT_NAMES = {Component.fwd: "fwd", Component.bwi: "bwi", Component.bww: "bww"}


@dataclasses.dataclass(frozen=True)
class LayerConfig:
    name: str
    shape: ConvShape  # registry batch size is 16 (bench.hpp:22-26)
    source: str


# name, source, C, K, H, W, R, S, O, P -- the 27 evaluated VGG / ResNet v1.5
# layers of the reference registry (bench.cpp:21-52), batch 16.
_REGISTRY = (
    ("vgg1_2", "vgg", 64, 64, 224, 224, 3, 3, 1, 1),
    ("vgg2_1", "vgg", 64, 128, 112, 112, 3, 3, 1, 1),
    ("vgg2_2", "vgg", 128, 128, 112, 112, 3, 3, 1, 1),
    ("vgg3_1", "vgg", 128, 256, 56, 56, 3, 3, 1, 1),
    ("vgg3_2", "vgg", 256, 256, 56, 56, 3, 3, 1, 1),
    ("vgg4_1", "vgg", 256, 512, 28, 28, 3, 3, 1, 1),
    ("vgg4_2", "vgg", 512, 512, 28, 28, 3, 3, 1, 1),
    ("vgg5_1", "vgg", 512, 512, 14, 14, 3, 3, 1, 1),
    ("resnet2_1a", "resnet", 64, 64, 56, 56, 1, 1, 1, 1),
    ("resnet2_1b", "resnet", 256, 64, 56, 56, 1, 1, 1, 1),
    ("resnet2_2", "resnet", 64, 64, 56, 56, 3, 3, 1, 1),
    ("resnet2_3", "resnet", 64, 256, 56, 56, 1, 1, 1, 1),
    ("resnet3_1a", "resnet", 256, 128, 56, 56, 1, 1, 1, 1),
    ("resnet3_1b", "resnet", 512, 128, 28, 28, 1, 1, 1, 1),
    ("resnet3_2", "resnet", 128, 128, 28, 28, 3, 3, 1, 1),
    ("resnet3_2/r", "resnet", 128, 128, 56, 56, 3, 3, 2, 2),
    ("resnet3_3", "resnet", 128, 512, 28, 28, 1, 1, 1, 1),
    ("resnet4_1a", "resnet", 512, 256, 28, 28, 1, 1, 1, 1),
    ("resnet4_1b", "resnet", 1024, 256, 14, 14, 1, 1, 1, 1),
    ("resnet4_2", "resnet", 256, 256, 14, 14, 3, 3, 1, 1),
    ("resnet4_2/r", "resnet", 256, 256, 28, 28, 3, 3, 2, 2),
    ("resnet4_3", "resnet", 256, 1024, 14, 14, 1, 1, 1, 1),
    ("resnet5_1a", "resnet", 1024, 512, 14, 14, 1, 1, 1, 1),
    ("resnet5_1b", "resnet", 2048, 512, 7, 7, 1, 1, 1, 1),
    ("resnet5_2", "resnet", 512, 512, 7, 7, 3, 3, 1, 1),
    ("resnet5_2/r", "resnet", 512, 512, 14, 14, 3, 3, 2, 2),
    ("resnet5_3", "resnet", 512, 2048, 7, 7, 1, 1, 1, 1),
)


def layer_registry() -> list[LayerConfig]:
    return [LayerConfig(n, ConvShape.make(16, c, k, h, w, r, s, o, p), src)
            for n, src, c, k, h, w, r, s, o, p in _REGISTRY]


def find_layer(name: str) -> LayerConfig | None:
    for lc in layer_registry():
        if lc.name == name:
            return lc
    return None


def scaled_shape(base: ConvShape, minibatch: int, scale: int) -> ConvShape:
    """Desk-scale variant (bench.cpp:67-78): batch override, H and W divided
    by `scale` (floored, min 1, and kept >= the filter inside the padding)."""
    if minibatch < 1 or scale < 1:
        raise SpconvError(_lib.SPC_ERR_ARG, "scaled_shape: bad minibatch or scale")
    H = max(1, base.H // scale, base.S - 2 * base.padH)
    W = max(1, base.W // scale, base.R - 2 * base.padW)
    sh = ConvShape.make_padded(minibatch, base.C, base.K, H, W, base.R, base.S, base.O, base.P,
                               base.padW, base.padH)
    sh.validate()
    return sh


def gen_sparse(n: int, c: int, h: int, w: int, sparsity: float, seed: int) -> np.ndarray:
    """The reference's gen_sparse stream (sparsity.cpp:42-55), plain [n][c][h][w]."""
    out = np.empty((n, c, h, w), np.float32)
    st = _lib.load().spc_gen_sparse(C.c_void_p(out.ctypes.data), out.size, float(sparsity), int(seed))
    if st:
        raise SpconvError(st, _lib.last_error())
    return out


@dataclasses.dataclass
class Prepared:
    plan: object
    a: BlockedTensor
    b: BlockedTensor
    check_used: BwwCheck


def prepare(sh: ConvShape, comp: Component, sparsity: float, V: int, check: BwwCheck | None,
            seed: int) -> Prepared:
    """Synthetic operands of one component (bench.cpp:127-180): the swept
    tensor at `sparsity` from `seed`, filters dense from seed+1, the
    unchecked BWW tensor dense from seed+2."""
    hp, wp = sh.out_h(), sh.out_w()
    if comp == Component.fwd:
        D = gen_sparse(sh.N, sh.C, sh.H, sh.W, sparsity, seed)
        G = gen_sparse(sh.K, sh.C, sh.S, sh.R, 0.0, seed + 1)
        return Prepared(plan(sh, comp, V), pack_act_nchwc(D, V), pack_filter(G, V), BwwCheck.input)
    if comp == Component.bwi:
        dY = gen_sparse(sh.N, sh.K, hp, wp, sparsity, seed)
        G = gen_sparse(sh.K, sh.C, sh.S, sh.R, 0.0, seed + 1)
        return Prepared(plan(sh, comp, V), pack_act_nchwc(dY, V), pack_filter(G, V, True), BwwCheck.input)
    D = gen_sparse(sh.N, sh.C, sh.H, sh.W, sparsity, seed)
    dY = gen_sparse(sh.N, sh.K, hp, wp, 0.0, seed + 2)
    if check is None:  # default: the sparser side (bench.cpp:160-166)
        use = BwwCheck.output_grad if float(np.mean(dY == 0)) > float(np.mean(D == 0)) else BwwCheck.input
    else:
        use = check
    pl = plan(sh, comp, V, 30, use)
    if use == BwwCheck.input:
        return Prepared(pl, pack_act_chwnn(D, V), pack_act_nchwc(dY, V), use)
    return Prepared(pl, pack_act_nchwc(D, V), pack_act_chwnn(dY, V), use)


def time_median_ns(fn, repeats: int, warmups: int = 2) -> float:
    """Median wall time of `repeats` calls after `warmups` (bench.cpp:80-98)."""
    if repeats < 1:
        raise SpconvError(_lib.SPC_ERR_ARG, "timing needs at least one repeat")
    for _ in range(warmups):
        fn()
    samples = []
    for _ in range(repeats):
        t0 = time.perf_counter_ns()
        fn()
        samples.append(float(time.perf_counter_ns() - t0))
    samples.sort()
    mid = repeats // 2
    return samples[mid] if repeats % 2 else 0.5 * (samples[mid - 1] + samples[mid])


def device_median_ns(pp: PreparedPass, repeats: int, warmups: int = 2) -> float:
    """Median of per-call CUDA-event durations of one resident pass."""
    import torch
    if repeats < 1:
        raise SpconvError(_lib.SPC_ERR_ARG, "timing needs at least one repeat")
    st = torch.cuda.current_stream()
    for _ in range(warmups):
        pp.launch(st.cuda_stream)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(repeats)]
    for e0, e1 in ev:
        e0.record(st)
        pp.launch(st.cuda_stream)
        e1.record(st)
    torch.cuda.synchronize()
    samples = sorted(e0.elapsed_time(e1) * 1e6 for e0, e1 in ev)
    mid = repeats // 2
    return samples[mid] if repeats % 2 else 0.5 * (samples[mid - 1] + samples[mid])


@dataclasses.dataclass
class BenchRecord:
    layer: str
    comp: Component
    sparsity: float
    mode: RunMode
    workers: int
    median_ns: float
    exec_fmas: int
    speedup_vs_dense: float


@dataclasses.dataclass
class SweepRequest:
    layers: list
    comps: list = dataclasses.field(default_factory=lambda: [Component.fwd])
    grid: list = dataclasses.field(default_factory=lambda: [0.0, 0.5, 0.9])
    minibatch: int = 4
    scale: int = 2
    V: int = 16
    workers: int = 1
    repeats: int = 5  # timed calls after 2 warmups
    seed: int = 1
    timing: str = "device"  # "device" (CUDA events, resident) or "host" (wall clock, host buffers)


def _timed_run(pr: Prepared, sh: ConvShape, mode: RunMode, req: SweepRequest) -> tuple[float, int]:
    if req.timing == "host":
        box = {}

        def call():
            box["r"] = run_parallel(pr.a, pr.b, sh, pr.plan, mode, req.workers)
        ns = time_median_ns(call, req.repeats)
        return ns, box["r"].counters.executed_vector_fmas
    if req.timing != "device":
        raise SpconvError(_lib.SPC_ERR_ARG, f"unknown timing {req.timing!r}")
    import torch
    a, b = pr.a.to("cuda"), pr.b.to("cuda")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    pp = PreparedPass(a, b, sh, pr.plan, mode, counters=cnt)
    ns = device_median_ns(pp, req.repeats)
    return ns, pp.read_counters().executed_vector_fmas  # the kernels re-zero the counters per call


def run_sweep(req: SweepRequest) -> list[BenchRecord]:
    """bench.cpp:215-292: a dense-mode baseline per (layer, component), one
    sparse record per grid point, then geo-mean speedup rows per
    (component, sparsity) under the layer name "geomean"."""
    records: list[BenchRecord] = []
    speedups: dict[tuple[int, float], list[float]] = {}
    for lname in req.layers:
        lc = find_layer(lname)
        if lc is None:
            raise SpconvError(_lib.SPC_ERR_ARG, "unknown layer: " + lname)
        sh = scaled_shape(lc.shape, req.minibatch, req.scale)
        for comp in req.comps:
            comp = Component(comp)
            dpr = prepare(sh, comp, 0.0, req.V, BwwCheck.input, req.seed)
            dense_ns, dense_fmas = _timed_run(dpr, sh, RunMode.dense, req)
            records.append(BenchRecord(lname, comp, 0.0, RunMode.dense, req.workers, dense_ns, dense_fmas, 1.0))
            for s in req.grid:
                pr = prepare(sh, comp, s, req.V, BwwCheck.input, req.seed)
                ns, fmas = _timed_run(pr, sh, RunMode.sparse, req)
                rec = BenchRecord(lname, comp, float(s), RunMode.sparse, req.workers, ns, fmas, dense_ns / ns)
                records.append(rec)
                speedups.setdefault((int(comp), float(s)), []).append(rec.speedup_vs_dense)
    for (comp, s), vals in sorted(speedups.items()):
        records.append(BenchRecord("geomean", Component(comp), s, RunMode.sparse, req.workers, 0.0, 0,
                                   geo_mean(vals)))
    return records


def geo_mean(xs) -> float:
    xs = list(xs)
    if not xs:
        raise SpconvError(_lib.SPC_ERR_ARG, "geo_mean of nothing")
    if any(x <= 0.0 for x in xs):
        raise SpconvError(_lib.SPC_ERR_ARG, "geo_mean needs positive values")
    return math.exp(sum(math.log(x) for x in xs) / len(xs))


def _num(x) -> str:
    """A double the way std::ostream prints it by default (%g, 6 digits)."""
    if isinstance(x, (int, np.integer)) and not isinstance(x, bool):
        return str(int(x))
    return "%g" % x


def write_sweep_csv(records, out) -> None:
    """bench.cpp:303-312."""
    out.write("layer,component,sparsity,mode,workers,median_ns,exec_fmas,speedup_vs_dense\n")
    for r in records:
        out.write(f"{r.layer},{COMPONENT_NAMES[Component(r.comp)]},{_num(float(r.sparsity))},"
                  f"{'sparse' if r.mode == RunMode.sparse else 'dense'},{r.workers},{_num(float(r.median_ns))},"
                  f"{int(r.exec_fmas)},{_num(float(r.speedup_vs_dense))}\n")


def write_curves_csv(records, out) -> None:
    """bench.cpp:314-327: sparse rows with their (layer, component) dense time."""
    dense = {(r.layer, int(r.comp)): r.median_ns for r in records if r.mode == RunMode.dense}
    out.write("layer,component,sparsity,median_ns,dense_ns\n")
    for r in records:
        if r.mode != RunMode.sparse or r.layer == "geomean":
            continue
        key = (r.layer, int(r.comp))
        if key not in dense:
            raise SpconvError(_lib.SPC_ERR_ARG, "curves: missing dense baseline for " + r.layer)
        out.write(f"{r.layer},{COMPONENT_NAMES[Component(r.comp)]},{_num(float(r.sparsity))},"
                  f"{_num(float(r.median_ns))},{_num(float(dense[key]))}\n")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="GPU sparsity sweep with the reference's CSV columns")
    ap.add_argument("--layers", nargs="+", default=["resnet2_2"])
    ap.add_argument("--comps", nargs="+", default=["fwd"], choices=["fwd", "bwi", "bww"])
    ap.add_argument("--grid", nargs="+", type=float, default=[0.0, 0.5, 0.9])
    ap.add_argument("--minibatch", type=int, default=4)
    ap.add_argument("--scale", type=int, default=2)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--timing", default="device", choices=["device", "host"])
    ap.add_argument("--csv", default="-", help="sweep CSV path ('-' = stdout)")
    ap.add_argument("--curves", default=None, help="projector curves CSV path")
    a = ap.parse_args(argv)
    req = SweepRequest(layers=a.layers, comps=[Component[c] for c in a.comps], grid=a.grid,
                       minibatch=a.minibatch, scale=a.scale, repeats=a.repeats, seed=a.seed, timing=a.timing)
    recs = run_sweep(req)
    if a.csv == "-":
        write_sweep_csv(recs, sys.stdout)
    else:
        with open(a.csv, "w") as f:
            write_sweep_csv(recs, f)
    if a.curves:
        with open(a.curves, "w") as f:
            write_curves_csv(recs, f)
    return 0


if __name__ == "__main__":
    sys.exit(main())
