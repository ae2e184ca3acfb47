"""bench.py -- dense-equivalent GFLOP/s of the sparse FWD/BWI/BWW conv passes.

Metric (BASELINE.json): dense-equiv GFLOP/s per FWD/BWI/BWW conv pass vs ReLU
sparsity, 1/2/4/8 GPUs.  Workload (BASELINE cfg 2): the 12 non-initial 3x3
convs of VGG16, batch 32 per GPU, 224x224, fp32, i.i.d. ReLU sparsity swept
over {0.4, 0.6, 0.8, 0.9} for both activations and output gradients.

One STEP = for each sparsity in the grid, for each of the 12 layers: FWD, BWI
and BWW (check = input, as the reference's sweep does, P/src/bench.cpp:228),
plus (N > 1) the NCCL allreduce of each layer's weight gradient.
Dense-equivalent FLOPs per pass = 2*N*K*C*R*S*H'*W'.

  value  = whole-job dense-equiv GFLOP/s, inputs resident in HBM, CUDA events,
           max over ranks.
  e2e    = same metric through the reference-facing C ABI with HOST buffers
           (spc_run_parallel_host: pinned H2D, kernels, D2H, sync per call).
  cpu_baseline / --impl reference = the UNMODIFIED reference library
           (oracle/_ref, run_parallel, all host threads) on a bounded sample.

Inputs are larger than L2 within a step (every layer's tensors are touched
once per step; the step's working set is ~25 GB), so no separate flush.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GRID = (0.4, 0.6, 0.8, 0.9)
METRIC = "dense-equiv GFLOP/s per FWD/BWI/BWW conv pass vs ReLU sparsity"
PASSES = ("fwd", "bwi", "bww")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# The result line goes to the real stdout; anything native libraries write to
# file descriptor 1 (e.g. NCCL's version banner) is redirected to stderr so the
# driver always sees exactly one JSON line.
_RESULT_FD = os.dup(1)
os.dup2(2, 1)


def emit(obj):
    os.write(_RESULT_FD, (json.dumps(obj) + "\n").encode())


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception as e:  # no nvidia-smi
            log("clock sampler unavailable:", e)
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        reasons = set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for s in self.samples:
            for n, v in zip(names, s[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = sorted(sm)[len(sm) // 4:] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(self.samples),
                "power_w_max": max((float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()),
                                   default=None)}


# ---------------------------------------------------------------- reference arm
def reference_sample(layers, grid, n_img, workers, seed=0):
    """Time the unmodified reference CPU library (run_parallel, backend
    automatic, `workers` threads) on a batch slice of every layer and sparsity.
    Returns (dense-equiv flops, seconds)."""
    import numpy as np

    import oracle
    from paper_1911_10175_b200 import workloads as wl
    rng = np.random.default_rng(seed)
    flops = 0.0
    secs = 0.0
    for s in grid:
        for layer in layers:
            sh = layer.shape.with_batch(n_img)
            t = sh.astuple()
            D = wl.host_activation((sh.N, sh.C, sh.H, sh.W), s, rng)
            G = wl.host_weights(sh.K, sh.C, sh.S, sh.R, rng)
            dY = wl.host_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, rng)
            for comp, a, b in ((0, D, G), (1, dY, G), (2, D, dY)):
                r = oracle.RefRun(comp, 0, t, 16, a, b)
                t0 = time.perf_counter()
                r.exec(0, workers)  # run_parallel: the reference's timed call (bench.cpp:249-271)
                secs += time.perf_counter() - t0
                flops += sh.dense_flops()
                r.close()
    return flops, secs


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from paper_1911_10175_b200 import workloads as wl
    if not oracle.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libspconv_ref.so was not built"})
        return
    layers = wl.CONFIGS[args.config]()
    workers = os.cpu_count() or 1
    n_img = args.ref_images
    for _ in range(args.warmup):
        reference_sample(layers, args.grid[:1], n_img, workers)
    tot_f = tot_s = 0.0
    for k in range(args.steps):
        f, s = reference_sample(layers, args.grid, n_img, workers, seed=k)
        tot_f += f
        tot_s += s
    value = tot_f / tot_s / 1e9
    sample = (f"{n_img} image(s) of batch {layers[0].shape.N} x {len(layers)} layers x FWD/BWI/BWW x sparsity "
              f"{list(args.grid)}; run_parallel (P/src/kernels.cpp:304), backend automatic")
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tot_s / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, ws), "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(out)


WORKLOAD_NAMES = {
    "vgg16_b32": "VGG16 non-initial 3x3 convs (12 layers) x FWD/BWI/BWW",
    "cfg1_single3x3_b16": "single 3x3 conv N=16 C=K=64 56x56 x FWD/BWI/BWW",
    "resnet34_b64": "ResNet-34 3x3 convs + 1x1 s2 projections (35 layers) x FWD/BWI/BWW",
    "resnet50_b64": "ResNet-50 v1.5 bottleneck convs (52 layers) x FWD/BWI/BWW",
    "fixup_resnet50_b256": "Fixup ResNet-50 conv stack (52 layers, batch 256) x FWD/BWI/BWW",
}


def config_dict(args, ws):
    from paper_1911_10175_b200 import workloads as wl
    n = wl.CONFIGS[args.config]()[0].shape.N
    return {"workload": f"{args.config}: {WORKLOAD_NAMES.get(args.config, args.config)}",
            "global_batch": n * ws, "per_gpu_batch": n, "resolution": 224, "vector_width": 16,
            "sparsity_grid": list(args.grid), "bww_check": "input",
            "parallelism": f"dp{ws} (batch-sharded, BWW dG allreduce)",
            "l2": "inputs larger than L2 (step working set ~25 GB, each tensor touched once per step)"}


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="vgg16_b32")
    ap.add_argument("--grid", type=float, nargs="+", default=list(GRID))
    ap.add_argument("--ref-images", type=int, default=1, help="reference-arm batch slice per layer")
    ap.add_argument("--cpu-images", type=int, default=8, help="cpu_baseline batch slice per layer")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tc", action="store_true", help="skip the 3xTF32 tensor-core variant")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_10175_b200 as sp
    from paper_1911_10175_b200 import workloads as wl

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (any world size) the collective path is live: NCCL
    # process group, per-layer dG allreduce on a comm stream, barriers and
    # max-over-ranks timing -- so a 1-GPU torchrun run exercises it too
    distributed = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    V = 16
    layers = wl.CONFIGS[args.config]()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    # ---------------- setup: resident inputs, prepared passes (untimed)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    work = []  # (s, layer_idx, pass, PreparedPass, dense_flops)
    dgs = []   # (s, layer_idx, dG tensor) for the allreduce
    t_setup = time.time()
    for s in args.grid:
        for li, layer in enumerate(layers):
            sh = layer.shape
            G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, gen)
            D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, gen)
            dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, gen)
            bD = sp.pack_act_nchwc(D, V)
            bDc = sp.nchwc_to_chwnn(bD)
            bY = sp.pack_act_nchwc(dY, V)
            del D, dY
            ops = {"fwd": (bD, sp.pack_filter(G, V)), "bwi": (bY, sp.pack_filter(G, V, True)), "bww": (bDc, bY)}
            for name in PASSES:
                a, b = ops[name]
                pl = sp.plan(sh, sp.Component[name], V, 30, sp.BwwCheck.input)
                cnt = torch.zeros(4, dtype=torch.int64, device=dev)
                pp = sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse, counters=cnt)
                work.append((s, li, name, pp, sh.dense_flops()))
                if name == "bww":
                    dgs.append((s, li, pp.out))
    torch.cuda.synchronize()
    log(f"[rank {rank}] setup {time.time() - t_setup:.1f}s, {len(work)} passes/step, "
        f"{torch.cuda.memory_allocated(dev) / 2**30:.1f} GiB resident")

    comm_stream = torch.cuda.Stream(device=dev) if distributed else None

    def step(events=None):
        for idx, (s, li, name, pp, _) in enumerate(work):
            if events is not None:
                events[idx][0].record(stream)
            pp.launch(sptr)
            if events is not None:
                events[idx][1].record(stream)
            if distributed and name == "bww":
                # BWW weight-gradient exchange: NCCL allreduce (sum) over NVLink,
                # on a comm stream so it overlaps the next layer's passes
                ev = torch.cuda.Event()
                ev.record(stream)
                comm_stream.wait_event(ev)
                with torch.cuda.stream(comm_stream):
                    dist.all_reduce(pp.out)
        if distributed:
            stream.wait_stream(comm_stream)

    # warmup (also validates every pass once, counters read back)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    exec_fmas = {}
    for (s, li, name, pp, _) in work:
        exec_fmas[(s, li, name)] = pp.read_counters().executed_vector_fmas
    # FFMA peak probe (roofline denominator for the FP32 CUDA-core pipe)
    peak = ffma_peak(sp, dev, sptr)

    # ---------------- timed region
    if distributed:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in work]
    per_launch_ms = np.zeros(len(work))
    launches0 = sp.launch_count()
    torch.cuda.synchronize()
    e_start = torch.cuda.Event(enable_timing=True)
    e_stop = torch.cuda.Event(enable_timing=True)
    e_start.record(stream)
    for _ in range(args.steps):
        step(events)
    e_stop.record(stream)
    torch.cuda.synchronize()
    launches = sp.launch_count() - launches0
    for idx, (a, b) in enumerate(events):
        per_launch_ms[idx] = a.elapsed_time(b)  # last step's per-pass durations
    total_ms = e_start.elapsed_time(e_stop)
    clocks.stop()
    if distributed:
        t = torch.tensor([total_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        dist.barrier()
    ms_per_step = total_ms / args.steps
    flops_step = sum(w[4] for w in work)
    value = ws * flops_step / (ms_per_step * 1e-3) / 1e9

    # per (sparsity, pass) breakdown from the last timed step
    sweep = {}
    for idx, (s, li, name, pp, fl) in enumerate(work):
        d = sweep.setdefault(f"{s:.1f}", {}).setdefault(name, {"ms": 0.0, "dense_flops": 0.0, "useful_flops": 0.0})
        d["ms"] += per_launch_ms[idx]
        d["dense_flops"] += fl
        d["useful_flops"] += 2.0 * V * exec_fmas[(s, li, name)]
    breakdown = {}
    for s, passes in sweep.items():
        breakdown[s] = {n: {"dense_equiv_gflops": round(v["dense_flops"] / v["ms"] / 1e6, 1),
                            "useful_gflops": round(v["useful_flops"] / v["ms"] / 1e6, 1),
                            "ms": round(v["ms"], 3)} for n, v in passes.items()}

    # roofline for the dominant kernel family (largest share of the step)
    fam_ms = {n: sum(per_launch_ms[i] for i, w in enumerate(work) if w[2] == n) for n in PASSES}
    dom = max(fam_ms, key=fam_ms.get)
    dom_idx = [i for i, w in enumerate(work) if w[2] == dom]
    useful = sum(2.0 * V * exec_fmas[(work[i][0], work[i][1], dom)] for i in dom_idx)
    dom_ms = sum(per_launch_ms[i] for i in dom_idx)
    achieved = useful / (dom_ms * 1e-3) / 1e12
    traffic, traffic_src = load_traffic(dom)
    roofline = {"bound": "fp32", "kernel": f"{dom} tile kernel ({len(dom_idx)} launches/step)",
                "achieved": round(achieved, 3), "peak": round(peak, 3), "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4) if peak else None,
                "traffic": traffic,
                "traffic_note": (f"dram__bytes_read+write per launch, {traffic_src['launch']}, "
                                 f"{traffic_src['traffic_over_algorithmic']}x its algorithmic bytes "
                                 f"({traffic_src['source']})") if traffic_src else None,
                "basis": "useful FLOPs = 2*V*executed_vector_fmas (exact in-kernel count) per launch / "
                         "CUDA-event launch duration; peak = live FFMA-pipe probe (MEASURED_PEAKS.json has no "
                         "FP32 entry)",
                "share_of_step": round(dom_ms / (ms_per_step), 3),
                "dense_equiv_tflops": round(sum(work[i][4] for i in dom_idx) / (dom_ms * 1e-3) / 1e12, 3)}

    # speedup vs the same kernels run dense (zero check off) at sparsity 0
    dense0 = dense_baseline(sp, wl, layers, dev, sptr, V)
    # the optional 3xTF32 tensor-core variant on the same resident work
    tc = None if args.no_tc else tf32x3_variant(args, sp, work, step, stream, ws, distributed)

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, ws), "gpu_launches": int(launches),
        "clocks": clocks.summary(), "roofline": roofline, "sweep": breakdown,
        "dense_mode_at_s0": dense0,
    }
    if tc is not None:
        out["tf32x3_variant"] = tc
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args, layers)
    if not args.no_e2e:
        out["e2e"] = e2e(args, sp, work, ws, rank, distributed)
    if rank == 0:
        emit(out)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()


def tf32x3_variant(args, sp, work, step, stream, ws, distributed):
    """The same step with spc_set_math(SPC_MATH_TF32X3): FWD/BWI/BWW on the
    tcgen05 tensor cores with 3xTF32 split products.  A
    separately stated tolerance; reported beside -- not instead of -- the FP32
    FFMA headline."""
    import numpy as np
    import torch
    prev = sp.set_math(sp.Math.tf32x3)
    try:
        step()  # warm-up (scratch pools, tensor maps)
        torch.cuda.synchronize()
        if distributed:
            import torch.distributed as dist
            dist.barrier()
        events = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in work]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(events)
        e1.record(stream)
        torch.cuda.synchronize()
    finally:
        sp.set_math(prev)
    total_ms = e0.elapsed_time(e1)
    if distributed:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_step = total_ms / args.steps
    per = np.array([a.elapsed_time(b) for a, b in events])
    flops_step = sum(w[4] for w in work)
    sweep = {}
    for idx, (s, li, name, pp, fl) in enumerate(work):
        d = sweep.setdefault(f"{s:.1f}", {}).setdefault(name, [0.0, 0.0])
        d[0] += fl
        d[1] += per[idx]
    fam = {n: [sum(w[4] for w in work if w[2] == n), sum(per[i] for i, w in enumerate(work) if w[2] == n)]
           for n in PASSES}
    dom = max(fam, key=lambda n: fam[n][1])
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        tf32_peak, peak_src = peaks["bf16_tflops"] / 2.0, "MEASURED_PEAKS.json bf16_tflops / 2 (tf32 = half bf16 rate)"
    except Exception:
        tf32_peak, peak_src = 1100.0, "B200_PROFILING.md nominal dense tf32 1.1 PFLOP/s (fallback)"
    mma_tflops = 3.0 * fam[dom][0] / (fam[dom][1] * 1e-3) / 1e12  # three tf32 products per fp32 product
    return {
        "math": "3xTF32 split products (hi*hi + hi*lo + lo*hi), fp32 accumulation in TMEM drained to fp32 "
                "registers every 8 pipeline stages; spc_set_math(SPC_MATH_TF32X3)",
        "tolerance": "max|got-ref|/max|ref| <= 1e-5 vs the 64-bit oracle (tests/test_gpu_tc.py); measured "
                     "0.5e-6 - 1.4e-6 (the reference CPU fp32 kernels: 0.4e-6 - 1.0e-6)",
        "value": round(ws * flops_step / (ms_step * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
        "ms_per_step": round(ms_step, 3),
        "sweep": {s: {n: {"dense_equiv_gflops": round(f / ms / 1e6, 1), "ms": round(ms, 3)}
                      for n, (f, ms) in d.items()} for s, d in sweep.items()},
        "roofline": {"bound": "tensor", "kernel": f"{dom} tcgen05 kernel", "achieved": round(mma_tflops, 1),
                     "peak": round(tf32_peak, 1), "unit": "TFLOP/s", "frac": round(mma_tflops / tf32_peak, 4),
                     "basis": "issued tf32 MMA FLOPs = 3 x dense-equiv FLOPs (padding rows not counted) / "
                              "CUDA-event pass durations (prep + GEMM + reduce); peak = " + peak_src},
    }


def ffma_peak(sp, dev, sptr):
    import ctypes

    import torch
    L = sp._lib.load()
    buf = torch.zeros(16, device=dev)
    fl = ctypes.c_double()
    blocks, iters = 148 * 16, 4096
    for _ in range(2):
        L.spc_ffma_peak_kernel(ctypes.c_void_p(buf.data_ptr()), blocks, iters, ctypes.byref(fl), ctypes.c_void_p(sptr))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        L.spc_ffma_peak_kernel(ctypes.c_void_p(buf.data_ptr()), blocks, iters, ctypes.byref(fl), ctypes.c_void_p(sptr))
    e1.record()
    torch.cuda.synchronize()
    return 5 * fl.value / (e0.elapsed_time(e1) * 1e-3) / 1e12


def load_traffic(family):
    """dram bytes per launch of the dominant kernel, from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))[family]
        return d["dram_bytes_per_launch"], d
    except Exception:
        return None, None


def dense_baseline(sp, wl, layers, dev, sptr, V):
    """Same kernels, run_mode::dense (zero check off), at sparsity 0 -- the
    speedup denominator (P/src/bench.cpp:227-236).  One pass of each layer."""
    import torch
    gen = torch.Generator(device=dev).manual_seed(7)
    tot = {n: [0.0, 0.0] for n in PASSES}
    for layer in layers:
        sh = layer.shape
        G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, gen)
        bD = sp.pack_act_nchwc(wl.device_activation((sh.N, sh.C, sh.H, sh.W), 0.0, gen), V)
        bY = sp.pack_act_nchwc(wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), 0.0, gen), V)
        ops = {"fwd": (bD, sp.pack_filter(G, V)), "bwi": (bY, sp.pack_filter(G, V, True)),
               "bww": (sp.nchwc_to_chwnn(bD), bY)}
        for n in PASSES:
            a, b = ops[n]
            pp = sp.PreparedPass(a, b, sh, sp.plan(sh, sp.Component[n], V), sp.RunMode.dense)
            pp.launch(sptr)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            pp.launch(sptr)
            e1.record()
            torch.cuda.synchronize()
            tot[n][0] += sh.dense_flops()
            tot[n][1] += e0.elapsed_time(e1)
        del ops, bD, bY
        torch.cuda.empty_cache()
    return {n: {"dense_equiv_gflops": round(f / ms / 1e6, 1), "ms": round(ms, 3)} for n, (f, ms) in tot.items()}


def cpu_baseline(args, layers):
    import oracle
    if not oracle.ref_available():
        return {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    workers = os.cpu_count() or 1
    f, s = reference_sample(layers, args.grid, args.cpu_images, workers)
    return {"value": round(f / s / 1e9, 3), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
            "sample": f"{args.cpu_images} image(s) per layer x {len(layers)} layers of {args.config} x FWD/BWI/BWW x sparsity "
                      f"{list(args.grid)} ({f / 1e9:.0f} dense-equiv GFLOP in {s:.1f} s); reference "
                      f"run_parallel, backend automatic, {workers} workers"}


def e2e(args, sp, work, ws, rank, distributed=False):
    """Same metric through the host-buffer C ABI (spc_run_parallel_host):
    pinned host inputs -> H2D -> kernels -> D2H of every output, per call."""
    import torch
    host = []
    h2d = d2h = 0
    for (s, li, name, pp, fl) in work:
        a = sp.BlockedTensor(**{**pp._a.header(), "data": pp._a.data.cpu().pin_memory().numpy()})
        b = sp.BlockedTensor(**{**pp._b.header(), "data": pp._b.data.cpu().pin_memory().numpy()})
        out = torch.empty(pp.out.numel(), dtype=torch.float32).pin_memory().numpy()
        host.append((a, b, pp, out, fl))
        h2d += (a.data.nbytes + b.data.nbytes)
        d2h += out.nbytes + 32
    import ctypes
    L = sp._lib.load()

    def one_step():
        for a, b, pp, out, fl in host:
            ca, cb = a.to_c(), b.to_c()
            cd = sp._lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.ctypes.data, out.size)
            cnt = sp._lib.spc_counters()
            st = L.spc_run_parallel_host(ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(pp._shape),
                                         ctypes.byref(pp._plan), 0, ctypes.byref(cd), ctypes.byref(cnt))
            if st:
                raise sp.SpconvError(st, sp._lib.last_error())

    one_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        one_step()
    secs = (time.perf_counter() - t0) / args.e2e_steps
    if distributed:
        import torch.distributed as dist
        t = torch.tensor([secs], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        secs = float(t.item())
    flops = sum(h[4] for h in host)
    return {"value": round(ws * flops / secs / 1e9, 1), "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "s_per_step": round(secs, 3),
            "path": "spc_run_parallel_host (include/spconv_b200.h), pinned host buffers, per-call H2D+D2H+sync"}


if __name__ == "__main__":
    main()
