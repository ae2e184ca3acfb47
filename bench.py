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
  e2e    = same metric through the reference-facing C ABI with HOST buffers:
           the step's passes as one spc_run_parallel_host_batch call (pinned
           H2D of every input, kernels, D2H of every output, pipelined across
           passes); e2e.per_call = one synchronous spc_run_parallel_host call
           per pass (the plain drop-in), e2e.pageable = pageable buffers.
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
# Everything on this arm runs the UNMODIFIED reference library (oracle/_ref,
# built from /root/reference's sources by oracle/Makefile) through its public
# API: shapes from the reference's conv_shape::make (P/src/tensor.cpp:11-14),
# operands packed by the reference (pack_act_* / pack_filter), the timed call
# spconv::run_parallel (P/src/kernels.cpp:304-313) with backend automatic and
# every host thread.  It never loads the product library: the layer table and
# the input generators are plain numpy (workloads.SPECS / *_host).
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_layers(config, n_img=None):
    """[(name, PlainShape)] of `config`, built by the reference's own conv_shape::make."""
    import oracle
    from paper_1911_10175_b200 import workloads as wl
    out = []
    for name, N, C, K, hw, R, stride in wl.SPECS[config]():
        t = oracle.ref_shape_make(n_img or N, C, K, hw, hw, R, R, stride, stride)
        out.append((name, wl.PlainShape(t)))
    return out


def reference_sample(config, grid, n_img, workers, mode=0, seed=0, passes=(0, 1, 2)):
    """Time the reference's run_parallel on `n_img` images of every layer of
    `config` at each sparsity of `grid` (FWD, BWI, BWW check = input, as the
    reference's own sweep, P/src/bench.cpp:228).  Inputs: the config's
    distributions (workloads.layer_inputs_host).  Returns (dense-equiv flops,
    seconds inside run_parallel)."""
    import oracle
    from paper_1911_10175_b200 import workloads as wl
    flops = secs = 0.0
    for s in grid:
        for li, (name, sh) in enumerate(ref_layers(config, n_img)):
            D, G, dY = wl.layer_inputs_host(config, li, sh, s, seed=seed)
            for comp in passes:
                a, b = ((D, G), (dY, G), (D, dY))[comp]
                r = oracle.RefRun(comp, 0, sh.astuple(), 16, a, b)
                t0 = time.perf_counter()
                r.exec(mode, workers)  # run_parallel: the reference's timed call (bench.cpp:249-271)
                secs += time.perf_counter() - t0
                flops += sh.dense_flops()
                r.close()
    return flops, secs


def ref_images(config):
    """Reference-arm sample per layer: one full 16-image ActCHWNn lane block
    (the BWW check tensor's N lanes are all live), or the whole batch when smaller."""
    from paper_1911_10175_b200 import workloads as wl
    return min(16, wl.SPECS[config]()[0][1])


def ref_grid(config, grid):
    from paper_1911_10175_b200 import workloads as wl
    return list(grid) if config in wl.GRID_CONFIGS else [None]


def assert_product_not_loaded():
    maps = open("/proc/self/maps").read()
    assert "libspconv_b200" not in maps, "reference arm loaded the product library"


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    if not oracle.ref_available():
        emit({"impl": "reference", "unavailable": "oracle/_ref/libspconv_ref.so was not built"})
        return
    workers = os.cpu_count() or 1
    n_img = args.ref_images or ref_images(args.config)
    grid = ref_grid(args.config, args.grid)
    # one step = every layer x FWD/BWI/BWW at ONE sparsity of the grid
    # (rotating through the grid step by step), n_img images per layer
    for k in range(args.warmup):
        reference_sample(args.config, [grid[k % len(grid)]], n_img, workers, seed=100 + k)
    tot_f = tot_s = 0.0
    for k in range(args.steps):
        f, s = reference_sample(args.config, [grid[k % len(grid)]], n_img, workers, seed=k)
        tot_f += f
        tot_s += s
    assert_product_not_loaded()
    value = tot_f / tot_s / 1e9
    n_full = ref_layers(args.config)[0][1].N
    sample = (f"{n_img} of {n_full} images x {len(ref_layers(args.config))} layers x FWD/BWI/BWW per step, "
              f"sparsity rotating over {grid} step by step; run_parallel (P/src/kernels.cpp:304), backend "
              f"automatic, {workers} threads; CPU: {cpu_model()}")
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(tot_s / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, ws), "impl": "reference",
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
                         "cpu_model": cpu_model(), "sample": sample},
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
    from paper_1911_10175_b200.dist import shard_range
    n = wl.SPECS[args.config]()[0][1]
    per = [shard_range(n, ws, r)[1] for r in range(ws)]
    return {"workload": f"{args.config}: {WORKLOAD_NAMES.get(args.config, args.config)}",
            "global_batch": n, "per_gpu_batch": per[0] if min(per) == max(per) else per,
            "resolution": 224, "vector_width": 16,
            "sparsity": (list(args.grid) if args.config in wl.GRID_CONFIGS else SPARSITY_NOTE.get(args.config)),
            "bww_check": "input",
            "parallelism": f"dp{ws} (global batch sharded over ranks, BWW dG NCCL allreduce)",
            "l2": "inputs larger than L2 (step working set > 1 GB, each tensor touched once per step)"}


SPARSITY_NOTE = {
    "cfg1_single3x3_b16": "D: i.i.d. ReLU(N(-t,1)) at 0.5; dY: N(0,1) x independent 50% Bernoulli mask (seed 0)",
    "resnet34_b64": "D: per-layer i.i.d. s_l ~ U[0.4, 0.8] (seeded); dY dense (BatchNorm)",
    "resnet50_b64": "D: spatially correlated ReLU(conv3x3_rand(N(0,1)) - tau), mean 0.6; dY dense (BatchNorm)",
    "fixup_resnet50_b256": "ReLU masks of the chain's own seeded forward pass (~0.7 activation sparsity)",
}


# ---------------------------------------------------------------- our arm
class TorchComm:
    """The product communicator's interface (window / allreduce / close) over a
    torch.distributed group -- only for SPC_BENCH_BACKEND=gloo dry runs."""

    def __init__(self, dist):
        self.dist = dist
        self.size = dist.get_world_size()

    def window(self, numel):
        import torch
        return torch.zeros(numel, dtype=torch.float32, device="cuda"), False

    def allreduce(self, buf, stream_ptr):
        import torch
        st = torch.cuda.ExternalStream(stream_ptr)
        st.synchronize()
        self.dist.all_reduce(buf)

    def close(self):
        pass


def relaunch_distributed(args) -> int:
    """`python bench.py --gpus N` outside torchrun: re-exec this script as N
    ranks under torch.distributed.run (one process per GPU, 127.0.0.1
    rendezvous); the rank-0 child prints the JSON line on our stdout."""
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        log(f"--gpus {args.gpus} requested but only {have} CUDA device(s) are visible")
        return 2
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"),
               NCCL_DEBUG_SUBSYS=os.environ.get("NCCL_DEBUG_SUBSYS", "INIT"))
    log("relaunch:", " ".join(cmd))
    return subprocess.run(cmd, env=env, stdout=_RESULT_FD).returncode


def build_work(args, sp, wl, dev, n_local, rank, dg_alloc):
    """Resident inputs and prepared passes of one step on this rank's batch
    shard: [(tag, layer_idx, pass, PreparedPass, global dense flops, dG buf)]."""
    import torch
    V = 16
    specs = wl.SPECS[args.config]()
    grid = list(args.grid) if args.config in wl.GRID_CONFIGS else [None]
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    work = []
    for s in grid:
        for li, spec in enumerate(specs):
            gsh = sp.ConvShape.make(spec[1], spec[2], spec[3], spec[4], spec[4], spec[5], spec[5], spec[6], spec[6])
            sh = gsh.with_batch(n_local)
            D, G, dY = wl.layer_inputs_device(args.config, li, sh, gen, s)
            bD = sp.pack_act_nchwc(D, V)
            bDc = sp.nchwc_to_chwnn(bD)
            bY = sp.pack_act_nchwc(dY, V)
            del D, dY
            ops = {"fwd": (bD, sp.pack_filter(G, V)), "bwi": (bY, sp.pack_filter(G, V, True)), "bww": (bDc, bY)}
            tag = f"{s:.1f}" if s is not None else "cfg"
            for name in PASSES:
                a, b = ops[name]
                pl = sp.plan(sh, sp.Component[name], V, 30, sp.BwwCheck.input)
                cnt = torch.zeros(4, dtype=torch.int64, device=dev)
                out = dg_alloc(gsh.K * gsh.C * gsh.R * gsh.S) if name == "bww" else None
                pp = sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse, out=out, counters=cnt)
                work.append((tag, li, name, pp, gsh.dense_flops(), out))
    return work


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="vgg16_b32", choices=sorted(WORKLOAD_NAMES))
    ap.add_argument("--grid", type=float, nargs="+", default=list(GRID))
    ap.add_argument("--ref-images", type=int, default=0,
                    help="reference-arm images per layer (0: one full 16-image lane block)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-tc", action="store_true", help="skip the 3xTF32 tensor-core variant")
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE configs' lines")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if args.impl == "reference":
        run_reference_arm(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1911_10175_b200 as sp
    from paper_1911_10175_b200 import workloads as wl
    from paper_1911_10175_b200.dist import Comm, shard_range

    ws, rank, local = dist_env()
    # SPC_BENCH_BACKEND=gloo: a dry run of the multi-rank logic (sharding,
    # max-over-ranks timing, the JSON line) with several ranks on ONE GPU --
    # NCCL refuses two ranks per device; the dG exchange then goes through
    # torch.distributed (gloo) instead of the product communicator.  Numbers
    # from such a run are not measurements.
    dry_backend = os.environ.get("SPC_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    dev = torch.device("cuda", local % max(1, torch.cuda.device_count()))
    # under torchrun (any world size) the collective path is live: the
    # product's NCCL communicator (csrc/comm.cu) with dG in a symmetric window,
    # per-layer allreduce on a comm stream, barriers, max-over-ranks timing
    distributed = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    comm = None
    if distributed and dry_backend == "gloo":
        dist.init_process_group("gloo")
        comm = TorchComm(dist)
        log(f"[rank {rank}] dry run: gloo process group, {ws} ranks on cuda:{dev.index}")
    elif distributed:
        dist.init_process_group("nccl", device_id=dev)
        comm = Comm()
        log(f"[rank {rank}] spc_comm: {comm.size} ranks, NCCL {sp._lib.load().spc_nccl_version()}")
    V = 16
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    N_global = wl.SPECS[args.config]()[0][1]
    _, n_local = shard_range(N_global, ws, rank)

    if args.config == "fixup_resnet50_b256":
        return run_chain_bench(args, sp, dev, stream, ws, rank, local, comm, distributed)

    # ---------------- setup: resident inputs, prepared passes (untimed)
    t_setup = time.time()
    specs = wl.SPECS[args.config]()
    grid = list(args.grid) if args.config in wl.GRID_CONFIGS else [None]
    dg_total = len(grid) * sum(t[2] * t[3] * t[5] * t[5] for t in specs)
    symmetric = False
    if comm is not None:
        dg_buf, symmetric = comm.window(dg_total)
    else:
        dg_buf = torch.empty(dg_total, dtype=torch.float32, device=dev)
    cursor = [0]

    def dg_alloc(n):
        start = cursor[0]
        cursor[0] += n
        return dg_buf.slice(start, n) if hasattr(dg_buf, "slice") else dg_buf[start:start + n]

    work = build_work(args, sp, wl, dev, n_local, rank, dg_alloc)
    torch.cuda.synchronize()
    log(f"[rank {rank}] setup {time.time() - t_setup:.1f}s, {len(work)} passes/step, batch {n_local} of "
        f"{N_global}, {torch.cuda.memory_allocated(dev) / 2**30:.1f} GiB resident")

    comm_stream = torch.cuda.Stream(device=dev) if comm is not None else None

    def step(events=None):
        for idx, (tag, li, name, pp, _, dgb) in enumerate(work):
            if events is not None:
                events[idx][0].record(stream)
            pp.launch(sptr)
            if events is not None:
                events[idx][1].record(stream)
            if comm is not None and name == "bww":
                # BWW weight-gradient exchange: in-place NCCL allreduce (sum) of
                # this layer's dG (symmetric window) on a comm stream, so it
                # overlaps the next layer's passes
                ev = torch.cuda.Event()
                ev.record(stream)
                comm_stream.wait_event(ev)
                comm.allreduce(dgb, comm_stream.cuda_stream)
        if comm is not None:
            stream.wait_stream(comm_stream)

    # warmup (also validates every pass once, counters read back)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    exec_fmas = {}
    for (tag, li, name, pp, _, _) in work:
        exec_fmas[(tag, li, name)] = pp.read_counters().executed_vector_fmas
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
    flops_step = sum(w[4] for w in work)  # global batch: every rank's shard
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # per (sparsity, pass) breakdown from the last timed step (this rank)
    sweep = {}
    for idx, (tag, li, name, pp, fl, _) in enumerate(work):
        d = sweep.setdefault(tag, {}).setdefault(name, {"ms": 0.0, "dense_flops": 0.0, "useful_flops": 0.0})
        d["ms"] += per_launch_ms[idx]
        d["dense_flops"] += fl * n_local / N_global
        d["useful_flops"] += 2.0 * V * exec_fmas[(tag, li, name)]
    breakdown = {}
    for tag, passes in sweep.items():
        breakdown[tag] = {n: {"dense_equiv_gflops": round(v["dense_flops"] / v["ms"] / 1e6, 1),
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
                "dense_equiv_tflops": round(sum(work[i][4] * n_local / N_global for i in dom_idx)
                                            / (dom_ms * 1e-3) / 1e12, 3)}

    # speedup vs the same kernels run dense (zero check off) at sparsity 0
    dense0 = dense_baseline(sp, wl, args.config, n_local, dev, sptr, V)
    # the optional 3xTF32 tensor-core variant on the same resident work
    tc = None if args.no_tc else tf32x3_variant(args, sp, work, step, stream, ws, distributed)

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(args, ws), "gpu_launches": int(launches),
        "clocks": clocks.summary(), "roofline": roofline, "sweep": breakdown,
        "dense_mode_at_s0": dense0,
    }
    if comm is not None and dry_backend == "gloo":
        out["collective"] = {"impl": "DRY RUN: torch.distributed gloo, several ranks on one GPU -- not a measurement"}
    elif comm is not None:
        out["collective"] = {"impl": "spc_bww_allreduce (csrc/comm.cu) on a comm stream",
                             "nccl_version": sp._lib.load().spc_nccl_version(), "ranks": comm.size,
                             "dG_symmetric_window": symmetric, "dG_bytes_per_step": 4 * dg_total}
    if tc is not None:
        out["tf32x3_variant"] = tc
    if not args.no_e2e:
        out["e2e"] = e2e(args, sp, work, ws, rank, comm)
    if rank == 0 and ws == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args)
    if rank == 0 and ws == 1 and not args.no_extra and args.config == "vgg16_b32":
        del work
        torch.cuda.empty_cache()
        out["other_configs"] = other_configs(args)
    if rank == 0:
        emit(out)
    if comm is not None:
        torch.cuda.synchronize()
        dist.barrier()
        comm.close()
    if distributed:
        dist.destroy_process_group()


def other_configs(args):
    """Driver-run numbers for the other BASELINE configs: each runs as its own
    bench process (`--config X --no-extra --no-cpu --no-e2e --no-tc`), short."""
    res = {}
    for cfg in ("cfg1_single3x3_b16", "resnet34_b64", "resnet50_b64", "fixup_resnet50_b256"):
        cmd = [sys.executable, os.path.abspath(__file__), "--config", cfg, "--steps", "5", "--warmup", "3",
               "--no-extra", "--no-cpu", "--no-e2e", "--no-tc"]
        t0 = time.time()
        try:
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
            line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            d = json.loads(line[-1]) if line else {"error": r.stderr[-500:]}
        except Exception as e:  # keep the headline line even if one config fails
            d = {"error": repr(e)}
        keep = ("value", "unit", "ms_per_step", "config", "dense_mode_at_s0", "sweep", "roofline",
                "activation_sparsity_mean", "gradient_sparsity_mean", "error")
        res[cfg] = {k: d[k] for k in keep if k in d}
        res[cfg]["wall_s"] = round(time.time() - t0, 1)
    return res


def run_chain_bench(args, sp, dev, stream, ws, rank, local, comm, distributed):
    """BASELINE cfg 5: the Fixup ResNet-50 training step (chain.py) -- FWD,
    BWI, BWW of all 52 convs with fused epilogues -- on this rank's shard of
    the global batch of 256, per-block dG allreduce through the product's
    communicator.  Same weights on every rank (one seed)."""
    import torch
    import torch.distributed as dist

    from paper_1911_10175_b200 import chain as CH
    from paper_1911_10175_b200.dist import CommAllreduce
    ar = CommAllreduce(comm, dev) if comm is not None else None
    t0 = time.time()
    ch = CH.fixup_resnet50(256, world=ws, rank=rank, allreduce=ar)
    torch.cuda.synchronize()
    setup = time.time() - t0
    for _ in range(args.warmup):
        ch.step(stream)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    launches0 = sp.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        ch.step(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if distributed:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    flops = ch.global_dense_flops()
    rep = ch.sparsity_report()
    out = {"metric": METRIC, "value": round(flops / (ms_step * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 3),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
           "data": "synthetic (seeded He weights, calibrated Fixup biases, ReLU(N(-t,1)) input)",
           "config": config_dict(args, ws), "gpu_launches": int((sp.launch_count() - launches0)),
           "activation_sparsity_mean": round(rep["activation_sparsity_mean"], 4),
           "gradient_sparsity_mean": round(rep["gradient_sparsity_mean"], 4),
           "passes_per_step": len(ch.passes), "setup_s": round(setup, 1)}
    if rank == 0:
        emit(out)
    if comm is not None:
        dist.barrier()
        comm.close()
    if distributed:
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
    for idx, (tag, li, name, pp, fl, _) in enumerate(work):
        d = sweep.setdefault(tag, {}).setdefault(name, [0.0, 0.0])
        d[0] += fl / ws
        d[1] += per[idx]
    fam = {n: [sum(w[4] / ws for w in work if w[2] == n), sum(per[i] for i, w in enumerate(work) if w[2] == n)]
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
        "value": round(flops_step / (ms_step * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
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


def dense_baseline(sp, wl, config, n_local, dev, sptr, V):
    """Same kernels, run_mode::dense (zero check off), at sparsity 0 -- the
    speedup denominator (P/src/bench.cpp:227-236).  One pass of each layer
    of `config` on this rank's batch shard."""
    import torch
    gen = torch.Generator(device=dev).manual_seed(7)
    tot = {n: [0.0, 0.0] for n in PASSES}
    for spec in wl.SPECS[config]():
        sh = sp.ConvShape.make(n_local, spec[2], spec[3], spec[4], spec[4], spec[5], spec[5], spec[6], spec[6])
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


def cpu_baseline(args):
    """The reference library on the box's host cores: sparse over the grid and
    dense mode at s = 0 (its own speedup denominator, P/src/bench.cpp:227-236),
    one full 16-image lane block per layer."""
    import oracle
    if not oracle.ref_available():
        return {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    workers = os.cpu_count() or 1
    n_img = args.ref_images or ref_images(args.config)
    grid = ref_grid(args.config, args.grid)
    f, s = reference_sample(args.config, grid, n_img, workers, seed=1)
    fd, sd = reference_sample(args.config, [0.0] if grid != [None] else [None], n_img, workers, mode=1, seed=2)
    return {"value": round(f / s / 1e9, 3), "unit": "GFLOP/s", "cores": workers, "kind": "reference",
            "cpu_model": cpu_model(),
            "dense_mode_at_s0": {"value": round(fd / sd / 1e9, 3), "unit": "GFLOP/s",
                                 "speedup_of_sparse": round((f / s) / (fd / sd), 3)},
            "sample": f"{n_img} image(s) per layer x {len(ref_layers(args.config))} layers of {args.config} x "
                      f"FWD/BWI/BWW x sparsity {grid} ({f / 1e9:.0f} dense-equiv GFLOP in {s:.1f} s); reference "
                      f"run_parallel, backend automatic, {workers} threads"}


def e2e(args, sp, work, ws, rank, comm=None):
    """Same metric through the host-buffer C ABI (spc_run_parallel_host):
    host inputs -> H2D -> kernels -> D2H of every output, per call; under
    N > 1 each BWW's partial dG is then summed across ranks (H2D, allreduce,
    D2H: counted in the bytes).  Pinned host buffers (the headline) and, for
    one step, pageable ones (what a std::vector caller passes)."""
    import ctypes

    import numpy as np
    import torch
    host, tags = [], []
    h2d = d2h = 0
    pinned = {}  # one host copy per device tensor: a layer's BWI and BWW name the same dY buffer

    def host_copy(t):
        key = t.data.data_ptr()
        if key not in pinned:
            pinned[key] = t.data.cpu().pin_memory().numpy()
        return sp.BlockedTensor(**{**t.header(), "data": pinned[key]})

    fwd_a = {}  # (sparsity tag, layer) -> the FWD pass's ActNCHWc input D on the host
    for (tag, li, name, pp, fl, dgb) in work:
        a, b = host_copy(pp._a), host_copy(pp._b)
        if name == "fwd":
            fwd_a[(tag, li)] = a
        out = torch.empty(pp.out.numel(), dtype=torch.float32).pin_memory().numpy()
        host.append((a, b, pp, out, fl, name))
        tags.append(tag)
        h2d += (a.data.nbytes + b.data.nbytes)
        d2h += out.nbytes + 32
        if comm is not None and name == "bww":
            h2d += out.nbytes
            d2h += out.nbytes
    # the batch call's operands: BWW (check = input) names the layer's ActNCHWc D -- the buffer its FWD pass
    # uploads -- and the library packs ActCHWNn on the device (SPC_PASS_CHECKED_NCHWC); bytes it uploads: every
    # buffer once per window of passes in flight (an activation the previous two passes uploaded is read in place)
    batch_ops, h2d_shared, recent = [], 0, []
    for (a, b, pp, out, fl, name), (tag, li, *_rest) in zip(host, work):
        if name == "bww" and (tag, li) in fwd_a and sp.BwwCheck(pp.plan_obj.check) == sp.BwwCheck.input:
            a = fwd_a[(tag, li)]
        batch_ops.append((a, b))
        seen = set().union(*recent) if recent else set()
        mine = set()
        for t in (a, b):
            key = t.data.ctypes.data
            mine.add(key)
            if key not in seen or t.layout == sp.Layout.filter_kcrs_blk:
                h2d_shared += t.data.nbytes
        recent = (recent + [mine])[-2:]
    L = sp._lib.load()
    scratch = None
    if comm is not None:
        scratch = torch.empty(max(h[3].size for h in host if h[5] == "bww"), dtype=torch.float32, device="cuda")

    def one_step(items):
        for a, b, pp, out, fl, name in items:
            ca, cb = a.to_c(), b.to_c()
            cd = sp._lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.ctypes.data, out.size)
            cnt = sp._lib.spc_counters()
            st = L.spc_run_parallel_host(ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(pp._shape),
                                         ctypes.byref(pp._plan), 0, ctypes.byref(cd), ctypes.byref(cnt))
            if st:
                raise sp.SpconvError(st, sp._lib.last_error())
            if comm is not None and name == "bww":
                d = scratch[:out.size]
                d.copy_(torch.from_numpy(out), non_blocking=True)
                comm.allreduce(d, torch.cuda.current_stream().cuda_stream)
                torch.from_numpy(out).copy_(d)

    def timed(items, steps):
        one_step(items)
        torch.cuda.synchronize()
        if comm is not None:
            import torch.distributed as dist
            dist.barrier()
        per = []
        for _ in range(steps):
            t0 = time.perf_counter()
            one_step(items)
            per.append(time.perf_counter() - t0)
        # median step: the host-buffer path shares PCIe and the host with the box's other tenants, and a
        # single step now and then takes 1.5-3x as long (every step's time is reported)
        secs = sorted(per)[len(per) // 2]
        timed.last = [round(t, 3) for t in per]
        if comm is not None:
            import torch.distributed as dist
            t = torch.tensor([secs], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            secs = float(t.item())
        return secs

    flops = sum(h[4] for h in host)
    secs = timed(host, args.e2e_steps)
    per_call = {"value": round(flops / secs / 1e9, 1), "s_per_step": round(secs, 3), "s_all_steps": timed.last,
                "h2d_bytes_per_step": int(h2d),
                "path": "spc_run_parallel_host, one synchronous call per pass (H2D + kernels + D2H + sync each)"}
    res = {"value": per_call["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "s_per_step": per_call["s_per_step"],
           "path": "spc_run_parallel_host (include/spconv_b200.h), pinned host buffers, per-call H2D+D2H+sync"
                   + ("; BWW dG allreduced across ranks" if comm is not None else "")}
    # the same passes, same host buffers, as ONE spc_run_parallel_host_batch call per step: copies and kernels
    # pipelined across passes (results bitwise those of the per-call form:
    # tests/test_gpu_parity.py::test_host_batch_equals_per_call); under N > 1 each rank runs its shard's batch, then
    # every BWW's partial dG is summed across ranks (H2D, allreduce, D2H), as in the per-call form
    hb = sp.HostBatch()
    for (a, b), (_a, _b, pp, out, fl, name) in zip(batch_ops, host):
        hb.add(a, b, pp.shape_obj, pp.plan_obj, sp.RunMode.sparse, out=out)

    def batch_step():
        hb.run()
        if comm is not None:
            for a, b, pp, out, fl, name in host:
                if name == "bww":
                    d = scratch[:out.size]
                    d.copy_(torch.from_numpy(out), non_blocking=True)
                    comm.allreduce(d, torch.cuda.current_stream().cuda_stream)
                    torch.from_numpy(out).copy_(d)

    batch_step()
    torch.cuda.synchronize()
    if comm is not None:
        import torch.distributed as dist
        dist.barrier()
    per = []
    for _ in range(args.e2e_steps):
        t0 = time.perf_counter()
        batch_step()
        per.append(time.perf_counter() - t0)
    bsecs = sorted(per)[len(per) // 2]
    if comm is not None:
        t = torch.tensor([bsecs], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        bsecs = float(t.item())
    bww_out = sum(h[3].nbytes for h in host if h[5] == "bww") if comm is not None else 0
    res.update({"value": round(flops / bsecs / 1e9, 1), "s_per_step": round(bsecs, 3),
                "s_all_steps": [round(t, 3) for t in per], "statistic": "median step",
                "h2d_bytes_per_step": int(h2d_shared + bww_out),
                "h2d_note": "every distinct input of the step (each layer's D, dY, filter and transposed filter) is "
                            "copied host->device inside the timed region, once: a layer's BWI and BWW name the "
                            "same dY host buffer, and its BWW names the ActNCHWc D its FWD uploads, packed "
                            "into ActCHWNn on the device (SPC_PASS_CHECKED_NCHWC); per_call uploads the "
                            "operands of every call, ActCHWNn D included",
                "path": "spc_run_parallel_host_batch (include/spconv_b200.h): the step's passes in one call, "
                        "pinned host buffers, every input H2D and every output D2H inside the timed region, "
                        "pipelined across passes"
                        + ("; BWW dG allreduced across ranks after the batch" if comm is not None else ""),
                "per_call": per_call})
    del hb
    sp.HostBatch.release()
    # pageable host memory (a std::vector caller): the same calls on the first
    # sparsity's passes (bounded host RAM), one step
    page = []
    for (a, b, pp, out, fl, name), tag in zip(host, tags):
        if tag != tags[0]:
            continue
        pa = sp.BlockedTensor(**{**a.header(), "data": np.array(a.data, copy=True)})
        pb = sp.BlockedTensor(**{**b.header(), "data": np.array(b.data, copy=True)})
        page.append((pa, pb, pp, np.empty_like(out), fl, name))
    pflops = sum(h[4] for h in page)
    del host
    ps = timed(page, 1)
    res["pageable"] = {"value": round(pflops / ps / 1e9, 1), "s_per_step": round(ps, 3),
                       "path": f"same calls with pageable (numpy) host buffers, sparsity {tags[0]} passes only"}
    return res


if __name__ == "__main__":
    main()
