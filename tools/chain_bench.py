"""Fixup ResNet-50 training-step benchmark (BASELINE cfg 5) through the layer
chain (paper_1911_10175_b200/chain.py): FWD + BWI + BWW of all 52 convs with
fused ReLU epilogues, batch-sharded, per-block dG allreduce over NCCL.

    python tools/chain_bench.py --batch 256 --steps 3
    torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/chain_bench.py --batch 256

Prints one JSON line (rank 0).  `value` = dense-equivalent GFLOP/s of the whole
job (all ranks' passes / max-over-ranks step time, CUDA events); strong scaling
(the global batch is fixed and sharded).  `--profile` adds a per-pass-family
time breakdown from one extra single-rank step.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
_OUT = os.dup(1)
os.dup2(2, 1)  # native banners to stderr; the result line to the real stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256, help="global batch (sharded over ranks)")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--scale", type=float, default=0.25, help="Fixup branch multiplier")
    ap.add_argument("--mode", default="sparse", choices=["sparse", "dense"])
    ap.add_argument("--x-sparsity", type=float, default=0.7)
    ap.add_argument("--profile", action="store_true")
    ap.add_argument("--math", default="fp32", choices=["fp32", "tf32x3"])
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    import paper_1911_10175_b200 as sp
    from paper_1911_10175_b200 import chain as CH
    from paper_1911_10175_b200.dist import Comm, CommAllreduce, shard_range

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    distributed = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    if distributed:
        dist.init_process_group("nccl", device_id=dev)
    sp.set_math(sp.Math[a.math])
    _, n_local = shard_range(a.batch, ws, rank)
    t0 = time.time()
    # the product's NCCL communicator (csrc/comm.cu): per-block dG allreduce on a side stream
    comm = Comm() if distributed else None
    ar = CommAllreduce(comm, dev) if comm is not None else None
    # one seed on every rank: the same weights, each rank its slice of the global batch
    ch = CH.fixup_resnet50(a.batch, scale=a.scale, seed=1234, mode=sp.RunMode[a.mode], allreduce=ar,
                           x_sparsity=a.x_sparsity, world=ws, rank=rank)
    st = torch.cuda.current_stream()
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    for _ in range(a.warmup):
        ch.step(st)
    torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    launches0 = sp.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.steps):
        ch.step(st)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    if distributed:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / a.steps
    total_flops = float(ch.global_dense_flops())
    rep = ch.sparsity_report()
    out = {"metric": "dense-equiv GFLOP/s per training step (FWD+BWI+BWW, all convs)",
           "value": round(total_flops / (ms_step * 1e-3) / 1e9, 1), "unit": "GFLOP/s", "n_gpus": ws,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
           "scaling": "strong", "dtype": "f32", "data": "synthetic (seeded He weights, ReLU(N(-t,1)) input)",
           "config": {"workload": "fixup_resnet50: 16 bottlenecks, 52 convs x FWD/BWI/BWW, 224x224",
                      "global_batch": a.batch, "per_gpu_batch": n_local, "mode": a.mode,
                      "fixup": f"calibrated scalar biases (0.7 target), branch multiplier {a.scale}, residual add, "
                               "ReLU (fused epilogues)",
                      "bww_check": "input", "parallelism": f"dp{ws} (batch-sharded, per-block dG allreduce)"},
           "gpu_launches": int((sp.launch_count() - launches0) / a.steps),
           "activation_sparsity_mean": round(rep["activation_sparsity_mean"], 4),
           "gradient_sparsity_mean": round(rep["gradient_sparsity_mean"], 4),
           "passes_per_step": len(ch.passes), "setup_s": round(setup_s, 1)}
    if a.profile and not distributed:
        out["breakdown_ms"] = profile(ch, st, torch)
    if rank == 0:
        os.write(_OUT, (json.dumps(out) + "\n").encode())
    if distributed:
        dist.barrier()
        comm.close()
        dist.destroy_process_group()


def profile(ch, st, torch):
    """Per-family time of one step: every launchable timed with its own events."""
    from paper_1911_10175_b200.api import PreparedPass
    items = [("fwd", p) for p in ch._fwd]
    items.append(("mask", ch._mask_last))
    for seq, _, _ in ch._bwd_blocks:
        items += [("bwd", p) for p in seq]
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in items]
    for (e0, e1), (_, p) in zip(ev, items):
        e0.record(st)
        p.launch(st.cuda_stream)
        e1.record(st)
    torch.cuda.synchronize()
    fam = {}
    for (e0, e1), (phase, p) in zip(ev, items):
        if isinstance(p, PreparedPass):
            comp = ["fwd", "bwi", "bww"][int(p._plan.comp)]
            sh = p._shape
            key = f"{comp} {sh.R}x{sh.S} s{sh.O}"
        else:
            key = type(p).__name__.strip("_").lower()
        fam[key] = fam.get(key, 0.0) + e0.elapsed_time(e1)
    return {k: round(v, 3) for k, v in sorted(fam.items(), key=lambda kv: -kv[1])}


if __name__ == "__main__":
    main()
