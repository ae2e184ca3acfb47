"""Quick per-layer kernel timing (development tool, not the bench contract)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl


def time_pass(pp, stream, reps=10, warm=3):
    for _ in range(warm):
        pp.launch(stream.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        pp.launch(stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1_single3x3_b16")
    ap.add_argument("--sparsity", type=float, nargs="+", default=[0.5])
    ap.add_argument("--layers", type=int, default=99)
    ap.add_argument("--bww-check", default="input")
    ap.add_argument("--math", default="fp32", choices=["fp32", "tf32x3"])
    ap.add_argument("--comps", nargs="+", default=["fwd", "bwi", "bww"])
    ap.add_argument("--config-layers", type=int, nargs="*", default=None, help="layer indices to run")
    args = ap.parse_args()
    sp.set_math(sp.Math[args.math])
    V = 16
    g = torch.Generator(device="cuda").manual_seed(0)
    stream = torch.cuda.current_stream()
    layers = wl.CONFIGS[args.config]()[: args.layers]
    if args.config_layers:
        layers = [layers[i] for i in args.config_layers]
    for layer in layers:
        sh = layer.shape
        flops = sh.dense_flops()
        G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
        for s in args.sparsity:
            D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, g)
            dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, g)
            ops = {
                "fwd": (sp.pack_act_nchwc(D, V), sp.pack_filter(G, V), sp.BwwCheck.input),
                "bwi": (sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True), sp.BwwCheck.input),
                "bww": ((sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V), sp.BwwCheck.input) if args.bww_check == "input" else (sp.pack_act_nchwc(D, V), sp.pack_act_chwnn(dY, V), sp.BwwCheck.output_grad)),
            }
            row = []
            for name, (a, b, chk) in ops.items():
                if name not in args.comps:
                    continue
                comp = sp.Component[name]
                pl = sp.plan(sh, comp, V, 30, chk)
                t_s = time_pass(sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse), stream)
                t_d = time_pass(sp.PreparedPass(a, b, sh, pl, sp.RunMode.dense), stream)
                row.append(f"{name}: sparse {t_s*1e3:8.1f}us {flops/t_s/1e9:7.1f} TF/s | dense {t_d*1e3:8.1f}us "
                           f"{flops/t_d/1e9:7.1f} TF/s")
            print(f"{layer.name:10s} s={s:.1f} " + " || ".join(row), flush=True)


if __name__ == "__main__":
    main()
