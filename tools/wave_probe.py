"""Wave-quantisation probe (development tool): per-image time of one sparse pass vs batch size.

If a launch's CTAs run in whole waves, time(N) steps up at wave boundaries instead of growing
linearly with N.  Usage: python tools/wave_probe.py [--sparsity 0.6] [--comps fwd bwi bww]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl
from tools.kbench import time_pass


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sparsity", type=float, default=0.6)
    ap.add_argument("--comps", nargs="+", default=["fwd", "bwi", "bww"])
    ap.add_argument("--batches", type=int, nargs="+", default=[24, 26, 28, 30, 31, 32, 33, 34, 36])
    ap.add_argument("--layers", nargs="+", default=["conv3_2", "conv4_2", "conv5_2"])
    args = ap.parse_args()
    V = 16
    g = torch.Generator(device="cuda").manual_seed(0)
    stream = torch.cuda.current_stream()
    base = {l.name: l.shape for l in wl.vgg16(32)}
    for name in args.layers:
        s0 = base[name]
        G = wl.device_weights(s0.K, s0.C, s0.S, s0.R, g)
        for N in args.batches:
            sh = sp.ConvShape.make(N, s0.C, s0.K, s0.H, s0.W, s0.R, s0.S, 1, 1)
            D = wl.device_activation((N, sh.C, sh.H, sh.W), args.sparsity, g)
            dY = wl.device_grad((N, sh.K, sh.out_h(), sh.out_w()), args.sparsity, g)
            ops = {
                "fwd": (sp.pack_act_nchwc(D, V), sp.pack_filter(G, V), sp.BwwCheck.input),
                "bwi": (sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True), sp.BwwCheck.input),
                "bww": (sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V), sp.BwwCheck.input),
            }
            row = []
            for comp_name in args.comps:
                a, b, chk = ops[comp_name]
                pl = sp.plan(sh, sp.Component[comp_name], V, 30, chk)
                t = time_pass(sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse), stream)
                row.append(f"{comp_name} {t * 1e3:8.1f}us {t * 1e3 / N:6.2f}us/img")
            print(f"{name} N={N:3d} " + " | ".join(row), flush=True)


if __name__ == "__main__":
    main()
