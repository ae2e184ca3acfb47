"""Zero-skip vs counted-dense on the geometries where the product executes
every FMA: 1x1 FWD / BWI / BWW and 3x3 stride-2 FWD, at the
sparsities of the ResNet configs (0.5 / 0.7 / 0.9).  One line per (layer,
pass, sparsity, variant) with the CUDA-event time; run it under each variant
knob:
    default               counted-dense (pw_gemm / pw_bww / JT=200 tile kernel)
    SPC_PW_GEMM=0         1x1: lane-per-channel kernel skipping all-zero 4-channel quads
    SPC_PW_OFF=1          1x1: the 3x3 tile kernel's per-pixel uniform branches
    SPC_FORCE_SKIP=1      3x3 s2 FWD: per-pixel uniform branches
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1911_10175_b200 as sp  # noqa: E402
from paper_1911_10175_b200 import workloads as wl  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from kbench import time_pass  # noqa: E402

LAYERS = {"s1b1expand": 3, "s1b2reduce": 4, "s3b2reduce": 27, "s2proj": 12, "s2b1conv3": 11, "s3b1conv3": 24}


def main():
    tag = sys.argv[1] if len(sys.argv) > 1 else "default"
    V = 16
    g = torch.Generator(device="cuda").manual_seed(0)
    st = torch.cuda.current_stream()
    layers = wl.resnet50(64)
    for name, idx in LAYERS.items():
        L = layers[idx]
        sh = L.shape
        assert L.name == name, (L.name, name)
        G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
        for s in (0.5, 0.7, 0.9):
            D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, g)
            dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, g)
            ops = {"fwd": (sp.pack_act_nchwc(D, V), sp.pack_filter(G, V)),
                   "bwi": (sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True)),
                   "bww": (sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V))}
            passes = ["fwd"] if sh.R == 3 else ["fwd", "bwi", "bww"]
            for p in passes:
                a, b = ops[p]
                pl = sp.plan(sh, sp.Component[p], V)
                ms = time_pass(sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse), st)
                print(f"{tag:14s} {name:11s} {sh.R}x{sh.R} s{sh.O} {p} s={s:.1f} {ms * 1e3:8.1f} us "
                      f"{sh.dense_flops() / ms / 1e9:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
