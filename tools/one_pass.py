"""Run one pass of one layer a few times (for ncu / compute-sanitizer)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg1_single3x3_b16")
ap.add_argument("--layer", type=int, default=0)
ap.add_argument("--comp", default="fwd")
ap.add_argument("--check", default="input")
ap.add_argument("--sparsity", type=float, default=0.5)
ap.add_argument("--mode", default="sparse")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--math", default="fp32", choices=["fp32", "tf32x3"])
a = ap.parse_args()
sp.set_math(sp.Math[a.math])
V = 16
sh = wl.CONFIGS[a.config]()[a.layer].shape
if a.batch:
    sh = sh.with_batch(a.batch)
g = torch.Generator(device="cuda").manual_seed(0)
G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), a.sparsity, g)
dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), a.sparsity, g)
chk = sp.BwwCheck[a.check]
if a.comp == "fwd":
    x, y = sp.pack_act_nchwc(D, V), sp.pack_filter(G, V)
elif a.comp == "bwi":
    x, y = sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True)
elif chk == sp.BwwCheck.input:
    x, y = sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V)
else:
    x, y = sp.pack_act_nchwc(D, V), sp.pack_act_chwnn(dY, V)
pl = sp.plan(sh, sp.Component[a.comp], V, 30, chk)
pp = sp.PreparedPass(x, y, sh, pl, sp.RunMode[a.mode])
torch.cuda.synchronize()
for _ in range(a.reps):
    pp.launch(torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", sh, a.comp, a.mode, a.sparsity)
