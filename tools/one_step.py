"""One bench step (VGG16 b32: 4 sparsities x 12 layers x FWD/BWI/BWW, the exact
passes bench.py times), run once -- for the ncu launch list under profiles/."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl

V = 16
# `python tools/one_step.py tf32x3`: the same step with the 3xTF32 tensor-core variant
if len(sys.argv) > 1:
    sp.set_math(sp.Math[sys.argv[1]])
gen = torch.Generator(device="cuda").manual_seed(1000)
work = []
for s in (0.4, 0.6, 0.8, 0.9):
    for layer in wl.CONFIGS["vgg16_b32"]():
        sh = layer.shape
        G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, gen)
        D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, gen)
        dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, gen)
        bD, bY = sp.pack_act_nchwc(D, V), sp.pack_act_nchwc(dY, V)
        ops = {"fwd": (bD, sp.pack_filter(G, V)), "bwi": (bY, sp.pack_filter(G, V, True)),
               "bww": (sp.nchwc_to_chwnn(bD), bY)}
        for name, (a, b) in ops.items():
            pl = sp.plan(sh, sp.Component[name], V, 30, sp.BwwCheck.input)
            work.append(sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse))
torch.cuda.synchronize()
n0 = sp.launch_count()
st = torch.cuda.current_stream().cuda_stream
for pp in work:
    pp.launch(st)
torch.cuda.synchronize()
print("one step:", len(work), "passes,", sp.launch_count() - n0, "launches", file=sys.stderr)
