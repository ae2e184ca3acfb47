"""Time tile-kernel variants (spc_debug_conv_variant) on one layer at several
sparsities; checks each variant's output against the default kernel."""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="vgg16_b32")
ap.add_argument("--layers", type=int, nargs="+", default=[4])
ap.add_argument("--comp", default="fwd")
ap.add_argument("--sparsity", type=float, nargs="+", default=[0.0, 0.6, 0.9])
ap.add_argument("--variants", type=int, nargs="+", default=list(range(14)))
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--check", default="input")
a = ap.parse_args()
L = sp._lib.load()
V = 16
g = torch.Generator(device="cuda").manual_seed(0)
st = torch.cuda.current_stream()
for li in a.layers:
    sh = wl.CONFIGS[a.config]()[li].shape
    G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
    for s in a.sparsity:
        chk = sp.BwwCheck[a.check]
        if a.comp == "fwd":
            x = sp.pack_act_nchwc(wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, g), V)
            y = sp.pack_filter(G, V)
        elif a.comp == "bww":
            Dd = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, g)
            dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, g)
            x, y = ((sp.pack_act_chwnn(Dd, V), sp.pack_act_nchwc(dY, V)) if chk == sp.BwwCheck.input
                    else (sp.pack_act_nchwc(Dd, V), sp.pack_act_chwnn(dY, V)))
        else:
            x = sp.pack_act_nchwc(wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, g), V)
            y = sp.pack_filter(G, V, True)
        pl = sp.plan(sh, sp.Component[a.comp], V, 30, chk)
        mode = 1 if s == 0.0 else 0
        ref = sp.PreparedPass(x, y, sh, pl, sp.RunMode(mode))
        ref.launch(st.cuda_stream)
        row = []
        for v in a.variants:
            out = torch.empty_like(ref.out)
            ca, cb, cs, cp = x.to_c(), y.to_c(), sh.to_c(), pl.to_c()
            cd = sp._lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.data_ptr(), out.numel())

            def go():
                return L.spc_debug_conv_variant(v, C.byref(ca), C.byref(cb), C.byref(cs), C.byref(cp), mode,
                                                C.byref(cd), None, C.c_void_p(st.cuda_stream))
            if go():
                row.append(f"v{v}: n/a")
                continue
            for _ in range(2):
                go()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                go()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            err = ((out - ref.out).abs().max() / ref.out.abs().max()).item()
            row.append(f"v{v}: {sh.dense_flops() / ms / 1e9:5.1f}{'!' if err > 1e-5 else ''}")
        print(f"L{li} {a.comp} s={s:.1f} {'dense' if mode else 'sparse'} | " + "  ".join(row), flush=True)
