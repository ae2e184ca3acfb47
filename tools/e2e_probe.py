"""Where the host-buffer path's time goes: per pass, the C-ABI host call vs
its H2D / D2H bytes at the measured PCIe rates and its device kernel time."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl

V = 16
L = sp._lib.load()
g = torch.Generator(device="cuda").manual_seed(0)
layers = wl.CONFIGS["vgg16_b32"]()
st = torch.cuda.current_stream()
LAYERS = [int(x) for x in sys.argv[1:]] or [0, 4, 9]
for li in LAYERS:
    sh = layers[li].shape
    G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
    D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), 0.6, g)
    dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), 0.6, g)
    bD = sp.pack_act_nchwc(D, V)
    ops = {"fwd": (bD, sp.pack_filter(G, V)), "bwi": (sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True)),
           "bww": (sp.nchwc_to_chwnn(bD), sp.pack_act_nchwc(dY, V))}
    for name, (a, b) in ops.items():
        pl = sp.plan(sh, sp.Component[name], V, 30, sp.BwwCheck.input)
        pp = sp.PreparedPass(a, b, sh, pl, sp.RunMode.sparse)
        for _ in range(3):
            pp.launch(st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            pp.launch(st.cuda_stream)
        e1.record()
        torch.cuda.synchronize()
        k_ms = e0.elapsed_time(e1) / 5
        ha = sp.BlockedTensor(**{**a.header(), "data": a.data.cpu().pin_memory().numpy()})
        hb = sp.BlockedTensor(**{**b.header(), "data": b.data.cpu().pin_memory().numpy()})
        out = torch.empty(pp.out.numel(), dtype=torch.float32).pin_memory().numpy()
        ca, cb = ha.to_c(), hb.to_c()
        cd = sp._lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.ctypes.data, out.size)
        cnt = sp._lib.spc_counters()
        call = lambda: L.spc_run_parallel_host(ctypes.byref(ca), ctypes.byref(cb), ctypes.byref(pp._shape),
                                               ctypes.byref(pp._plan), 0, ctypes.byref(cd), ctypes.byref(cnt))
        call()
        t0 = time.perf_counter()
        for _ in range(3):
            assert call() == 0
        host_ms = (time.perf_counter() - t0) / 3 * 1e3
        hin = (ha.data.nbytes + hb.data.nbytes) / 1e9
        hout = out.nbytes / 1e9
        print(f"{layers[li].name:8s} {name}: host call {host_ms:7.2f} ms | kernel {k_ms:6.2f} ms | "
              f"H2D {hin:5.2f} GB -> {hin / 55.5 * 1e3:6.2f} ms | D2H {hout:5.2f} GB -> {hout / 57.2 * 1e3:6.2f} ms",
              flush=True)
