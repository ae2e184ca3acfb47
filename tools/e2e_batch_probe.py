"""e2e through spc_run_parallel_host_batch on the VGG16 b32 sweep (one sparsity), for tuning
SPC_BATCH_SLOTS / SPC_BATCH_CHUNK_MB (read once per process: run one setting per process)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1911_10175_b200 as sp
from paper_1911_10175_b200 import workloads as wl

V = 16
g = torch.Generator(device="cuda").manual_seed(0)
hb = sp.HostBatch()
flops = 0
nbytes = 0
pin = lambda t: sp.BlockedTensor(**{**t.header(), "data": t.data.cpu().pin_memory().numpy()})
for layer in wl.CONFIGS["vgg16_b32"]():
    sh = layer.shape
    G = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
    D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), 0.6, g)
    dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), 0.6, g)
    bD = sp.pack_act_nchwc(D, V)
    bdY = sp.pack_act_nchwc(dY, V)
    ops = {"fwd": (pin(bD), pin(sp.pack_filter(G, V))), "bwi": (pin(bdY), pin(sp.pack_filter(G, V, True))),
           "bww": (pin(sp.nchwc_to_chwnn(bD)), pin(bdY))}
    for name, (a, b) in ops.items():
        pl = sp.plan(sh, sp.Component[name], V, 30, sp.BwwCheck.input)
        _, numel = sp.api.output_desc(sh, pl)
        out = torch.empty(numel, dtype=torch.float32).pin_memory().numpy()
        hb.add(a, b, sh, pl, sp.RunMode.sparse, out=out)
        flops += sh.dense_flops()
        nbytes += a.data.nbytes + b.data.nbytes + out.nbytes
    del D, dY, bD, bdY
torch.cuda.empty_cache()
hb.run()
ts = []
for _ in range(6):
    t0 = time.perf_counter()
    hb.run()
    ts.append(time.perf_counter() - t0)
print("per run ms:", [round(t * 1e3, 1) for t in ts], flush=True)
s = sorted(ts)[len(ts) // 2]
print(f"slots {os.environ.get('SPC_BATCH_SLOTS', 'default')} chunk {os.environ.get('SPC_BATCH_CHUNK_MB', 'default')}: "
      f"{s*1e3:.1f} ms per quarter step, {flops/s/1e12:.2f} TF/s, {nbytes/s/1e9:.1f} GB/s PCIe (both directions)", flush=True)
