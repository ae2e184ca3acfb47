"""The product's NCCL path (csrc/comm.cu) on the GPU: a communicator made
through the C ABI (unique id over torch.distributed), dG in an NCCL symmetric
window, spc_bww_sharded == spc_sparse_bww + allreduce, counters summed.
Runs under torchrun with as many ranks as there are GPUs (1 on the test box:
the collective degenerates to a copy, but every entry point executes)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import ctypes as C, os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, os.environ["ROOT"])
import oracle as O
import paper_1911_10175_b200 as sp
from paper_1911_10175_b200.dist import Comm, ShardPlan
rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
comm = Comm()
L = sp._lib.load()
assert L.spc_nccl_version() >= 22700, L.spc_nccl_version()
V = 16
N = 2 * max(ws, 3) + 1
gsh = sp.ConvShape.make(N, 64, 128, 14, 14, 3, 3, 1, 1)
plan = ShardPlan(N, ws, rank)
sh = plan.shape(gsh)
D = O.gen_sparse(N, 64, 14, 14, 0.7, 5)
dY = O.gen_sparse(N, 128, 14, 14, 0.5, 6)
a = sp.pack_act_chwnn(plan.slice_plain(D), V).to("cuda")
b = plan.slice_nchwc(sp.pack_act_nchwc(dY, V)).to("cuda")
pl = sp.plan(sh, sp.Component.bww, V)
n = 128 * 64 * 9
win, sym = comm.window(n)
cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
cd = sp._lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, win.data_ptr(), n)
st = L.spc_bww_sharded(comm.h, C.byref(a.to_c()), C.byref(b.to_c()), C.byref(sh.to_c()), C.byref(pl.to_c()), 0,
                       C.byref(cd), C.c_void_p(cnt.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
assert st == 0, sp._lib.last_error()
torch.cuda.synchronize()
# read the window (a raw device pointer) back with the CUDA runtime torch loaded
import ctypes
got_ptr = win.data_ptr()
host = np.empty(n, np.float32)
rt = ctypes.CDLL("libcudart.so.12")
assert rt.cudaMemcpy(ctypes.c_void_p(host.ctypes.data), ctypes.c_void_p(got_ptr), ctypes.c_size_t(4 * n), 2) == 0
blk = sp.BlockedTensor(sp.Layout.filter_kcrs_blk, V, k=128, c=64, s=3, r=3, data=host)
dG = sp.unpack(blk)
ref = O.dense(2, gsh.astuple(), D, dY)
err = O.max_abs_rel(dG, ref)
want = O.expected_counts(gsh.astuple(), O.plan(gsh.astuple(), 2, V), D)["executed_vector_fmas"]
c = cnt.cpu().numpy().view(np.uint64)
if rank == 0:
    print(f"ranks={ws} symmetric={sym} err={err:.2e} exec={int(c[1])} want={want}")
assert err <= 1e-5, err
assert int(c[1]) == want
# plain allreduce of a torch tensor through spc_bww_allreduce
t = torch.full((1000,), float(rank + 1), device="cuda")
comm.allreduce(t, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
assert torch.all(t == ws * (ws + 1) / 2)
dist.barrier()
comm.close()
dist.destroy_process_group()
print("ok")
'''


def test_product_comm_sharded_bww_matches_full_batch(tmp_path):
    import torch
    n = max(1, min(torch.cuda.device_count(), 8))
    script = tmp_path / "comm_check.py"
    script.write_text(SCRIPT)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", "--master-port=29517", str(script)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=dict(os.environ, ROOT=ROOT))
    print(r.stdout[-2000:])
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-4000:]
