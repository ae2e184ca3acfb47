"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
smoke() (tile FFMA kernels incl. branch + jump-table pairs, 1x1 GEMM kernels,
3xTF32 tcgen05/TMA kernels), the gated host-buffer FWD/BWI path
(SPC_HOST_GATE=1: mapped-memory gate), BWW with a non-finite checked tensor
(exact fallback), and a few passes of every tuned geometry (3x3 s1/s2, 1x1
s1/s2) in both modes.  Sizes are tiny: the sanitizer slows kernels 10-100x."""
import os
import sys

os.environ.setdefault("SPC_HOST_GATE", "1")
os.environ.setdefault("SPC_HOST_CHUNK_MB", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import __graft_entry__ as g  # noqa: E402
import oracle as O  # noqa: E402
import paper_1911_10175_b200 as sp  # noqa: E402


def main():
    g.smoke()
    V = 16
    for dims in [(5, 64, 128, 9, 10, 3, 1), (3, 128, 128, 10, 9, 3, 2), (4, 64, 256, 7, 7, 1, 1),
                 (3, 64, 128, 8, 8, 1, 2)]:
        N, C, K, H, W, R, st = dims
        sh = sp.ConvShape.make(N, C, K, H, W, R, R, st, st)
        D = O.gen_sparse(N, C, H, W, 0.6, 1)
        G = O.gen_sparse(K, C, R, R, 0.0, 2)
        dY = O.gen_sparse(N, K, sh.out_h(), sh.out_w(), 0.5, 3)
        for mode in (sp.RunMode.sparse, sp.RunMode.dense):
            for comp, a, b in ((sp.Component.fwd, sp.pack_act_nchwc(D, V), sp.pack_filter(G, V)),
                               (sp.Component.bwi, sp.pack_act_nchwc(dY, V), sp.pack_filter(G, V, True)),
                               (sp.Component.bww, sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V))):
                pl = sp.plan(sh, comp, V)
                sp.run_parallel(a.to("cuda"), b.to("cuda"), sh, pl, mode)  # device path
                sp.run_parallel(a, b, sh, pl, mode)                         # host path (gated FWD/BWI)
        D[0, 1, 0, 0] = np.inf  # non-finite checked tensor: exact BWW fallback
        sp.run_parallel(sp.pack_act_chwnn(D, V).to("cuda"), sp.pack_act_nchwc(dY, V).to("cuda"), sh,
                        sp.plan(sh, sp.Component.bww, V), sp.RunMode.sparse)
    import torch
    torch.cuda.synchronize()
    print("sanitize workload OK, launches:", sp.launch_count())


if __name__ == "__main__":
    main()
