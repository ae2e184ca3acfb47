"""A/B of BWW kernel variants on the VGG16 b32 layers (development tool).

Each variant runs in its own process (the kernel-selection knobs are read
once per process): the parent spawns `--child` runs with the variant's
environment, each prints per-(layer, sparsity) times and compares its dG and
counters with the first variant's (saved under /tmp)."""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

VARIANTS = {
    "tile": {},
    "tma0": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "0"},
    "tma1": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "1"},
    "tma2": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "2"},
    "tma3": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "3"},
    "tma4": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "4"},
    "tma5": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "5"},
    "tma6": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "6"},
    "tma7": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "7"},
    "tma8": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "8"},
    "tma9": {"SPC_TMA_BWW": "1", "SPC_TMA_BWW_CFG": "9"},
    "k2_10": {"SPC_TMA_BWW": "2", "SPC_TMA_BWW_CFG": "10"},
    "k2_11": {"SPC_TMA_BWW": "2", "SPC_TMA_BWW_CFG": "11"},
    "k2_12": {"SPC_TMA_BWW": "2", "SPC_TMA_BWW_CFG": "12"},
    "k2_13": {"SPC_TMA_BWW": "2", "SPC_TMA_BWW_CFG": "13"},
    "k2_14": {"SPC_TMA_BWW": "2", "SPC_TMA_BWW_CFG": "14"},
}


def child(args):
    import torch

    import paper_1911_10175_b200 as sp
    from paper_1911_10175_b200 import workloads as wl

    V = 16
    stream = torch.cuda.current_stream()
    layers = wl.CONFIGS[args.config]()
    for li in args.layers:
        layer = layers[li]
        sh = layer.shape
        flops = sh.dense_flops()
        for s in args.sparsity:
            g = torch.Generator(device="cuda").manual_seed(1000 * li + int(s * 100))
            D = wl.device_activation((sh.N, sh.C, sh.H, sh.W), s, g)
            dY = wl.device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, g)
            a, b = sp.pack_act_chwnn(D, V), sp.pack_act_nchwc(dY, V)
            pl = sp.plan(sh, sp.Component.bww, V, 30, sp.BwwCheck.input)
            row = []
            for mode in (sp.RunMode.sparse, sp.RunMode.dense):
                cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
                pp = sp.PreparedPass(a, b, sh, pl, mode, counters=cnt)
                for _ in range(3):
                    pp.launch(stream.cuda_stream)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for _ in range(args.reps):
                    pp.launch(stream.cuda_stream)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1) / args.reps
                cnt.zero_()
                pp.launch(stream.cuda_stream)
                torch.cuda.synchronize()
                out = pp.out.clone()
                tag = f"/tmp/bww_ab_{args.config}_{li}_{s}_{int(mode)}.pt"
                chk = ""
                if args.save:
                    torch.save((out.cpu(), cnt.cpu()), tag)
                elif os.path.exists(tag):
                    ref, rc = torch.load(tag)
                    ref = ref.cuda()
                    err = ((out - ref).abs().max() / ref.abs().max()).item()
                    same = bool((cnt.cpu() == rc).all())
                    chk = f" err {err:.1e} cnt {'ok' if same else 'DIFF'}"
                row.append(f"{'sparse' if mode == sp.RunMode.sparse else 'dense'} {t*1e3:7.1f}us "
                           f"{flops/t/1e9:6.1f}TF{chk}")
            print(f"  {layer.name:9s} s={s:.1f} " + " | ".join(row), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="vgg16_b32")
    ap.add_argument("--layers", type=int, nargs="+", default=[2, 4, 7, 10])
    ap.add_argument("--sparsity", type=float, nargs="+", default=[0.4, 0.9])
    ap.add_argument("--variants", nargs="+", default=["tile", "tma0"])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--save", action="store_true")
    args = ap.parse_args()
    if args.child:
        return child(args)
    for i, v in enumerate(args.variants):
        env = dict(os.environ)
        env.update(VARIANTS[v])
        print(f"== {v} {VARIANTS[v]}", flush=True)
        cmd = [sys.executable, os.path.abspath(__file__), "--child", "--config", args.config, "--reps", str(args.reps),
               "--layers", *map(str, args.layers), "--sparsity", *map(str, args.sparsity)]
        if i == 0:
            cmd.append("--save")
        subprocess.run(cmd, env=env, timeout=900)


if __name__ == "__main__":
    main()
