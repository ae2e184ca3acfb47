"""Layer chains: a whole ResNet-50 bottleneck stack (Fixup form) trained step
by step through the sparse FWD/BWI/BWW passes, on device, batch-sharded.

SURVEY.md section 8(f)2 / BASELINE cfg 5 ("Fixup ResNet-50 ... full
non-initial conv stack run FWD+BWI+BWW, batch-sharded ... with the BWW
weight-gradient NCCL allreduce").  The reference has no network-level driver
(its registry is per layer, P/src/bench.cpp:21-52); this one strings the
reference-semantics passes together with the fused epilogues
(include/spconv_b200.h spc_epilogue), so every ReLU mask comes from the
forward pass itself and no tensor leaves the GPU:

  block(x):  a   = relu(conv1x1(x))                      FWD, epilogue relu
             b   = relu(conv3x3_s(a))                    FWD, epilogue relu
             sc  = x  or  conv1x1_s(x)  (projection)     FWD
             out = relu(scale * conv1x1(b) + sc)         FWD, epilogue alpha/add/relu

  backward, dz = dL/dz with z = scale*c + sc (already masked by out > 0):
             dG3 = scale * BWW(b, dz)                     BWW + standalone epilogue
             db  = (b > 0) ? scale * BWI3(dz) : 0         BWI, epilogue alpha/mask
             dG2 = BWW(a, db);  da = (a > 0) ? BWI2(db) : 0
             dG1 = BWW(x, da);  dGp = BWW(x, dz) [projection]
             dz' = (x > 0) ? BWI1(da) + (dz or BWIp(dz)) : 0    BWI, epilogue add/mask

Fixup details: one scalar multiplier per residual branch, and a scalar bias
before each ReLU (fused as the epilogue's `beta`):
    a = relu(conv1(x) + b1), b = relu(conv2(a) + b2), out = relu(scale*conv3(b) + sc + b3).
BASELINE cfg 5 asks for "ReLU masks from a seeded forward pass with ~0.7 mean
activation sparsity"; with He-normal weights and zero biases the pre-
activations are centred and ReLU zeroes only ~half of them, so the biases
are CALIBRATED on that seeded forward pass: each is minus the
`target_sparsity` quantile of its pre-activation over the first
`calib_images` images of the global batch (rank 0 computes them and, under
torch.distributed, broadcasts them, so every rank -- and every world size --
runs the same network).  BWW checks the input side (ActCHWNn copies made on
device per layer, P/src/tensor.cpp:94-108).  Each block's weight gradients
are summed across ranks (NCCL on a side stream) as soon as its BWW passes
are enqueued, overlapping the rest of the backward pass.

Data parallelism: the global batch `N` is generated once from `seed` and
each rank keeps its contiguous slice (``dist.shard_range``); the weights come
from the same seed on every rank, so a multi-rank step equals the
single-rank full-batch step up to the summation order of dG.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math

from . import _lib
from .api import (BlockedTensor, BwwCheck, Component, ConvShape, Epilogue, Layout, PreparedPass, RunMode,
                  SpconvError, output_desc, plan)


@dataclasses.dataclass(frozen=True)
class Bottleneck:
    cin: int
    width: int
    stride: int
    H: int  # input resolution
    W: int

    @property
    def proj(self) -> bool:
        return self.stride != 1 or self.cin != 4 * self.width


def resnet50_blocks(H=56, W=56, cin=64, stages=((64, 3), (128, 4), (256, 6), (512, 3))) -> list[Bottleneck]:
    """ResNet-50 v1.5 bottlenecks (stride 2 on the first 3x3 of stages 2-4),
    the same 52 conv shapes as workloads.resnet50."""
    out = []
    for si, (width, nb) in enumerate(stages):
        for bi in range(nb):
            s = 2 if (bi == 0 and si > 0) else 1
            out.append(Bottleneck(cin, width, s, H, W))
            cin = 4 * width
            H, W = (H - 1) // s + 1, (W - 1) // s + 1
    return out


class _Transpose:
    """ActNCHWc -> ActCHWNn into a preallocated buffer, launchable on a stream."""

    def __init__(self, src: BlockedTensor, out):
        V = src.V
        self.dst = BlockedTensor(Layout.act_chwnn, V, src.n, src.c, src.h, src.w, data=out)
        self._cs = src.to_c()
        self._cd = _lib.spc_tensor(0, 0, 0, 0, 0, 0, 0, 0, 0, out.data_ptr(),
                                   ((src.n + V - 1) // V) * src.c * src.h * src.w * V)
        self._keep = (src, out)

    def launch(self, stream_ptr: int) -> None:
        st = _lib.load().spc_nchwc_to_chwnn(C.byref(self._cs), C.byref(self._cd), C.c_void_p(stream_ptr))
        if st:
            raise SpconvError(st, _lib.last_error())


class _Scale:
    """In-place standalone epilogue (alpha) over a device buffer."""

    def __init__(self, alpha: float, buf):
        self._e = Epilogue(alpha=alpha).to_c()
        self._buf = buf

    def launch(self, stream_ptr: int) -> None:
        st = _lib.load().spc_epilogue_apply(C.byref(self._e), C.c_void_p(self._buf.data_ptr()), self._buf.numel(),
                                            C.c_void_p(stream_ptr))
        if st:
            raise SpconvError(st, _lib.last_error())


@dataclasses.dataclass
class ConvRecord:
    name: str
    shape: ConvShape
    fwd_input: str  # which tensor feeds it (for sparsity reports)


class FixupChain:
    """Preallocated, device-resident training step of a bottleneck stack.

    ``step(stream)`` enqueues FWD through all blocks, the upstream gradient
    mask, then BWI/BWW in reverse with per-block dG allreduce; nothing
    synchronises the host.  ``passes`` lists every launched conv pass with
    its shape for FLOP accounting; ``grads`` is the flat dG buffer (one
    FilterKCRSblk (K, C) slice per conv, in ``convs`` order)."""

    def __init__(self, N: int, blocks: list[Bottleneck], scale: float = 0.25, seed: int = 0, V: int = 16,
                 device="cuda", mode: RunMode = RunMode.sparse, allreduce=None, x_sparsity: float = 0.7,
                 target_sparsity: float | None = 0.7, calib_images: int = 8, world: int = 1, rank: int = 0,
                 bias: dict | None = None):
        import torch
        from . import workloads as wl
        from .dist import shard_range
        self.torch = torch
        self.N_global = N
        self.shard = shard_range(N, world, rank)
        N = self.shard[1]
        self.N, self.blocks, self.scale, self.V, self.mode = N, blocks, scale, V, mode
        self.allreduce = allreduce
        g = torch.Generator(device=device).manual_seed(seed)
        self.gen = g
        self.convs: list[ConvRecord] = []
        self.passes: list[tuple[str, Component, ConvShape]] = []
        self._fwd: list = []     # launchables in order
        self._bwd: list = []     # list per block (reverse order filled later)
        mk = ConvShape.make

        def filt(sh):
            Gp = wl.device_weights(sh.K, sh.C, sh.S, sh.R, g)
            from .api import pack_filter
            return pack_filter(Gp, V), pack_filter(Gp, V, True), Gp

        # ---- shapes and weights
        specs = []
        for bi, b in enumerate(blocks):
            Ho, Wo = (b.H - 1) // b.stride + 1, (b.W - 1) // b.stride + 1
            s1 = mk(N, b.cin, b.width, b.H, b.W, 1, 1, 1, 1)
            s2 = mk(N, b.width, b.width, b.H, b.W, 3, 3, b.stride, b.stride)
            s3 = mk(N, b.width, 4 * b.width, Ho, Wo, 1, 1, 1, 1)
            sp_ = mk(N, b.cin, 4 * b.width, b.H, b.W, 1, 1, b.stride, b.stride) if b.proj else None
            if sp_ is not None:
                assert (sp_.out_h(), sp_.out_w()) == (Ho, Wo)
            specs.append((s1, s2, s3, sp_))
        self.weights = {}
        names = []
        for bi, (s1, s2, s3, sp_) in enumerate(specs):
            for tag, sh in (("c1", s1), ("c2", s2), ("c3", s3), ("proj", sp_)):
                if sh is None:
                    continue
                name = f"b{bi}.{tag}"
                names.append((name, sh))
                self.weights[name] = filt(sh)
        # flat dG buffer
        sizes = [sh.K * sh.C * sh.S * sh.R for _, sh in names]
        self.grads = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
        self.grad_slice = {}
        off = 0
        for (name, sh), n in zip(names, sizes):
            self.grad_slice[name] = self.grads[off:off + n]
            off += n

        # ---- activations: network input x0 = ReLU(N(-t,1)) at x_sparsity, the
        # whole global batch from the seed, this rank's slice kept
        b0 = blocks[0]
        x0 = wl.device_activation((self.N_global, b0.cin, b0.H, b0.W), x_sparsity, g)
        x0 = x0[self.shard[0]:self.shard[0] + N].contiguous()
        from .api import pack_act_nchwc
        self.x0 = pack_act_nchwc(x0, V)
        del x0
        x = self.x0
        self.acts = []  # per block: dict of BlockedTensors
        self._relu_passes = []  # (conv name, FWD pass with a ReLU epilogue) in forward order
        max_chwnn = 0
        for bi, (b, (s1, s2, s3, sp_)) in enumerate(zip(blocks, specs)):
            G1, G2, G3 = self.weights[f"b{bi}.c1"], self.weights[f"b{bi}.c2"], self.weights[f"b{bi}.c3"]
            p1 = PreparedPass(x, G1[0], s1, plan(s1, Component.fwd, V), mode, epilogue=Epilogue(relu=True))
            a = p1.desc
            p2 = PreparedPass(a, G2[0], s2, plan(s2, Component.fwd, V), mode, epilogue=Epilogue(relu=True))
            self._relu_passes += [(f"b{bi}.c1", p1), (f"b{bi}.c2", p2)]
            bt = p2.desc
            launch = [p1, p2]
            if sp_ is not None:
                Gp = self.weights[f"b{bi}.proj"]
                pp = PreparedPass(x, Gp[0], sp_, plan(sp_, Component.fwd, V), mode)
                sc = pp.desc
                launch.append(pp)
                self.passes.append((f"b{bi}.proj", Component.fwd, sp_))
            else:
                sc = x
            p3 = PreparedPass(bt, G3[0], s3, plan(s3, Component.fwd, V), mode,
                              epilogue=Epilogue(alpha=scale, add=sc.data, relu=True))
            out = p3.desc
            launch.append(p3)
            self._relu_passes.append((f"b{bi}.c3", p3))
            self._fwd += launch
            for nm, sh in (("c1", s1), ("c2", s2), ("c3", s3)):
                self.passes.append((f"b{bi}.{nm}", Component.fwd, sh))
            self.acts.append(dict(x=x, a=a, b=bt, sc=sc, out=out, s1=s1, s2=s2, s3=s3, sp=sp_))
            for t in (x, a, bt):
                max_chwnn = max(max_chwnn, ((t.n + V - 1) // V) * t.c * t.h * t.w * V)
            x = out
        self.out = x
        self.bias = {name: 0.0 for name, _ in self._relu_passes}
        if bias is not None:  # given (e.g. another rank's calibration)
            for name, p in self._relu_passes:
                self.bias[name] = float(bias[name])
                p._epi.beta = self.bias[name]
        elif target_sparsity is not None:
            self._calibrate(target_sparsity, calib_images, device)

        # ---- backward
        self.chwnn = torch.empty(max_chwnn, dtype=torch.float32, device=device)
        last = self.acts[-1]["out"]
        self.dout = torch.empty_like(last.data)  # upstream gradient w.r.t. the last block output
        self.dz_last = BlockedTensor(Layout.act_nchwc, V, last.n, last.c, last.h, last.w,
                                     data=torch.empty_like(last.data))
        # dz_last = (out > 0) ? dout : 0
        self._mask_last = _MaskedCopy(self.dout, last.data, self.dz_last.data)
        self._bwd_blocks = []
        dz = self.dz_last
        for bi in reversed(range(len(blocks))):
            A = self.acts[bi]
            s1, s2, s3, sp_ = A["s1"], A["s2"], A["s3"], A["sp"]
            G1, G2, G3 = self.weights[f"b{bi}.c1"], self.weights[f"b{bi}.c2"], self.weights[f"b{bi}.c3"]
            seq = []
            # conv3: dG3 = scale * BWW(b, dz); db = (b > 0) ? scale * BWI(dz) : 0
            tb = _Transpose(A["b"], self.chwnn[:_chwnn_numel(A["b"])])
            w3 = PreparedPass(tb.dst, dz, s3, plan(s3, Component.bww, V, 30, BwwCheck.input), mode,
                              out=self.grad_slice[f"b{bi}.c3"])
            seq += [tb, w3, _Scale(scale, self.grad_slice[f"b{bi}.c3"])]
            i3 = PreparedPass(dz, G3[1], s3, plan(s3, Component.bwi, V), mode,
                              epilogue=Epilogue(alpha=scale, mask=A["b"].data))
            db = i3.desc
            seq.append(i3)
            # conv2
            ta = _Transpose(A["a"], self.chwnn[:_chwnn_numel(A["a"])])
            w2 = PreparedPass(ta.dst, db, s2, plan(s2, Component.bww, V, 30, BwwCheck.input), mode,
                              out=self.grad_slice[f"b{bi}.c2"])
            i2 = PreparedPass(db, G2[1], s2, plan(s2, Component.bwi, V), mode, epilogue=Epilogue(mask=A["a"].data))
            da = i2.desc
            seq += [ta, w2, i2]
            # conv1 (+ projection)
            tx = _Transpose(A["x"], self.chwnn[:_chwnn_numel(A["x"])])
            w1 = PreparedPass(tx.dst, da, s1, plan(s1, Component.bww, V, 30, BwwCheck.input), mode,
                              out=self.grad_slice[f"b{bi}.c1"])
            seq += [tx, w1]
            if sp_ is not None:
                Gp = self.weights[f"b{bi}.proj"]
                wp = PreparedPass(tx.dst, dz, sp_, plan(sp_, Component.bww, V, 30, BwwCheck.input), mode,
                                  out=self.grad_slice[f"b{bi}.proj"])
                ip = PreparedPass(dz, Gp[1], sp_, plan(sp_, Component.bwi, V), mode)
                seq += [wp, ip]
                skip = ip.desc
                self.passes += [(f"b{bi}.proj", Component.bww, sp_), (f"b{bi}.proj", Component.bwi, sp_)]
            else:
                skip = dz
            # dz' = (x > 0) ? BWI1(da) + skip : 0   (x is the previous block's relu output / x0)
            i1 = PreparedPass(da, G1[1], s1, plan(s1, Component.bwi, V), mode,
                              epilogue=Epilogue(add=skip.data, mask=A["x"].data))
            seq.append(i1)
            for nm, sh in (("c3", s3), ("c2", s2), ("c1", s1)):
                self.passes += [(f"b{bi}.{nm}", Component.bww, sh), (f"b{bi}.{nm}", Component.bwi, sh)]
            names_b = [f"b{bi}.c1", f"b{bi}.c2", f"b{bi}.c3"] + ([f"b{bi}.proj"] if sp_ is not None else [])
            self._bwd_blocks.append((seq, names_b, dict(db=db, da=da, dz_in=dz)))
            dz = i1.desc
        self.dx0 = dz

    # ------------------------------------------------------------------
    def _calibrate(self, target: float, calib_images: int, device) -> None:
        """Fixup biases from a seeded forward pass: run the forward with each
        ReLU pass's epilogue switched to identity, take the `target` quantile
        tau of its pre-activation over the first `calib_images` images of
        the global batch (rank 0's slice), set beta = -tau, apply the ReLU
        (so the next layer sees the calibrated activation), continue.  Rank 0's
        values are broadcast when torch.distributed is initialised."""
        torch = self.torch
        st = torch.cuda.current_stream()
        relu_of = {id(p): name for name, p in self._relu_passes}
        ncal = max(1, min(calib_images, self.N))
        for p in self._fwd:
            name = relu_of.get(id(p))
            if name is None:
                p.launch(st.cuda_stream)
                continue
            p._epi.relu = 0
            p._epi.beta = 0.0
            p.launch(st.cuda_stream)
            z = p.out[: p.out.numel() // self.N * ncal]
            idx = torch.randint(0, z.numel(), (min(z.numel(), 1 << 22),), device=z.device,
                                generator=torch.Generator(device=z.device).manual_seed(17))
            tau = float(torch.quantile(z[idx].double(), target))
            beta = self._bcast(-tau)
            self.bias[name] = beta
            p._epi.relu = 1
            p._epi.beta = beta
            # the calibrated activation for the layers that follow (setup only)
            v = p.out + beta
            p.out.copy_(torch.where(v > 0, v, torch.zeros((), device=v.device)))
        torch.cuda.synchronize()

    def _bcast(self, v: float) -> float:
        torch = self.torch
        import torch.distributed as dist
        v = float(self.torch.tensor(v, dtype=torch.float32))  # the float32 the epilogue applies
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            t = torch.tensor([v], dtype=torch.float32, device="cuda" if dist.get_backend() == "nccl" else "cpu")
            dist.broadcast(t, src=0)
            v = float(t.item())
        return v

    def global_dense_flops(self) -> int:
        """Dense-equivalent FLOPs of one step over the GLOBAL batch (all ranks)."""
        return sum(sh.with_batch(self.N_global).dense_flops() for _, _, sh in self.passes)

    def set_upstream(self, dout_plain=None, sparsity: float = 0.0):
        """Upstream gradient w.r.t. the last block output: N(0,1) over the
        global batch from the chain's generator, this rank's slice (default)."""
        torch = self.torch
        from .api import pack_act_nchwc
        last = self.acts[-1]["out"]
        if dout_plain is None:
            full = torch.randn((self.N_global, last.c, last.h, last.w), device=self.dout.device, generator=self.gen)
            dout_plain = full[self.shard[0]:self.shard[0] + last.n]
        self.dout.copy_(pack_act_nchwc(dout_plain, self.V).data)

    def forward(self, stream_ptr: int) -> None:
        for p in self._fwd:
            p.launch(stream_ptr)

    def backward(self, stream_ptr: int, stream=None) -> None:
        self._mask_last.launch(stream_ptr)
        for seq, names, _ in self._bwd_blocks:
            for p in seq:
                p.launch(stream_ptr)
            if self.allreduce is not None:
                for n in names:
                    self.allreduce.submit(self.grad_slice[n], stream)
        if self.allreduce is not None:
            self.allreduce.wait(stream)

    def step(self, stream=None) -> None:
        torch = self.torch
        st = stream or torch.cuda.current_stream()
        self.forward(st.cuda_stream)
        self.backward(st.cuda_stream, st)

    def dense_flops(self) -> int:
        return sum(sh.dense_flops() for _, _, sh in self.passes)

    def sparsity_report(self) -> dict:
        """Zero fraction of each conv's checked tensor after a step (not timed)."""
        torch = self.torch
        zs = lambda t: float((t.data == 0).float().mean())
        fwd_in, bwd_in = [], []
        for A in self.acts:
            fwd_in += [zs(A["x"]), zs(A["a"]), zs(A["b"])]
        for _, _, T in self._bwd_blocks:
            bwd_in += [zs(T["dz_in"]), zs(T["db"]), zs(T["da"])]
        del torch
        return {"activation_sparsity_mean": sum(fwd_in) / len(fwd_in),
                "gradient_sparsity_mean": sum(bwd_in) / len(bwd_in),
                "activation_sparsity": fwd_in, "gradient_sparsity": bwd_in}


def _chwnn_numel(t: BlockedTensor) -> int:
    return ((t.n + t.V - 1) // t.V) * t.c * t.h * t.w * t.V


class _MaskedCopy:
    """dst = (pre > 0) ? up : 0  -- the reference's relu_grad_mask (sparsity.cpp:26)."""

    def __init__(self, up, pre, dst):
        self._a = (up, pre, dst)

    def launch(self, stream_ptr: int) -> None:
        up, pre, dst = self._a
        st = _lib.load().spc_relu_grad_mask(C.c_void_p(pre.data_ptr()), C.c_void_p(up.data_ptr()),
                                            C.c_void_p(dst.data_ptr()), up.numel(), C.c_void_p(stream_ptr))
        if st:
            raise SpconvError(st, _lib.last_error())


def fixup_resnet50(N: int, **kw) -> FixupChain:
    """BASELINE cfg 5 at global batch N (224x224 input, so 56x56 into stage 1);
    `world`/`rank` select this rank's batch shard."""
    ch = FixupChain(N, resnet50_blocks(), **kw)
    ch.set_upstream()
    return ch


__all__ = ["Bottleneck", "resnet50_blocks", "FixupChain", "fixup_resnet50", "math"]
