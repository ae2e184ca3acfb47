"""BASELINE.json workloads: layer lists and seeded synthetic inputs.

The reference measures on "synthetic input with random sparse patterns"
(PAPER.md:559); BASELINE.json fixes the distributions restated here:

* activations  D = ReLU(x), x ~ N(-t, 1), t = Phi^-1(s)  => P(D == 0) = s, i.i.d.
  (ReLU with the reference's semantics v > 0 ? v : 0, P/src/sparsity.cpp:13)
* weights      G ~ N(0, sqrt(2 / (C*R*S)))               (He-normal)
* output grads dY ~ N(0, 1) * Bernoulli(1 - s) mask       (independent ReLU mask)

Per configuration (``layer_inputs_host`` / ``layer_inputs_device``):

* cfg 1, cfg 2 (VGG16): the three lines above at the grid sparsity s.
* cfg 3 (ResNet-34): per-layer sparsity s_l ~ U[0.4, 0.8] (seeded,
  ``layer_sparsity``) for D; dY DENSE N(0,1): a BatchNorm sits between each
  conv and its ReLU, so the conv's output gradient carries no ReLU zeros
  (the reference projector's rule, P/src/projector.cpp:120-125).
* cfg 4 (ResNet-50): spatially correlated D = ReLU(conv3x3_rand(X) - tau),
  X ~ N(0,1), random C->C weights built on a smoothing kernel (see
  spatial_activation), tau the 0.6-quantile of the conv output (estimated on
  a seeded sample) => mean sparsity 0.6 with zeros clustered in space;
  dY dense N(0,1) (BatchNorm, as cfg 3).
* cfg 5 (Fixup ResNet-50): inputs come from the chain's own seeded forward
  pass (``chain.FixupChain``), not from here.

Generation is seeded; host arrays come from numpy's PCG64, device tensors
from torch's CUDA generator (same distributions, different streams).  Parity
tests that compare the GPU with the CPU always feed the SAME arrays to both.
"""
from __future__ import annotations

import dataclasses
import statistics

import numpy as np

from .api import ConvShape


@dataclasses.dataclass(frozen=True)
class Layer:
    name: str
    shape: ConvShape


def _L(name, N, C, K, HW, R, stride=1):
    return Layer(name, ConvShape.make(N, C, K, HW, HW, R, R, stride, stride))


# Layer tables as plain tuples (name, N, C, K, H=W, R=S, stride): importable and
# usable without loading the product library (bench.py's reference arm builds
# its shapes from these with the reference's own conv_shape::make).
def config1_spec(N=16):
    """BASELINE cfg 1: N=16, C=K=64, 56x56, 3x3 s1 p1."""
    return [("cfg1", N, 64, 64, 56, 3, 1)]


def vgg16_spec(N=32):
    """BASELINE cfg 2: the 12 non-initial 3x3 convs of VGG16 at 224x224."""
    spec = [("conv1_2", 64, 64, 224), ("conv2_1", 64, 128, 112), ("conv2_2", 128, 128, 112),
            ("conv3_1", 128, 256, 56), ("conv3_2", 256, 256, 56), ("conv3_3", 256, 256, 56),
            ("conv4_1", 256, 512, 28), ("conv4_2", 512, 512, 28), ("conv4_3", 512, 512, 28),
            ("conv5_1", 512, 512, 14), ("conv5_2", 512, 512, 14), ("conv5_3", 512, 512, 14)]
    return [(n, N, c, k, hw, 3, 1) for n, c, k, hw in spec]


def resnet34_spec(N=64):
    """BASELINE cfg 3: ResNet-34 basic-block 3x3 convs + 1x1 s2 projections."""
    out = []
    cin, hw = 64, 56
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            out.append((f"s{stage + 1}b{b + 1}c1", N, cin, width, hw, 3, stride))
            if stride == 2:
                out.append((f"s{stage + 1}proj", N, cin, width, hw, 1, 2))
                hw //= 2
            out.append((f"s{stage + 1}b{b + 1}c2", N, width, width, hw, 3, 1))
            cin = width
    return out


def resnet50_spec(N=64):
    """BASELINE cfg 4/5: ResNet-50 v1.5 bottlenecks (stride 2 on the 3x3)."""
    out = []
    cin, hw = 64, 56
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            out.append((f"s{stage + 1}b{b + 1}reduce", N, cin, width, hw, 1, 1))
            out.append((f"s{stage + 1}b{b + 1}conv3", N, width, width, hw, 3, stride))
            if b == 0:
                out.append((f"s{stage + 1}proj", N, cin, 4 * width, hw, 1, stride))
            hw //= stride
            out.append((f"s{stage + 1}b{b + 1}expand", N, width, 4 * width, hw, 1, 1))
            cin = 4 * width
    return out


SPECS = {
    "cfg1_single3x3_b16": lambda: config1_spec(16),
    "vgg16_b32": lambda: vgg16_spec(32),
    "resnet34_b64": lambda: resnet34_spec(64),
    "resnet50_b64": lambda: resnet50_spec(64),
    "fixup_resnet50_b256": lambda: resnet50_spec(256),
}


def _layers(spec):
    return [_L(*t) for t in spec]


def config1() -> list[Layer]:
    return _layers(config1_spec())


def vgg16(N=32) -> list[Layer]:
    return _layers(vgg16_spec(N))


def resnet34(N=64) -> list[Layer]:
    return _layers(resnet34_spec(N))


def resnet50(N=64) -> list[Layer]:
    return _layers(resnet50_spec(N))


CONFIGS = {name: (lambda f=f: _layers(f())) for name, f in SPECS.items()}


class PlainShape:
    """conv_shape fields from an 11-int tuple (no library needed)."""

    def __init__(self, t):
        (self.N, self.C, self.K, self.H, self.W, self.R, self.S, self.O, self.P, self.padW, self.padH) = t

    def astuple(self):
        return (self.N, self.C, self.K, self.H, self.W, self.R, self.S, self.O, self.P, self.padW, self.padH)

    def out_w(self):
        return (self.W + 2 * self.padW - self.R) // self.O + 1

    def out_h(self):
        return (self.H + 2 * self.padH - self.S) // self.P + 1

    def dense_flops(self):
        return 2 * self.N * self.K * self.C * self.R * self.S * self.out_h() * self.out_w()

    def with_batch(self, n):
        return PlainShape((n,) + self.astuple()[1:])


def relu_threshold(s: float) -> float:
    """t with P(N(-t,1) <= 0) = s."""
    if s <= 0.0:
        return -np.inf
    if s >= 1.0:
        return np.inf
    return statistics.NormalDist().inv_cdf(s)


# ---------------------------------------------------------------- per-config inputs
GRID_CONFIGS = ("vgg16_b32",)  # i.i.d. D and masked dY swept over the sparsity grid (cfg 1: fixed s = 0.5)
BN_CONFIGS = ("resnet34_b64", "resnet50_b64")         # dense dY (BatchNorm before the ReLU)
R50_TARGET = 0.6


def layer_sparsity(config: str, li: int, s: float | None = None, seed: int = 0) -> float:
    """D's sparsity for layer `li` of `config`: the swept s (cfg 1/2), a seeded
    U[0.4, 0.8] draw per layer (cfg 3), the 0.6 target (cfg 4)."""
    if config == "resnet34_b64":
        n = len(SPECS[config]())
        return float(np.random.default_rng([seed, 34]).uniform(0.4, 0.8, n)[li])
    if config == "resnet50_b64":
        return R50_TARGET
    if s is None:
        return 0.5 if config == "cfg1_single3x3_b16" else 0.6
    return float(s)


def grad_sparsity(config: str, s: float) -> float:
    """dY's sparsity: masked like D for the nets without BatchNorm, 0 (dense) for cfg 3/4."""
    return 0.0 if config in BN_CONFIGS else s


def _layer_seed(config: str, li: int, seed: int) -> list[int]:
    return [seed, sum(map(ord, config)), li]


def spatial_activation(shape4, target: float, gen, device="cpu"):
    """cfg 4: ReLU(conv3x3_rand(X) - tau), X ~ N(0,1), tau = the `target`
    quantile of the conv output (estimated from 1 M seeded samples).

    The random conv's weights are w[co, ci] = a[co, ci] * B + e[co, ci] with
    a ~ N(0, 1/C), B the 3x3 binomial (smoothing) kernel and a small He-normal
    part e: every output channel is a random mix of smoothed input channels,
    so neighbouring pixels correlate (~0.6 at lag 1) and the ReLU zeros come
    in spatial clusters, as in real feature maps.  (Purely zero-mean He-normal
    weights would leave neighbours uncorrelated in expectation.)  torch on
    `device` (CPU for parity fixtures, CUDA in the bench setup)."""
    import torch
    import torch.nn.functional as F
    N, C, H, W = shape4
    b1 = torch.tensor([1.0, 2.0, 1.0], device=device)
    blur = torch.outer(b1, b1) / 16.0
    a = torch.randn((C, C, 1, 1), generator=gen, device=device, dtype=torch.float32) / float(np.sqrt(C))
    e = torch.randn((C, C, 3, 3), generator=gen, device=device, dtype=torch.float32) * float(0.25 / np.sqrt(9 * C))
    w = a * blur + e
    out = torch.empty(shape4, device=device, dtype=torch.float32)
    step = max(1, (1 << 26) // max(1, C * H * W))  # bound the conv's temporary
    for i in range(0, N, step):
        x = torch.randn((min(step, N - i), C, H, W), generator=gen, device=device, dtype=torch.float32)
        out[i:i + x.shape[0]] = F.conv2d(x, w, padding=1)
    flat = out.view(-1)
    idx = torch.randint(0, flat.numel(), (min(flat.numel(), 1 << 20),), generator=gen, device=device)
    tau = float(torch.quantile(flat[idx], target))
    out.sub_(tau)
    return torch.where(out > 0, out, torch.zeros((), device=device))


def layer_inputs_host(config: str, li: int, sh, s: float | None = None, seed: int = 0):
    """Plain (D, G, dY) numpy float32 arrays for layer `li` of `config` at the
    shape `sh` (its batch may be a slice of the config's), seeded by (seed,
    config, layer)."""
    sd = layer_sparsity(config, li, s, seed)
    sg = grad_sparsity(config, sd)
    rng = np.random.default_rng(_layer_seed(config, li, seed) + [int(round(sd * 1000))])
    if config == "resnet50_b64":
        import torch
        gen = torch.Generator().manual_seed(int(rng.integers(1 << 62)))
        D = spatial_activation((sh.N, sh.C, sh.H, sh.W), sd, gen).numpy()
    else:
        D = host_activation((sh.N, sh.C, sh.H, sh.W), sd, rng)
    G = host_weights(sh.K, sh.C, sh.S, sh.R, rng)
    dY = host_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), sg, rng)
    return D, G, dY


def layer_inputs_device(config: str, li: int, sh, gen, s: float | None = None, seed: int = 0):
    """The same distributions as ``layer_inputs_host`` as CUDA tensors (torch's
    CUDA generator `gen`; a different stream from the host arrays)."""
    sd = layer_sparsity(config, li, s, seed)
    sg = grad_sparsity(config, sd)
    dev = gen.device
    if config == "resnet50_b64":
        D = spatial_activation((sh.N, sh.C, sh.H, sh.W), sd, gen, dev)
    else:
        D = device_activation((sh.N, sh.C, sh.H, sh.W), sd, gen, dev)
    G = device_weights(sh.K, sh.C, sh.S, sh.R, gen, dev)
    dY = device_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), sg, gen, dev)
    return D, G, dY


# ---------------------------------------------------------------- host (numpy)
def host_activation(shape4, s, rng: np.random.Generator) -> np.ndarray:
    if s <= 0.0:  # no ReLU zeros: |x| (zero with probability 0)
        return np.abs(rng.standard_normal(shape4, dtype=np.float32))
    x = rng.standard_normal(shape4, dtype=np.float32) - np.float32(relu_threshold(s))
    return np.where(x > 0, x, np.float32(0)).astype(np.float32)


def host_weights(K, C, S, R, rng: np.random.Generator) -> np.ndarray:
    return (rng.standard_normal((K, C, S, R), dtype=np.float32) * np.float32(np.sqrt(2.0 / (C * R * S))))


def host_grad(shape4, s, rng: np.random.Generator) -> np.ndarray:
    g = rng.standard_normal(shape4, dtype=np.float32)
    keep = rng.random(shape4, dtype=np.float32) >= np.float32(s)
    return np.where(keep, g, np.float32(0)).astype(np.float32)


def config1_inputs_host(seed=0, s=0.5):
    """cfg 1 plain inputs (D, G, dY) on the host, seeded."""
    sh = config1()[0].shape
    rng = np.random.default_rng(seed)
    D = host_activation((sh.N, sh.C, sh.H, sh.W), s, rng)
    G = host_weights(sh.K, sh.C, sh.S, sh.R, rng)
    dY = host_grad((sh.N, sh.K, sh.out_h(), sh.out_w()), s, rng)
    return D, G, dY


# ---------------------------------------------------------------- device (torch)
def device_activation(shape4, s, gen, device="cuda"):
    import torch
    if s <= 0.0:
        return torch.randn(shape4, generator=gen, device=device, dtype=torch.float32).abs_()
    x = torch.randn(shape4, generator=gen, device=device, dtype=torch.float32) - float(relu_threshold(s))
    return torch.where(x > 0, x, torch.zeros((), device=device))


def device_weights(K, C, S, R, gen, device="cuda"):
    import torch
    return torch.randn((K, C, S, R), generator=gen, device=device, dtype=torch.float32) * float(
        np.sqrt(2.0 / (C * R * S)))


def device_grad(shape4, s, gen, device="cuda"):
    import torch
    g = torch.randn(shape4, generator=gen, device=device, dtype=torch.float32)
    keep = torch.rand(shape4, generator=gen, device=device, dtype=torch.float32) >= float(s)
    return torch.where(keep, g, torch.zeros((), device=device))
