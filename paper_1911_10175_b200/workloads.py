"""BASELINE.json workloads: layer lists and seeded synthetic inputs.

The reference measures on "synthetic input with random sparse patterns"
(PAPER.md:559); BASELINE.json fixes the distributions restated here:

* activations  D = ReLU(x), x ~ N(-t, 1), t = Phi^-1(s)  => P(D == 0) = s, i.i.d.
  (ReLU with the reference's semantics v > 0 ? v : 0, P/src/sparsity.cpp:13)
* weights      G ~ N(0, sqrt(2 / (C*R*S)))               (He-normal)
* output grads dY ~ N(0, 1) * Bernoulli(1 - s) mask       (independent ReLU mask)

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


def config1() -> list[Layer]:
    """BASELINE cfg 1: N=16, C=K=64, 56x56, 3x3 s1 p1."""
    return [_L("cfg1", 16, 64, 64, 56, 3)]


def vgg16(N=32) -> list[Layer]:
    """BASELINE cfg 2: the 12 non-initial 3x3 convs of VGG16 at 224x224."""
    spec = [("conv1_2", 64, 64, 224), ("conv2_1", 64, 128, 112), ("conv2_2", 128, 128, 112),
            ("conv3_1", 128, 256, 56), ("conv3_2", 256, 256, 56), ("conv3_3", 256, 256, 56),
            ("conv4_1", 256, 512, 28), ("conv4_2", 512, 512, 28), ("conv4_3", 512, 512, 28),
            ("conv5_1", 512, 512, 14), ("conv5_2", 512, 512, 14), ("conv5_3", 512, 512, 14)]
    return [_L(n, N, c, k, hw, 3) for n, c, k, hw in spec]


def resnet34(N=64) -> list[Layer]:
    """BASELINE cfg 3: ResNet-34 basic-block 3x3 convs + 1x1 s2 projections."""
    out = []
    cin, hw = 64, 56
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            out.append(_L(f"s{stage + 1}b{b + 1}c1", N, cin, width, hw, 3, stride))
            if stride == 2:
                out.append(_L(f"s{stage + 1}proj", N, cin, width, hw, 1, 2))
                hw //= 2
            out.append(_L(f"s{stage + 1}b{b + 1}c2", N, width, width, hw, 3))
            cin = width
    return out


def resnet50(N=64) -> list[Layer]:
    """BASELINE cfg 4/5: ResNet-50 v1.5 bottlenecks (stride 2 on the 3x3)."""
    out = []
    cin, hw = 64, 56
    for stage, (width, blocks) in enumerate([(64, 3), (128, 4), (256, 6), (512, 3)]):
        for b in range(blocks):
            stride = 2 if (b == 0 and stage > 0) else 1
            out.append(_L(f"s{stage + 1}b{b + 1}reduce", N, cin, width, hw, 1))
            out.append(_L(f"s{stage + 1}b{b + 1}conv3", N, width, width, hw, 3, stride))
            if b == 0:
                out.append(_L(f"s{stage + 1}proj", N, cin, 4 * width, hw, 1, stride))
            hw //= stride
            out.append(_L(f"s{stage + 1}b{b + 1}expand", N, width, 4 * width, hw, 1))
            cin = 4 * width
    return out


CONFIGS = {
    "cfg1_single3x3_b16": config1,
    "vgg16_b32": lambda: vgg16(32),
    "resnet34_b64": lambda: resnet34(64),
    "resnet50_b64": lambda: resnet50(64),
    "fixup_resnet50_b256": lambda: resnet50(256),
}


def relu_threshold(s: float) -> float:
    """t with P(N(-t,1) <= 0) = s."""
    if s <= 0.0:
        return -np.inf
    if s >= 1.0:
        return np.inf
    return statistics.NormalDist().inv_cdf(s)


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
