"""ResNet-50 v1.5 convolution layer table (the BASELINE.json cfg4/cfg5 workload)
and VGG-16's 3x3 layers (cfg3). Shapes only; used by bench.py and tests."""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class ConvLayer:
    name: str
    c: int
    k: int
    h: int      # input extent (square)
    r: int      # filter extent (square)
    stride: int
    pad: int

    @property
    def out_h(self) -> int:
        return (self.h + 2 * self.pad - self.r) // self.stride + 1

    def flops(self, n: int) -> float:
        """Direct-convolution algorithmic FLOPs of one direction: 2*N*K*C*R*S*P*Q."""
        return 2.0 * n * self.k * self.c * self.r * self.r * self.out_h * self.out_h


def resnet50_layers() -> list[ConvLayer]:
    L = [ConvLayer("conv1", 3, 64, 224, 7, 2, 3)]
    cin, h = 64, 56
    for stage, (width, blocks, stride) in enumerate(((64, 3, 1), (128, 4, 2), (256, 6, 2),
                                                     (512, 3, 2)), start=2):
        out = width * 4
        for b in range(blocks):
            s = stride if b == 0 else 1
            pre = f"conv{stage}_{b + 1}"
            L.append(ConvLayer(pre + "a", cin, width, h, 1, 1, 0))
            L.append(ConvLayer(pre + "b", width, width, h, 3, s, 1))  # v1.5: stride on the 3x3
            ho = (h + 2 - 3) // s + 1
            L.append(ConvLayer(pre + "c", width, out, ho, 1, 1, 0))
            if b == 0:
                L.append(ConvLayer(pre + "ds", cin, out, h, 1, s, 0))
            cin, h = out, ho
    assert len(L) == 53
    return L


def vgg16_layers() -> list[ConvLayer]:
    cfg = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112), (128, 256, 56),
           (256, 256, 56), (256, 256, 56), (256, 512, 28), (512, 512, 28), (512, 512, 28),
           (512, 512, 14), (512, 512, 14), (512, 512, 14)]
    return [ConvLayer(f"vgg{i}", c, k, h, 3, 1, 1) for i, (c, k, h) in enumerate(cfg)]
