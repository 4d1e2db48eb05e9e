"""Gradient-set shapes of the paper's workloads (metadata only, no weights).

* ResNet-50 (He et al. 2016), the benchmark of PAPER.md:550-556 (§6.4): the
  161 parameter tensors in model-traversal order ("parameters ... collected
  easily by traversing"), i.e. conv1, bn1, then per bottleneck
  conv1/bn1/conv2/bn2/conv3/bn3 (+ downsample conv/bn on the first block of
  each stage), stages of [3, 4, 6, 3] blocks with widths 64/128/256/512 and
  expansion 4, then fc (2048 -> 1000).  P = 25,557,032.
* The tiny MLP 784-100-100-10 of Fig. `fig:link-chain`,
  weights laid out (n_out, n_in) as in Chainer's Linear.  P = 89,610.
"""
from __future__ import annotations

from math import prod


def numel(shape) -> int:
    return int(prod(shape)) if len(shape) else 1


def resnet50_shapes(num_classes: int = 1000):
    shapes = [(64, 3, 7, 7), (64,), (64,)]
    inplanes = 64
    for width, blocks in ((64, 3), (128, 4), (256, 6), (512, 3)):
        for b in range(blocks):
            out = width * 4
            shapes += [(width, inplanes, 1, 1), (width,), (width,),
                       (width, width, 3, 3), (width,), (width,),
                       (out, width, 1, 1), (out,), (out,)]
            if b == 0:
                shapes += [(out, inplanes, 1, 1), (out,), (out,)]
            inplanes = out
    shapes += [(num_classes, 2048), (num_classes,)]
    return shapes


def mlp_shapes():
    return [(100, 784), (100,), (100, 100), (100,), (10, 100), (10,)]


WORKLOADS = {
    "mlp": mlp_shapes,
    "r50": resnet50_shapes,
}
