"""The paper's convolution workloads as parameter tuples (host-side tables only).

Tuple order is Fig. 1's caption: "window size, stride, image rows, image
columns, input features, output features".

* RESNET50_SETS: the 26 ResNet-50 sets of Fig. 1.  The paper
  gives only the count; reading R9 takes the
  union of the distinct conv tuples of ResNet-50 v1 and v1.5, which is exactly 26.
* VGG16_LAYERS: VGG-16 config D, 9 distinct shapes / 13 layers, 3x3 SAME s1 on
  224x224 (PAPER.md:220 names VGG; reading R10).
* RESNET50_V15_STACK: the 53 convs of ResNet-50 v1.5 with multiplicities
  (BASELINE.json config 5; reading R11).
"""
from __future__ import annotations

from dataclasses import dataclass

SAME, VALID = 0, 1


@dataclass(frozen=True)
class Layer:
    name: str
    window: int
    stride: int
    rows: int
    cols: int
    channels: int
    features: int
    padding: int = SAME

    def params(self, batch: int) -> dict:
        return dict(batch=batch, in_rows=self.rows, in_cols=self.cols, channels=self.channels,
                    features=self.features, window_rows=self.window, window_cols=self.window,
                    stride_rows=self.stride, stride_cols=self.stride, padding=self.padding)

    def flops(self, batch: int) -> int:
        ho = -(-self.rows // self.stride) if self.padding == SAME else (self.rows - self.window) // self.stride + 1
        wo = -(-self.cols // self.stride) if self.padding == SAME else (self.cols - self.window) // self.stride + 1
        return 2 * batch * ho * wo * self.window * self.window * self.channels * self.features


def _L(name, k, s, h, w, c, f):
    return Layer(name, k, s, h, w, c, f, SAME)


RESNET50_SETS = [
    _L("R1", 7, 2, 224, 224, 3, 64),
    _L("R2", 1, 1, 56, 56, 64, 256),
    _L("R3", 1, 1, 56, 56, 64, 64),
    _L("R4", 3, 1, 56, 56, 64, 64),
    _L("R5", 1, 1, 56, 56, 256, 64),
    _L("R6", 1, 2, 56, 56, 256, 512),
    _L("R7", 1, 2, 56, 56, 256, 128),
    _L("R8", 1, 1, 56, 56, 256, 128),
    _L("R9", 3, 2, 56, 56, 128, 128),
    _L("R10", 3, 1, 28, 28, 128, 128),
    _L("R11", 1, 1, 28, 28, 128, 512),
    _L("R12", 1, 1, 28, 28, 512, 128),
    _L("R13", 1, 2, 28, 28, 512, 1024),
    _L("R14", 1, 2, 28, 28, 512, 256),
    _L("R15", 1, 1, 28, 28, 512, 256),
    _L("R16", 3, 2, 28, 28, 256, 256),
    _L("R17", 3, 1, 14, 14, 256, 256),
    _L("R18", 1, 1, 14, 14, 256, 1024),
    _L("R19", 1, 1, 14, 14, 1024, 256),
    _L("R20", 1, 2, 14, 14, 1024, 2048),
    _L("R21", 1, 2, 14, 14, 1024, 512),
    _L("R22", 1, 1, 14, 14, 1024, 512),
    _L("R23", 3, 2, 14, 14, 512, 512),
    _L("R24", 3, 1, 7, 7, 512, 512),
    _L("R25", 1, 1, 7, 7, 512, 2048),
    _L("R26", 1, 1, 7, 7, 2048, 512),
]

VGG16_LAYERS = [  # (layer, multiplicity in the 13-layer net)
    (_L("V1", 3, 1, 224, 224, 3, 64), 1),
    (_L("V2", 3, 1, 224, 224, 64, 64), 1),
    (_L("V3", 3, 1, 112, 112, 64, 128), 1),
    (_L("V4", 3, 1, 112, 112, 128, 128), 1),
    (_L("V5", 3, 1, 56, 56, 128, 256), 1),
    (_L("V6", 3, 1, 56, 56, 256, 256), 2),
    (_L("V7", 3, 1, 28, 28, 256, 512), 1),
    (_L("V8", 3, 1, 28, 28, 512, 512), 2),
    (_L("V9", 3, 1, 14, 14, 512, 512), 3),
]

# ResNet-50 v1.5 conv stack: tuple name -> multiplicity (53 convs, 8.174 GFLOP/image).
RESNET50_V15_MULT = {
    "R1": 1, "R3": 1, "R6": 1, "R8": 1, "R9": 1, "R13": 1, "R15": 1, "R16": 1, "R20": 1, "R22": 1, "R23": 1,
    "R5": 2, "R24": 2, "R26": 2,
    "R4": 3, "R10": 3, "R12": 3, "R25": 3,
    "R2": 4, "R11": 4,
    "R17": 5, "R19": 5,
    "R18": 6,
}

CONFIG1 = _L("C1", 3, 1, 8, 8, 4, 8)  # BASELINE.json configs[0]


def by_name(name: str) -> Layer:
    for l in RESNET50_SETS:
        if l.name == name:
            return l
    for l, _ in VGG16_LAYERS:
        if l.name == name:
            return l
    if name == "C1":
        return CONFIG1
    raise KeyError(name)


def resnet50_v15_stack():
    """The 53 convs as (layer_id, Layer) in network order of first appearance per tuple.

    Network order matters only for timing realism; every conv runs on its own
    seeded input (no chaining: BN/ReLU/pool/add are out of scope, reading R11).
    """
    order = []
    # Build the v1.5 network order from the generator: stage widths p, blocks, stride.
    def t(k, s, h, c, f):
        for l in RESNET50_SETS:
            if (l.window, l.stride, l.rows, l.channels, l.features) == (k, s, h, c, f):
                return l
        raise KeyError((k, s, h, c, f))

    order.append(t(7, 2, 224, 3, 64))
    h = 56
    c_in = 64
    for p, nblocks, s in ((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2)):
        for b in range(nblocks):
            stride = s if b == 0 else 1
            order.append(t(1, 1, h, c_in, p))              # 1x1 reduce (v1.5: stride 1)
            order.append(t(3, stride, h, p, p))            # 3x3 (v1.5: carries the stride)
            ho = h // stride
            order.append(t(1, 1, ho, p, 4 * p))            # 1x1 expand
            if b == 0:
                order.append(t(1, stride, h, c_in, 4 * p))  # projection shortcut
            c_in = 4 * p
            h = ho
    return list(enumerate(order))
