"""Seeded synthetic inputs shared by the oracle and the product path.

This module holds NO arithmetic of the method (no pruning, quantization,
indexing, coding or inference).  It only draws the random dense weights,
biases and activations that stand in for the paper's trained AlexNet /
VGG-16 models and ImageNet images (§5.1), with the shapes,
densities and bit widths of BASELINE.json configs C1..C5.  The recipe is
stated in DESIGN.md §"Input recipe".

Both `oracle/` and the product (`paper_1711_00244_b200/`, `bench.py`) import
this module; neither imports the other.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class FCSpec:
    """One fully-connected layer b = W a + v (Eq. 1)."""
    name: str
    rows: int            # N = output features
    cols: int            # K = input features
    density: float       # kept fraction after magnitude pruning
    sigma: float         # std of the N(0, sigma) synthetic weights
    r: int = 5           # quantization bits (codebook has 2^r entries)
    k: int = 4           # relative-index bits
    relu: bool = True    # ReLU after this layer (not after the last)
    seed_offset: int = 0


@dataclasses.dataclass(frozen=True)
class ConvSpec:
    """One CONV layer lowered to a matrix product (§3.1)."""
    name: str
    out_ch: int          # M filters (rows of the weight matrix)
    in_ch: int           # C input channels (all groups)
    kh: int
    kw: int
    stride: int
    pad: int
    groups: int
    density: float
    r: int = 8
    k: int = 8
    relu: bool = True
    lrn: bool = False    # LRN after ReLU (AlexNet norm1/norm2)
    pool: bool = False   # 3x3/s2 max-pool after (AlexNet pool1/2/5)
    seed_offset: int = 100

    @property
    def cols(self) -> int:
        return self.kh * self.kw * (self.in_ch // self.groups)

    @property
    def rows(self) -> int:
        return self.out_ch

    @property
    def sigma(self) -> float:
        return float(np.sqrt(2.0 / self.cols))


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    fc: Tuple[FCSpec, ...]
    conv: Tuple[ConvSpec, ...] = ()
    batches: Tuple[int, ...] = (1,)
    seed: int = 0
    tot_bytes: Optional[int] = None
    image_hw: int = 227
    image_c: int = 3


def _fc_stack(names_rows_cols_d, sigma=0.005):
    out = []
    n = len(names_rows_cols_d)
    for i, (nm, rows, cols, d) in enumerate(names_rows_cols_d):
        out.append(FCSpec(nm, rows, cols, d, sigma, relu=(i != n - 1), seed_offset=i))
    return tuple(out)


ALEXNET_FC = _fc_stack([("fc6", 4096, 9216, 0.09), ("fc7", 4096, 4096, 0.09),
                        ("fc8", 1000, 4096, 0.25)])
VGG16_FC = _fc_stack([("fc6", 4096, 25088, 0.04), ("fc7", 4096, 4096, 0.04),
                      ("fc8", 1000, 4096, 0.23)])

# AlexNet conv geometry (reading C-19: conv1 s4 p0; conv2 p2 g2; conv3 p1;
# conv4/conv5 p1 g2; LRN after conv1/conv2; 3x3/s2 max-pool after conv1,2,5).
ALEXNET_CONV = (
    ConvSpec("conv1", 96, 3, 11, 11, 4, 0, 1, 0.84, lrn=True, pool=True, seed_offset=100),
    ConvSpec("conv2", 256, 96, 5, 5, 1, 2, 2, 0.38, lrn=True, pool=True, seed_offset=101),
    ConvSpec("conv3", 384, 256, 3, 3, 1, 1, 1, 0.35, seed_offset=102),
    ConvSpec("conv4", 384, 384, 3, 3, 1, 1, 2, 0.37, seed_offset=103),
    ConvSpec("conv5", 256, 384, 3, 3, 1, 1, 2, 0.37, pool=True, seed_offset=104),
)

CONFIGS = {
    "C1": Config("C1", (FCSpec("fc", 1024, 1024, 0.10, 0.02, relu=False),), batches=(1,)),
    "C2": Config("C2", (FCSpec("fc6", 4096, 9216, 0.09, 0.005, relu=False),),
                 batches=(1, 8, 32, 128)),
    "C3": Config("C3", ALEXNET_FC, batches=tuple(range(1, 257)), tot_bytes=64 << 20),
    "C4": Config("C4", ALEXNET_FC, conv=ALEXNET_CONV, batches=(64,)),
    "C5": Config("C5", VGG16_FC, batches=(1, 8, 32, 128, 256, 512)),
}


def fc_weights(spec, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Dense fp32 W (rows x cols) ~ N(0, sigma) and bias v ~ N(0, 0.01).

    For a ConvSpec, W is (out_ch x kh*kw*in_ch/groups) with K flattened as
    (r, s, c), channel fastest (reading C-18)."""
    rng = np.random.default_rng(seed + spec.seed_offset)
    W = rng.standard_normal((spec.rows, spec.cols), dtype=np.float32)
    W *= np.float32(spec.sigma)
    v = rng.standard_normal(spec.rows, dtype=np.float32) * np.float32(0.01)
    return W, v.astype(np.float32)


def fc_inputs(features: int, batch: int, seed: int) -> np.ndarray:
    """Image-major activations [batch][features] = ReLU(N(0,1)), fp32.

    Every smaller batch is a prefix of a larger one (same seed), so a given
    image's output does not depend on the batch it is run in."""
    rng = np.random.default_rng(seed + 1000)
    a = rng.standard_normal((batch, features), dtype=np.float32)
    return np.maximum(a, np.float32(0.0))


def conv_inputs(batch: int, hw: int = 227, c: int = 3, seed: int = 0) -> np.ndarray:
    """NHWC fp32 images ~ U(0,1)."""
    rng = np.random.default_rng(seed + 2000)
    return rng.random((batch, hw, hw, c), dtype=np.float32)


def random_matrix(rows: int, cols: int, seed: int, scale: float = 1.0) -> np.ndarray:
    """Small random fp32 matrices for edge-case fixtures."""
    rng = np.random.default_rng(seed)
    return (rng.standard_normal((rows, cols), dtype=np.float32) * np.float32(scale))


def random_activations(features: int, batch: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return np.maximum(rng.standard_normal((batch, features), dtype=np.float32), np.float32(0))
