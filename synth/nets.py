"""Synthetic CNN workloads of BASELINE.json configs 1, 3, 4, 5 (shapes, seeds, sigmas only).

This module is workload DATA shared by the oracle side and the CUDA side: layer shapes as the
configs state them, the seeded float64 weights / images (A34) and the fixed activation
coefficients (A25).  It holds no encrypted-evaluation logic: the HW-tiled lowering (layouts,
rotation amounts, folding, masks, level plan) is implemented independently by
``paper_1810_00845_b200/driver.py`` and ``oracle/nets.py``.

Layer tuples (PyTorch semantics for the float64 definition):
    ("conv", oc, k, stride, pad[, "chw"])   cross-correlation, zero padding `pad`; "chw" selects the
                                   CHW-tiled encrypted lowering (NEXT-1), not semantics
    ("act",)                       a0 + a1 x + a2 x^2 with ACT_COEFFS (A25)
    ("square",)                    x^2 (config 1)
    ("avgpool",)                   2x2, stride 2
    ("fc", out[, R[, "chw"]])      W @ flatten(x) (flatten order c, y, x); R = replicas per
                                   ciphertext in the encrypted lowering (A27), "chw" the CHW-tiled
                                   FC lowering (NEXT-1, R = 1); not semantics
    ("fire", sq, e1, e3)           SqueezeNet fire module (config 5): s = act(conv1x1(x));
                                   out = concat(act(conv1x1(s)) [e1 ch], act(conv3x3 SAME(s)) [e3 ch])
    ("gap",)                       global average pool (config 5)
Convs and FCs have no bias (A34).
"act_gains" (A41): compile-time gain (a power of 4) of every activation in execution order (a fire
module's squeeze, then its expand), written from tools/calibrate_gains.py (float64 network on a
calibration image, T = 16); a lowering choice like R, not semantics.
"""
from __future__ import annotations

import numpy as np

from . import image as _image, weights as _weights

# A25: (a0, a1, a2) -- SPEC's example activation values a = 0.25 (x^2), b = 0.5 (x)
ACT_COEFFS = (0.0, 0.5, 0.25)

NETS = {
    # config 1: tiny encrypted conv (BASELINE.json configs[0])
    "tiny": dict(log_n=13, q_bits=[60, 40, 40], p_bits=60, scale=2.0 ** 40, input=(1, 8, 8),
                 layers=[("conv", 2, 3, 1, 0), ("square",)], sigma=[0.1]),
    # config 3: LeNet-5-small-shaped (A31: pad 1 -> 30x30, 5x5 stride 2 -> 13x13x5 = 845); FC1
    # lowered with R = 8 replicas (A27: the measured-cheaper lowering on B200, 6 of 6 levels)
    "lenet_small": dict(log_n=14, q_bits=[60] + [40] * 6, p_bits=60, scale=2.0 ** 40, input=(1, 28, 28),
                        layers=[("conv", 5, 5, 2, 1), ("act",), ("fc", 100, 8), ("act",), ("fc", 10)],
                        sigma=[0.1, 0.1, 0.1], act_gains=[4.0 ** 3, 4.0 ** 2]),
    # config 4: LeNet-5-large-shaped (A32: SAME 5x5 convs, 28 -> 14 -> 7, 7*7*64 = 3136)
    "lenet_large": dict(log_n=15, q_bits=[60] + [40] * 13, p_bits=60, scale=2.0 ** 40, input=(1, 28, 28),
                        layers=[("conv", 32, 5, 1, 2), ("act",), ("avgpool",), ("conv", 64, 5, 1, 2), ("act",),
                                ("avgpool",), ("fc", 512, 16), ("act",), ("fc", 10)],
                        sigma=[0.05, 0.05, 0.05, 0.05], act_gains=[4.0 ** 2, 4.0 ** 3, 4.0 ** 3]),
    # config 4 with its second conv CHW-tiled (several channels per ciphertext; the paper's
    # layout comparison, Fig. tilings)
    "lenet_large_chw": dict(log_n=15, q_bits=[60] + [40] * 13, p_bits=60, scale=2.0 ** 40, input=(1, 28, 28),
                            layers=[("conv", 32, 5, 1, 2), ("act",), ("avgpool",), ("conv", 64, 5, 1, 2, "chw"),
                                    ("act",), ("avgpool",), ("fc", 512, 16), ("act",), ("fc", 10)],
                            sigma=[0.05, 0.05, 0.05, 0.05], act_gains=[4.0 ** 2, 4.0 ** 3, 4.0 ** 3]),
    # NEXT-1 layout strategies (Fig. tilings) on configs 3 / 4 -- lowering choices only,
    # the same weights (seeds) and float64 network as the base config:
    #   "CHW-fc HW-before": HW convs, CHW-tiled FC1 (also this build's "HW-conv CHW-rest": the
    #   activations and pools act per channel in both, see DESIGN.md NEXT-1)
    #   "CHW": every stride-1 conv and FC1 CHW-tiled
    "lenet_small_chwfc": dict(log_n=14, q_bits=[60] + [40] * 6, p_bits=60, scale=2.0 ** 40, input=(1, 28, 28),
                              layers=[("conv", 5, 5, 2, 1), ("act",), ("fc", 100, 1, "chw"), ("act",), ("fc", 10)],
                              sigma=[0.1, 0.1, 0.1], act_gains=[4.0 ** 3, 4.0 ** 2]),
    "lenet_large_chwfc": dict(log_n=15, q_bits=[60] + [40] * 13, p_bits=60, scale=2.0 ** 40, input=(1, 28, 28),
                              layers=[("conv", 32, 5, 1, 2), ("act",), ("avgpool",), ("conv", 64, 5, 1, 2), ("act",),
                                      ("avgpool",), ("fc", 512, 1, "chw"), ("act",), ("fc", 10)],
                              sigma=[0.05, 0.05, 0.05, 0.05], act_gains=[4.0 ** 2, 4.0 ** 3, 4.0 ** 3]),
    "lenet_large_chw_all": dict(log_n=15, q_bits=[60] + [40] * 13, p_bits=60, scale=2.0 ** 40, input=(1, 28, 28),
                                layers=[("conv", 32, 5, 1, 2, "chw"), ("act",), ("avgpool",), ("conv", 64, 5, 1, 2, "chw"),
                                        ("act",), ("avgpool",), ("fc", 512, 1, "chw"), ("act",), ("fc", 10)],
                                sigma=[0.05, 0.05, 0.05, 0.05], act_gains=[4.0 ** 2, 4.0 ** 3, 4.0 ** 3]),
    # config 5: SqueezeNet-CIFAR-shaped (A33: conv1 + 4 fire modules + 1x1 conv + global avg pool;
    # 1 + 4*2 + 1 = 10 conv layers, 9 activations), N = 2^16, 24 limbs
    "squeezenet": dict(log_n=16, q_bits=[60] + [40] * 23, p_bits=60, scale=2.0 ** 40, input=(3, 32, 32),
                       layers=[("conv", 64, 3, 1, 1), ("act",), ("avgpool",), ("fire", 16, 32, 32),
                               ("fire", 16, 32, 32), ("avgpool",), ("fire", 32, 64, 64), ("fire", 32, 64, 64),
                               ("conv", 10, 1, 1, 0), ("gap",)],
                       sigma=[0.05] * 14, act_gains=[4.0 ** 2] + [4.0 ** e for e in range(4, 12)]),
}


def linear_shapes(name: str):
    """Weight shapes of the net's conv / fc layers in order (OC, IC, K, K) / (OUT, IN)."""
    net = NETS[name]
    c, h, w = net["input"]
    shapes = []
    for layer in net["layers"]:
        if layer[0] == "conv":
            _, oc, k, s, p = layer[:5]
            shapes.append((oc, c, k, k))
            c, h, w = oc, (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        elif layer[0] == "avgpool":
            h, w = h // 2, w // 2
        elif layer[0] == "fc":
            shapes.append((layer[1], c * h * w))
            c, h, w = layer[1], 1, 1
        elif layer[0] == "fire":
            _, sq, e1, e3 = layer
            shapes += [(sq, c, 1, 1), (e1, sq, 1, 1), (e3, sq, 3, 3)]
            c = e1 + e3
        elif layer[0] == "gap":
            h, w = 1, 1
    return shapes


def net_weights(name: str, seed: int = 1000):
    """A34: N(0, sigma_i) float64 weights, layer i drawn from PCG64(seed + i)."""
    net = NETS[name]
    return [_weights(seed + i, shp, net["sigma"][i]) for i, shp in enumerate(linear_shapes(name))]


def net_image(name: str, seed: int = 0) -> np.ndarray:
    """A34: uniform[0, 1] (C, H, W) image from PCG64(seed) (stand-in for MNIST / CIFAR-10)."""
    return _image(seed, NETS[name]["input"])
