"""Float64 plaintext evaluation of the synthetic CNNs (TEST INFRASTRUCTURE ONLY).

The reference the decrypted outputs are held to (max-abs 1e-3, BASELINE.json north star,
A36).  It is the plain definition of each tensor operation of the paper's tensor circuits
(convolution, matmul, pooling, elementwise activation), with the activation NOT
folded (A25 folding is an encrypted-side rewrite, checked against this unfolded form):
    conv    out[o, y, x] = sum_{c, i, j} W[o, c, i, j] * xpad[c, s*y + i, s*x + j]
    act     a0 + a1 x + a2 x^2          ("f(x) = ax^2 + bx", config coefficients A25)
    square  x^2                         (config 1)
    avgpool mean over 2x2 windows, stride 2 (max-pool replaced by average pool)
    fc      W @ flatten(x), flatten order (c, y, x)
    fire    SqueezeNet module: s = act(conv1x1(x)); concat(act(conv1x1(s)), act(conv3x3 SAME(s)))
    gap     mean over H x W
"""
from __future__ import annotations

import numpy as np


def conv2d(x: np.ndarray, w: np.ndarray, stride: int, pad: int) -> np.ndarray:
    c, h, wd = x.shape
    oc, ic, k, _ = w.shape
    assert ic == c
    xp = np.zeros((c, h + 2 * pad, wd + 2 * pad))
    xp[:, pad:pad + h, pad:pad + wd] = x
    ho = (h + 2 * pad - k) // stride + 1
    wo = (wd + 2 * pad - k) // stride + 1
    out = np.zeros((oc, ho, wo))
    for o in range(oc):
        for y in range(ho):
            for xx in range(wo):
                win = xp[:, stride * y:stride * y + k, stride * xx:stride * xx + k]
                out[o, y, xx] = float(np.sum(w[o] * win))
    return out


def act(x: np.ndarray, coeffs) -> np.ndarray:
    a0, a1, a2 = coeffs
    return a0 + a1 * x + a2 * x * x


def avgpool2(x: np.ndarray) -> np.ndarray:
    c, h, w = x.shape
    return x[:, :h // 2 * 2, :w // 2 * 2].reshape(c, h // 2, 2, w // 2, 2).mean(axis=(2, 4))


def forward(net: dict, image: np.ndarray, weights, act_coeffs, trace=None) -> np.ndarray:
    """Evaluate the network on one (C, H, W) image; returns the final activations (flattened
    for FC outputs, (C, H, W) otherwise).  `trace` (a list, optional) receives (layer index,
    output of that layer) after every layer."""
    x = np.asarray(image, dtype=np.float64)
    wi = 0
    for layer in net["layers"]:
        kind = layer[0]
        if kind == "conv":
            _, _oc, _k, s, p = layer[:5]
            x = conv2d(x, weights[wi], s, p)
            wi += 1
        elif kind == "act":
            x = act(x, act_coeffs)
        elif kind == "square":
            x = x * x
        elif kind == "avgpool":
            x = avgpool2(x)
        elif kind == "fc":
            x = weights[wi] @ x.reshape(-1)
            wi += 1
        elif kind == "fire":
            _, _sq, _e1, _e3 = layer
            sq = act(conv2d(x, weights[wi], 1, 0), act_coeffs)
            e1 = act(conv2d(sq, weights[wi + 1], 1, 0), act_coeffs)
            e3 = act(conv2d(sq, weights[wi + 2], 1, 1), act_coeffs)
            x = np.concatenate([e1, e3], axis=0)
            wi += 3
        elif kind == "gap":
            x = x.mean(axis=(1, 2))
        else:
            raise ValueError(kind)
        if trace is not None:
            trace.append((len(trace), x))
    return x
