"""Derive the compile-time activation gains (A41) of the synthetic networks.

CHET's compiler chooses the fixed-point scaling of every tensor (the scale
must keep values "sufficiently larger" than the CKKS error).  Here the scale Delta = 2^40 and the
40-bit primes are fixed by the configs, so the knob left is a per-activation gain G (a power of
4): the encrypted tensor after activation n holds G_n times its float64 value.  Rule:

    e_n = max(0, floor(log4(T / m_n))),  G_n = 4^e_n,  T = 16,

m_n = max |output of activation n| of the float64 network (oracle/plain.py, the unfolded
definition) on a CALIBRATION image (seed 1000 + 7, never a test or bench image).  The result is
written into synth/nets.py by hand ("act_gains"); tests/test_driver_host.py re-runs this rule and
checks the stored values.

Usage: python tools/calibrate_gains.py [net ...]
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import plain          # noqa: E402  (float64 definition only)
from synth import nets as SN      # noqa: E402

TARGET = 16.0
CALIB_SEED = 1007


def act_maxima(net, weights, image, coeffs):
    """max |activation output| of every activation, execution order (fire: squeeze, expand)."""
    x = np.asarray(image, dtype=np.float64)
    wi, out = 0, []
    for layer in net["layers"]:
        kind = layer[0]
        if kind == "conv":
            x = plain.conv2d(x, weights[wi], layer[3], layer[4])
            wi += 1
        elif kind == "fc":
            x = weights[wi] @ x.reshape(-1)
            wi += 1
        elif kind == "act":
            x = plain.act(x, coeffs)
            out.append(float(np.abs(x).max()))
        elif kind == "square":
            x = x * x
        elif kind == "avgpool":
            x = plain.avgpool2(x)
        elif kind == "gap":
            x = x.mean(axis=(1, 2))
        elif kind == "fire":
            s = plain.act(plain.conv2d(x, weights[wi], 1, 0), coeffs)
            e1 = plain.act(plain.conv2d(s, weights[wi + 1], 1, 0), coeffs)
            e3 = plain.act(plain.conv2d(s, weights[wi + 2], 1, 1), coeffs)
            x = np.concatenate([e1, e3], axis=0)
            out += [float(np.abs(s).max()), float(np.abs(x).max())]
            wi += 3
    return out


def gains_for(net, weights, image, coeffs=SN.ACT_COEFFS):
    return [4.0 ** max(0, math.floor(math.log(TARGET / m, 4))) for m in act_maxima(net, weights, image, coeffs)]


def main(names):
    for name in names:
        net = SN.NETS[name]
        img = SN._image(CALIB_SEED, net["input"])
        g = gains_for(net, SN.net_weights(name), img)
        print(name, "[" + ", ".join(f"4.0 ** {int(round(math.log(x, 4)))}" for x in g) + "]")


if __name__ == "__main__":
    main(sys.argv[1:] or ["lenet_small", "lenet_large", "squeezenet"])
