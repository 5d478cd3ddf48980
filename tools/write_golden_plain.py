"""Write tests/golden/plain_outputs.json: the float64 network outputs (oracle/plain.py, the
unfolded definition) of every synthetic network on image seeds 0..19 -- the reference bench.py's
inference entries report their decrypted error against (20 images).  Calls only
oracle/ and synth/ (the stored values never come from the CUDA path).

Usage: python tools/write_golden_plain.py
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import plain          # noqa: E402
from synth import nets as SN      # noqa: E402

NETS = ["tiny", "lenet_small", "lenet_large", "lenet_large_chw", "squeezenet"]
IMAGES = 20


def main():
    out = {"source": "oracle/plain.py float64 forward, weights synth.nets.net_weights(name), "
                     "images synth.nets.net_image(name, seed)", "images": IMAGES, "outputs": {}}
    for name in NETS:
        W = SN.net_weights(name)
        out["outputs"][name] = [plain.forward(SN.NETS[name], SN.net_image(name, s), W, SN.ACT_COEFFS).ravel().tolist()
                                for s in range(IMAGES)]
    path = os.path.join(ROOT, "tests", "golden", "plain_outputs.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print(path)


if __name__ == "__main__":
    main()
