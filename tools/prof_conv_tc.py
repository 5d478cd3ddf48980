"""ncu target: one K8 conv accumulation at a SqueezeNet-like shape (N = 2^16, 23 x 40-bit + one
60-bit limb, T = 144 inputs, OC = 64 outputs) inside a profiler window."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1810_00845_b200 import hisa as H  # noqa: E402

T, OC = int(sys.argv[1]) if len(sys.argv) > 1 else 144, int(sys.argv[2]) if len(sys.argv) > 2 else 64
g = H.Context(16, [60] + [40] * 15, 60, seed=0, arena_bytes=40 << 30)
hs = [g.ct_random(t, 15) for t in range(T)]
W = np.random.default_rng(0).normal(0, 0.05, (OC, T))
for _ in range(2):
    for h in g.conv_accumulate(hs, W.ravel()):
        g.free(h)
g.sync()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for h in g.conv_accumulate(hs, W.ravel()):
    g.free(h)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
macs = OC * T * 2 * 16 * 65536
print(f"T={T} OC={OC}: {ms:.3f} ms (incl. host weight prep), {macs / ms / 1e9:.2f} TMAC/s")
torch.cuda.profiler.start()
for h in g.conv_accumulate(hs, W.ravel()):
    g.free(h)
g.sync()
torch.cuda.profiler.stop()
