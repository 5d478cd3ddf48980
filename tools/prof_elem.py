"""ncu target (--profile-from-start off): the HBM-bound kernels at the bench configuration
(N = 2^16, L = 24): mulPlain, add, tensor (mulNoRelin), mulPlain-accumulate (FC: C = 16 inputs,
J = 8 neurons), each launched once inside the profiler window."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1810_00845_b200 import hisa as H  # noqa: E402

L = 24
ctx = H.Context(16, [50] * L, 60, seed=0)
cts = [ctx.ct_random(b, L - 1) for b in range(16)]
pts = [ctx.pt_random(100 + b, L - 1) for b in range(16 * 8)]
for _ in range(2):   # warm-up
    for h in [ctx.mul_plain(cts[0], pts[0]), ctx.add(cts[0], cts[1]), ctx.mul_norelin(cts[0], cts[1])]:
        ctx.free(h)
    for h in ctx.mul_plain_accumulate(cts, pts, 8):
        ctx.free(h)
ctx.sync()
torch.cuda.profiler.start()
outs = [ctx.mul_plain(cts[0], pts[0]), ctx.add(cts[0], cts[1]), ctx.mul_norelin(cts[0], cts[1])]
outs += ctx.mul_plain_accumulate(cts, pts, 8)
ctx.sync()
torch.cuda.profiler.stop()
ctx.close()
print("prof_elem ok")
