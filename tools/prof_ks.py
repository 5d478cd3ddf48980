"""ncu target: one batched (K4) rotation of B ciphertexts and one hoisted (K7) rotation at the
bench configuration, inside a cudaProfilerStart/Stop window (ncu --profile-from-start off)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_1810_00845_b200 import hisa as H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--log-n", type=int, default=16)
ap.add_argument("--limbs", type=int, default=24)
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--hoist-r", type=int, default=8)
a = ap.parse_args()
N = 1 << a.log_n
k = synth.rot_amount(0, a.log_n, a.limbs)
amts = sorted({int(x) for x in synth.rng(0, 11, a.log_n, a.limbs).integers(1, N // 2, size=a.hoist_r)})
ctx = H.Context(a.log_n, [50] * a.limbs, 60, seed=0)
ctx.keygen([k] + amts, False)
cts = [ctx.ct_random(b, a.limbs - 1) for b in range(a.batch)]
for _ in range(2):   # warm-up
    for h in ctx.rot_left_batch(cts, k):
        ctx.free(h)
ctx.sync()
torch.cuda.profiler.start()
for h in ctx.rot_left_batch(cts, k):
    ctx.free(h)
for h in ctx.rot_left_hoisted(cts[0], amts):
    ctx.free(h)
ctx.sync()
torch.cuda.profiler.stop()
ctx.close()
print("prof_ks ok")
