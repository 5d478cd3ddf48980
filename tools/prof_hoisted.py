"""Per-kernel CUDA-event profile of one batched hoisted rotation (B ciphertexts x R amounts) at the
bench configuration; optional --lib side build (A/B of compile-time variants)."""
import argparse
import json
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
ap.add_argument("--r", type=int, default=8)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--lib", default=None)
a = ap.parse_args()
if a.lib:
    H.LIB_PATH = os.path.abspath(a.lib)
    H.load(build=False)
N = 1 << a.log_n
amts = sorted({int(x) for x in synth.rng(0, 11, a.log_n, a.limbs).integers(1, N // 2, size=a.r)})
ctx = H.Context(a.log_n, [50] * a.limbs, 60, seed=0)
ctx.keygen(amts, False)
cts = [ctx.ct_random(b, a.limbs - 1) for b in range(a.batch)]
for row in ctx.rot_left_hoisted_batch(cts, amts):
    for h in row:
        ctx.free(h)
ctx.sync()
st = torch.cuda.current_stream()
ctx.profile(True)
torch.cuda.profiler.start()   # ncu --profile-from-start off captures the timed iterations only
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(a.iters):
    for row in ctx.rot_left_hoisted_batch(cts, amts):
        for h in row:
            ctx.free(h)
e1.record(st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ms = e0.elapsed_time(e1) / a.iters
prof = ctx.profile_read()
print(json.dumps({"lib": a.lib or "default", "batch": a.batch, "R": len(amts), "ms_per_step": ms,
                  "rot_per_s": a.batch * len(amts) / (ms / 1e3),
                  "kernels": {k: [round(v[0] / a.iters, 4), v[1] // a.iters] for k, v in
                              sorted(prof.items(), key=lambda kv: -kv[1][0])}}))
ctx.close()
