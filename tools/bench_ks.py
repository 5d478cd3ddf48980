"""Time the batched (K4) rotation at the bench configuration; prints one JSON line with the
per-kernel profile (used to compare compile-time variants built with _build.py OUT.so DEFS)."""
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
ap.add_argument("--iters", type=int, default=6)
ap.add_argument("--lib", default=None, help="a side build of libhisa.so (paper_1810_00845_b200/_build.py OUT DEFS)")
a = ap.parse_args()
if a.lib:
    H.LIB_PATH = os.path.abspath(a.lib)
    H.load(build=False)
k = synth.rot_amount(0, a.log_n, a.limbs)
ctx = H.Context(a.log_n, [50] * a.limbs, 60, seed=0)
ctx.keygen([k], False)
cts = [ctx.ct_random(b, a.limbs - 1) for b in range(a.batch)]
ref = ctx.ct_export(ctx.rot_left_batch(cts[:1], k)[0])
for _ in range(2):
    for h in ctx.rot_left_batch(cts, k):
        ctx.free(h)
ctx.sync()
ctx.profile(True)
st = torch.cuda.current_stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(a.iters):
    outs = ctx.rot_left_batch(cts, k)
    for h in outs[1:]:
        ctx.free(h)
    last = outs[0]
e1.record(st)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
prof = ctx.profile_read()
ok = bool((ctx.ct_export(last) == ref).all())
print(json.dumps({"lib": a.lib or "default", "ok": ok,
                  "ms_per_batch": ms, "rot_s": a.batch / (ms / 1e3),
                  "kernels": {n: round(v[0] / a.iters, 4) for n, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}}))
ctx.close()
