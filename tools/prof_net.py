"""Per-kernel profile of one encrypted inference (driver) on the GPU: kernel class, total ms,
launches -- where the latency of configs 1 / 3 / 4 / 5 goes."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from synth import nets as SN  # noqa: E402
from paper_1810_00845_b200 import hisa as H  # noqa: E402
from paper_1810_00845_b200.driver import EncryptedNet  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lenet_small"
net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 0)
ctx = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=0, arena_bytes=64 << 30)
plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, ctx.moduli)
EncryptedNet.keygen(ctx, plan)
en = EncryptedNet(ctx, net, W, SN.ACT_COEFFS)
cts, lay = en.encrypt_image(img)
out, _ = en.forward(cts, lay)       # warm-up (weight plaintexts encoded once)
ctx.sync()
for h in out:
    ctx.free(h)
layer_ms = []
ctx.profile(True)
torch.cuda.synchronize()
t0 = time.perf_counter()
ev = [torch.cuda.Event(enable_timing=True)]
ev[0].record()


def trace(li, hs, ly):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    ev.append(e)


out, _ = en.forward(cts, lay, trace=trace)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
prof = ctx.profile_read()
print(f"{name}: wall {wall * 1e3:.2f} ms, launches {ctx.launch_count()}")
for li, (a, b) in enumerate(zip(ev[:-1], ev[1:])):
    print(f"  layer {li} {net['layers'][li]}: {a.elapsed_time(b):.3f} ms")
tot = sum(v[0] for v in prof.values())
for n, (ms, c) in sorted(prof.items(), key=lambda kv: -kv[1][0]):
    print(f"  {n:24s} {ms:9.3f} ms {c:6d} launches  {100 * ms / tot:5.1f}%")
ctx.close()
