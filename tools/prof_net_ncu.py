"""ncu target for the network kernels: one LeNet-large forward (K7 multi, K8 conv accumulation,
mulPlain accumulation) inside a cudaProfilerStart/Stop window."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from synth import nets as SN  # noqa: E402
from paper_1810_00845_b200 import hisa as H  # noqa: E402
from paper_1810_00845_b200.driver import EncryptedNet  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "lenet_large"
net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 0)
ctx = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=0, arena_bytes=64 << 30)
plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, ctx.moduli)
EncryptedNet.keygen(ctx, plan)
en = EncryptedNet(ctx, net, W, SN.ACT_COEFFS)
cts, lay = en.encrypt_image(img)
out, _ = en.forward(cts, lay)
ctx.sync()
for h in out:
    ctx.free(h)
torch.cuda.profiler.start()
out, _ = en.forward(cts, lay)
ctx.sync()
torch.cuda.profiler.stop()
ctx.close()
print("prof_net_ncu ok")
