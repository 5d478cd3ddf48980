"""Encode throughput: GPU double-double encoder (hisa_encode_batch) at N = 2^15 / 2^16 on weight-like
(sparse) and dense slot vectors."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1810_00845_b200 import hisa as H  # noqa: E402

for log_n, L in ((15, 14), (16, 24)):
    g = H.Context(log_n, [60] + [40] * (L - 1), 60, seed=0, arena_bytes=16 << 30)
    rng = np.random.default_rng(0)
    dense = rng.uniform(0, 1, (64, g.slots))
    g.encode_batch(dense[:2], 2.0 ** 40, 5)
    g.sync()
    t0 = time.perf_counter()
    hs = g.encode_batch(dense, 2.0 ** 40, 5)
    g.sync()
    dt = time.perf_counter() - t0
    print(f"N=2^{log_n}: {len(hs) / dt:.0f} plaintexts/s ({dt / len(hs) * 1e3:.3f} ms each, 6 limbs)")
    g.close()
