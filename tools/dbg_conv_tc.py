"""Debug harness for the tensor-core K8 path: known inputs / weights, print output patterns."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1810_00845_b200 import hisa as H  # noqa: E402

g = H.Context(10, [60, 40, 40], 60, seed=1, arena_bytes=1 << 30)
N = 1024
L = 3


def run(data, W, T, label):
    hs = [g.ct_import(d, L - 1, 2, 1.0) for d in data]
    outs = g.conv_accumulate(hs, np.asarray(W, dtype=np.float64).ravel(), 1.0)
    res = [g.ct_export(h) for h in outs]
    print(label, "out[0][poly0][limb1][0:12] =", res[0][0, 1, :12].tolist())
    return res


# 1) T=1, OC=1, weight 1, input = 1 everywhere
d = np.ones((2, L, N), dtype=np.uint64)
run([d], [[1.0]], 1, "ones*1")
# 2) input = row index x, weight 1
d = np.tile(np.arange(N, dtype=np.uint64), (2, L, 1))
run([d], [[1.0]], 1, "x*1")
# 3) input = 1, weight 2
d = np.ones((2, L, N), dtype=np.uint64)
run([d], [[2.0]], 1, "ones*2")
# 4) input = 256, weight 1  (byte plane 1)
d = np.full((2, L, N), 256, dtype=np.uint64)
run([d], [[1.0]], 1, "256*1")
# 5) input = 1, weight 256
d = np.ones((2, L, N), dtype=np.uint64)
run([d], [[256.0]], 1, "ones*256")
# 6) two inputs t=0 (1) and t=1 (10), weights (1, 100)
run([np.ones((2, L, N), dtype=np.uint64), np.full((2, L, N), 10, dtype=np.uint64)], [[1.0, 100.0]], 2, "t2")
# 7) OC=2: weights [[1],[3]]
res = run([np.ones((2, L, N), dtype=np.uint64)], [[1.0], [3.0]], 1, "oc2")
print("   oc1:", res[1][0, 1, :8].tolist())


def check(data, W, label):
    W = np.asarray(W, dtype=np.float64)
    OC, T = W.shape
    res = run(data, W, T, label)
    nbad = 0
    for o in range(OC):
        for p in range(2):
            for i in range(L):
                ref = [sum(int(W[o, t]) % q[i] * int(data[t][p, i, x]) for t in range(T)) % q[i] for x in range(N)]
                got = res[o][p, i].tolist()
                bad = [x for x in range(N) if got[x] != ref[x]]
                if bad and nbad < 4:
                    x = bad[0]
                    print(f"   o{o} p{p} limb{i}: {len(bad)} bad, x={x} got={got[x]} ref={ref[x]} diff={(got[x]-ref[x]) % q[i]}")
                nbad += len(bad)
    print("  ", label, "bad words:", nbad)


rng = np.random.default_rng(0)
q = g.moduli[:L]
rnd = lambda: np.stack([np.stack([rng.integers(0, q[i], N, dtype=np.uint64) for i in range(L)]) for _p in range(2)])
one = np.ones((2, L, N), dtype=np.uint64)
check([rnd()], [[1.0]], "rand_in*1")
check([one], [[-1.0]], "one*(-1)")
check([one], [[123456789.0]], "one*123456789")
check([rnd(), rnd()], [[1.0, 1.0]], "rand2*1")
check([one], [[float(1 << 33)]], "one*2^33")
# 8) random full residues, random signed integer weights, T=5, OC=3: compare with big ints
rng = np.random.default_rng(0)
q = g.moduli[:L]
T, OC = 5, 3
data = [np.stack([np.stack([rng.integers(0, q[i], N, dtype=np.uint64) for i in range(L)]) for _p in range(2)])
        for _t in range(T)]
W = rng.integers(-1000, 1000, (OC, T)).astype(np.float64)
res = run(data, W, T, "rand")
for o in range(OC):
    for p in range(2):
        for i in range(L):
            ref = [sum(int(W[o, t]) % q[i] * int(data[t][p, i, x]) for t in range(T)) % q[i] for x in range(N)]
            got = res[o][p, i].tolist()
            bad = [x for x in range(N) if got[x] != ref[x]]
            if bad:
                x = bad[0]
                print(f"o{o} p{p} limb{i} q={q[i]}: {len(bad)} bad, x={x} got={got[x]} ref={ref[x]}")
print("rand check done")
# 9) single big input value per limb with weight 1
for v in (1 << 32, 1 << 40, (1 << 56) + 5):
    d = np.full((2, L, N), v, dtype=np.uint64)
    d[:, 1:, :] %= np.array(q[1:], dtype=np.uint64)[:, None]
    r = run([d], [[1.0]], 1, f"v={v}")
    print("   limb0:", r[0][0, 0, :4].tolist(), "expect", v % q[0])
