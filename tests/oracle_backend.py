"""A host-memory test double of the libhisa Context API on the CPU oracle (TESTS ONLY).

It lets the product driver (paper_1810_00845_b200/driver.py) and its multi-GPU exchange
(parallel.py) run numerically on a CPU box: tests/test_parallel_cpu.py shards a network over
gloo ranks (world 2 / 4 / 8) and checks the outputs are bit-identical to the one-rank run.
Every operation is the oracle's plain per-ciphertext HISA op (oracle/ckks.py), so this class
holds no batching, fusion or kernel logic of its own; the "device" views are numpy arrays whose
addresses parallel.py wraps as host tensors (`host_memory = True`).
"""
from __future__ import annotations

import ctypes

import numpy as np

from oracle.ckks import Ct, Oracle, Pt


class OracleBackend:
    host_memory = True

    def __init__(self, log_n, q_bits, p_bits, seed=0, nthreads=1):
        self.o = Oracle(log_n, q_bits, p_bits, seed=seed, nthreads=nthreads)
        self.slots = self.o.slots
        self.moduli = self.o.moduli
        self.q = list(self.o.q)
        self.objs = {}
        self.next = 1

    # ---- handles
    def _put(self, x):
        h = self.next
        self.next += 1
        self.objs[h] = x
        return h

    def free(self, h):
        self.objs.pop(h, None)

    def ct_info(self, h):
        c = self.objs[h]
        return c.level, c.npolys, c.scale

    # ---- keys / client
    def keygen(self, rots, relin=True, max_level=-1):
        # the oracle keeps full keys; a truncated key holds the same words on the levels it serves
        if getattr(self, "_keyed", False) and not relin:
            for k in rots:
                self.o.add_rot_key(k)
            return
        self.o.keygen(rot_amounts=list(rots), relin=relin)
        self._keyed = True

    def encode(self, v, scale, level=-1):
        return self._put(self.o.encode(np.asarray(v, dtype=np.float64), scale, None if level < 0 else level))

    def encode_batch(self, vs, scale, level=-1):
        return [self.encode(v, scale, level) for v in vs]

    def encrypt(self, pt):
        return self._put(self.o.encrypt(self.objs[pt]))

    def decrypt(self, ct):
        return self._put(self.o.decrypt(self.objs[ct]))

    def decode(self, pt, n):
        return self.o.decode(self.objs[pt])[:n]

    # ---- HISA ops (one oracle call per ciphertext)
    def copy(self, h):
        return self._put(self.o.copy(self.objs[h]))

    def add(self, a, b):
        return self._put(self.o.add(self.objs[a], self.objs[b]))

    def add_scalar(self, a, x):
        return self._put(self.o.add_scalar(self.objs[a], x))

    def mul_plain(self, a, p):
        return self._put(self.o.mul_plain(self.objs[a], self.objs[p]))

    def mul_batch(self, a, b):
        return [self._put(self.o.mul(self.objs[x], self.objs[y])) for x, y in zip(a, b)]

    def rescale_batch(self, hs):
        return [self._put(self.o.rescale(self.objs[h])) for h in hs]

    def rot_left_batch(self, hs, k):
        return [self._put(self.o.rot_left(self.objs[h], k)) for h in hs]

    def rot_left_hoisted_batch(self, hs, ks):
        return [[self._put(self.o.rot_left(self.objs[h], k)) for k in ks] for h in hs]

    def rot_add_batch(self, hs, k):
        return [self._put(self.o.add(self.objs[h], self.o.rot_left(self.objs[h], k))) for h in hs]

    def _sum_scalar(self, hs, row):
        acc = None
        for h, w in zip(hs, row):
            t = self.o.mul_scalar(self.objs[h], float(w))
            acc = t if acc is None else self.o.add(acc, t)
        return acc

    def conv_accumulate(self, hs, W, pt_scale=0.0):
        W = np.asarray(W, dtype=np.float64).reshape(-1, len(hs))
        return [self._put(self._sum_scalar(hs, row)) for row in W]

    def mul_plain_accumulate(self, hs, pts, J):
        C = len(hs)
        out = []
        for j in range(J):
            acc = None
            for c in range(C):
                t = self.o.mul_plain(self.objs[hs[c]], self.objs[pts[j * C + c]])
                acc = t if acc is None else self.o.add(acc, t)
            out.append(self._put(acc))
        return out

    # ---- host-memory "device" views (parallel.py)
    @staticmethod
    def _array(ptr, words):
        return np.ctypeslib.as_array((ctypes.c_uint64 * words).from_address(ptr))

    def ct_device_view(self, h):
        c = self.objs[h]
        c.data = np.ascontiguousarray(c.data)
        return c.data.ctypes.data, c.data.size

    def ct_adopt_device(self, ptr, level, npolys, scale):
        N = 2 * self.slots
        d = self._array(ptr, npolys * (level + 1) * N).copy().reshape(npolys, level + 1, N)
        return self._put(Ct(d, level, scale))

    def ct_adopt_sum(self, ptr, level, npolys, scale):
        """Partial sums (int64, each < 2^63) reduced mod q_i."""
        N = 2 * self.slots
        d = self._array(ptr, npolys * (level + 1) * N).reshape(npolys, level + 1, N)
        out = np.empty_like(d)
        for i in range(level + 1):
            out[:, i] = d[:, i] % np.uint64(self.q[i])
        return self._put(Ct(out, level, scale))

    def conv_accumulate_dev(self, hs, W, ptr, pt_scale=0.0):
        W = np.asarray(W, dtype=np.float64).reshape(-1, len(hs))
        lv = self.objs[hs[0]].level
        N = 2 * self.slots
        per = 2 * (lv + 1) * N
        buf = self._array(ptr, W.shape[0] * per)
        for o, row in enumerate(W):
            buf[o * per:(o + 1) * per] = self._sum_scalar(hs, row).data.ravel()

    def close(self):
        self.objs.clear()


__all__ = ["OracleBackend", "Pt", "Ct"]
