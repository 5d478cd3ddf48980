"""ctypes wrapper around ckks_oracle.c plus a HISA-shaped API (TEST INFRASTRUCTURE ONLY).

Every method cites the PAPER.md passage (P:n) or DESIGN.md reading (A<n>) it follows.
Scale / level bookkeeping follows reading A8; errors follow the HISA error kinds of
DESIGN.md "Boundary" (raised here as ``OracleError(code_name)``).
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ckks_oracle.c")
_LIB = os.path.join(_HERE, "libckks_oracle.so")

u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")

# ChaCha20 domain tags (A11)
TAG_SK, TAG_PK_A, TAG_PK_E, TAG_ENC_V, TAG_ENC_E0, TAG_ENC_E1 = 1, 2, 3, 4, 5, 6
TAG_KSK_A, TAG_KSK_E, TAG_BENCH, TAG_ROT_K = 7, 8, 9, 10


def build(force: bool = False) -> str:
    """Compile the oracle (plain gcc; no CUDA)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-shared", "-fPIC", "-o", _LIB, _SRC,
               "-lquadmath", "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, c_int, c_u64, c_i64, c_u32, c_d = (ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64,
                                               ctypes.c_int64, ctypes.c_uint32, ctypes.c_double)
        sig = {
            "orc_create": (vp, [c_int, c_int, ctypes.POINTER(c_int), c_int, c_int]),
            "orc_destroy": (None, [vp]),
            "orc_moduli": (None, [vp, u64p]),
            "orc_psis": (None, [vp, u64p]),
            "orc_ntt": (None, [vp, c_int, u64p]),
            "orc_intt": (None, [vp, c_int, u64p]),
            "orc_ntt_limbs": (None, [vp, u64p, c_int, c_int]),
            "orc_intt_limbs": (None, [vp, u64p, c_int, c_int]),
            "orc_chacha20_block": (None, [u32p, c_u32, u32p, u32p]),
            "orc_stream_u64": (None, [c_u64, c_u32, c_u64, c_u64, c_u64, u64p]),
            "orc_sample_uniform": (None, [vp, c_u64, c_u32, c_u64, c_u64, u64p]),
            "orc_sample_ternary": (None, [vp, c_u64, c_u32, c_u64, i64p]),
            "orc_sample_cbd": (None, [vp, c_u64, c_u32, c_u64, i64p]),
            "orc_keygen_secret": (None, [vp, c_u64, i64p, u64p]),
            "orc_keygen_public": (None, [vp, c_u64, u64p, u64p]),
            "orc_keygen_ksk": (None, [vp, c_u64, c_u64, u64p, u64p, u64p]),
            "orc_rot_target": (None, [vp, i64p, c_i64, u64p]),
            "orc_relin_target": (None, [vp, u64p, u64p]),
            "orc_galois_elt": (c_u64, [vp, c_i64]),
            "orc_automorphism_coeff_int": (None, [c_u64, c_u64, i64p, i64p]),
            "orc_automorphism_ntt_limb": (None, [vp, c_int, c_u64, u64p, u64p]),
            "orc_encrypt": (None, [vp, c_u64, c_u64, u64p, u64p, c_int, u64p]),
            "orc_decrypt": (None, [vp, u64p, u64p, c_int, c_int, u64p]),
            "orc_encode_coeffs": (c_int, [vp, f64p, c_u64, c_d, i64p]),
            "orc_encode": (c_int, [vp, f64p, c_u64, c_d, c_int, u64p]),
            "orc_decode": (None, [vp, u64p, c_d, c_u64, f64p]),
            "orc_add": (None, [vp, u64p, u64p, c_int, c_int, u64p]),
            "orc_sub": (None, [vp, u64p, u64p, c_int, c_int, u64p]),
            "orc_add_plain": (None, [vp, u64p, u64p, c_int, c_int, c_int, u64p]),
            "orc_mul_plain": (None, [vp, u64p, u64p, c_int, c_int, u64p]),
            "orc_mul_scalar_int": (None, [vp, u64p, c_i64, c_int, c_int, u64p]),
            "orc_add_scalar_int": (None, [vp, u64p, c_i64, c_int, c_int, u64p]),
            "orc_tensor": (None, [vp, u64p, u64p, c_int, u64p]),
            "orc_keyswitch": (None, [vp, u64p, c_int, u64p, u64p]),
            "orc_relinearize": (None, [vp, u64p, c_int, u64p, u64p]),
            "orc_rotate": (None, [vp, u64p, c_int, c_i64, u64p, u64p]),
            "orc_rescale": (None, [vp, u64p, c_int, c_int, u64p]),
            "orc_mod_switch": (None, [vp, u64p, c_int, c_int, c_int, u64p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(Exception):
    """Raised with one of the HISA error names."""

    def __init__(self, code: str, msg: str = ""):
        super().__init__(f"{code}: {msg}")
        self.code = code


def llround(x: float) -> int:
    """C llround: round half away from zero of a double, exactly (A20)."""
    if not math.isfinite(x):
        raise OracleError("PARAMS", "non-finite scalar")
    t = math.trunc(x)
    r = x - t          # exact in binary64
    if r >= 0.5:
        t += 1
    elif r <= -0.5:
        t -= 1
    return int(t)


@dataclass
class Pt:
    data: np.ndarray   # [(level+1), N] uint64 NTT form
    level: int
    scale: float


@dataclass
class Ct:
    data: np.ndarray   # [npolys, (level+1), N] uint64 NTT form
    level: int
    scale: float

    @property
    def npolys(self) -> int:
        return self.data.shape[0]


SCALE_RTOL = 2.0 ** -30   # A8


class Oracle:
    """Textbook RNS-CKKS with HISA semantics on the host.

    ``q_bits`` lists q_0..q_{L-1} bit sizes (bottom first), ``p_bits`` the single special prime
    (A3, A14, A29).  ``seed`` keys every ChaCha20 stream (A11).
    """

    def __init__(self, log_n: int, q_bits, p_bits: int, seed: int = 0, nthreads: int | None = None):
        self.lib = lib()
        self.log_n = log_n
        self.N = 1 << log_n
        self.slots = self.N // 2
        self.L = len(q_bits)
        self.seed = seed
        self.nthreads = nthreads or os.cpu_count() or 1
        arr = (ctypes.c_int * self.L)(*q_bits)
        self.ctx = self.lib.orc_create(log_n, self.L, arr, p_bits, self.nthreads)
        if not self.ctx:
            raise OracleError("PARAMS", "orc_create failed")
        m = np.zeros(self.L + 1, dtype=np.uint64)
        self.lib.orc_moduli(self.ctx, m)
        self.moduli = [int(v) for v in m]
        self.q = self.moduli[: self.L]
        self.p = self.moduli[self.L]
        ps = np.zeros(self.L + 1, dtype=np.uint64)
        self.lib.orc_psis(self.ctx, ps)
        self.psi = [int(v) for v in ps]
        self.enc_counter = 0
        self.s_int = None
        self.s_ntt = None
        self.pk = None
        self.rlk = None
        self.rot_keys: dict[int, np.ndarray] = {}

    def __del__(self):
        try:
            if getattr(self, "ctx", None):
                self.lib.orc_destroy(self.ctx)
                self.ctx = None
        except Exception:
            pass

    # ---------------------------------------------------------------- primitives
    def ntt(self, a: np.ndarray, midx0: int = 0) -> np.ndarray:
        """a1: forward negacyclic NTT per limb (A5); a is [limbs, N]."""
        x = np.ascontiguousarray(a, dtype=np.uint64).copy()
        x2 = x.reshape(-1, self.N)
        self.lib.orc_ntt_limbs(self.ctx, x2, x2.shape[0], midx0)
        return x2.reshape(a.shape)

    def intt(self, a: np.ndarray, midx0: int = 0) -> np.ndarray:
        """a2: inverse NTT per limb."""
        x = np.ascontiguousarray(a, dtype=np.uint64).copy()
        x2 = x.reshape(-1, self.N)
        self.lib.orc_intt_limbs(self.ctx, x2, x2.shape[0], midx0)
        return x2.reshape(a.shape)

    def norm_rot(self, k: int) -> int:
        return k % self.slots

    def galois(self, k: int) -> int:
        return int(self.lib.orc_galois_elt(self.ctx, k))

    # ---------------------------------------------------------------- keys
    def keygen(self, rot_amounts=(), relin: bool = True):
        N, L = self.N, self.L
        self.s_int = np.zeros(N, dtype=np.int64)
        self.s_ntt = np.zeros((L + 1, N), dtype=np.uint64)
        self.lib.orc_keygen_secret(self.ctx, self.seed, self.s_int, self.s_ntt)
        self.pk = np.zeros((2, L, N), dtype=np.uint64)
        self.lib.orc_keygen_public(self.ctx, self.seed, self.s_ntt, self.pk)
        if relin:
            sp = np.zeros((L + 1, N), dtype=np.uint64)
            self.lib.orc_relin_target(self.ctx, self.s_ntt, sp)
            self.rlk = self._ksk(0, sp)
        for k in rot_amounts:
            self.add_rot_key(k)

    def _ksk(self, keyid: int, sp: np.ndarray) -> np.ndarray:
        L, N = self.L, self.N
        out = np.zeros((L, 2, L + 1, N), dtype=np.uint64)
        self.lib.orc_keygen_ksk(self.ctx, self.seed, keyid, self.s_ntt, np.ascontiguousarray(sp), out)
        return out

    def add_rot_key(self, k: int):
        """One key per distinct left-rotation amount (A15); keyid = k mod s."""
        kk = self.norm_rot(k)
        if kk == 0 or kk in self.rot_keys:
            return
        sp = np.zeros((self.L + 1, self.N), dtype=np.uint64)
        self.lib.orc_rot_target(self.ctx, self.s_int, kk, sp)
        self.rot_keys[kk] = self._ksk(kk, sp)

    # ---------------------------------------------------------------- encode / decode
    def encode_coeffs(self, z, scale: float) -> np.ndarray:
        z = np.ascontiguousarray(z, dtype=np.float64)
        if z.size > self.slots:
            raise OracleError("CAPACITY", "n > N/2")
        m = np.zeros(self.N, dtype=np.int64)
        if self.lib.orc_encode_coeffs(self.ctx, z, z.size, float(scale), m) != 0:
            raise OracleError("PARAMS", "encoded coefficient >= 2^62")
        return m

    def encode(self, z, scale: float, level: int | None = None) -> Pt:
        level = self.L - 1 if level is None else level
        z = np.ascontiguousarray(z, dtype=np.float64)
        if z.size > self.slots:
            raise OracleError("CAPACITY", "n > N/2")
        pt = np.zeros((level + 1, self.N), dtype=np.uint64)
        if self.lib.orc_encode(self.ctx, z, z.size, float(scale), level, pt) != 0:
            raise OracleError("PARAMS", "encoded coefficient >= 2^62")
        return Pt(pt, level, float(scale))

    def pt_from_int_coeffs(self, m: np.ndarray, scale: float, level: int) -> Pt:
        """Plaintext from integer coefficients (reduced per prime, then NTT)."""
        rows = []
        for i in range(level + 1):
            q = self.q[i]
            rows.append(np.array([int(v) % q for v in m], dtype=np.uint64))
        return Pt(self.ntt(np.stack(rows)), level, float(scale))

    def decode(self, pt: Pt, n: int | None = None) -> np.ndarray:
        n = self.slots if n is None else n
        z = np.zeros(n, dtype=np.float64)
        self.lib.orc_decode(self.ctx, np.ascontiguousarray(pt.data[0]), pt.scale, n, z)
        return z

    # ---------------------------------------------------------------- encryption profile
    def encrypt(self, pt: Pt) -> Ct:
        """Public-key encryption at the plaintext's level (A12); one counter step per call."""
        ct = np.zeros((2, pt.level + 1, self.N), dtype=np.uint64)
        self.lib.orc_encrypt(self.ctx, self.seed, self.enc_counter, self.pk, np.ascontiguousarray(pt.data),
                             pt.level, ct)
        self.enc_counter += 1
        return Ct(ct, pt.level, pt.scale)

    def decrypt(self, ct: Ct) -> Pt:
        pt = np.zeros((ct.level + 1, self.N), dtype=np.uint64)
        self.lib.orc_decrypt(self.ctx, self.s_ntt, np.ascontiguousarray(ct.data), ct.npolys, ct.level, pt)
        return Pt(pt, ct.level, ct.scale)

    def copy(self, ct: Ct) -> Ct:
        return Ct(ct.data.copy(), ct.level, ct.scale)

    # ---------------------------------------------------------------- integers profile
    def _check_pair(self, a: Ct, b):
        if a.level != b.level:
            raise OracleError("LEVEL_MISMATCH", f"{a.level} vs {b.level}")
        if abs(a.scale / b.scale - 1.0) > SCALE_RTOL:
            raise OracleError("SCALE_MISMATCH", f"{a.scale} vs {b.scale}")

    def _need2(self, a: Ct):
        if a.npolys != 2:
            raise OracleError("NOT_RELINEARIZED", "3-poly ciphertext")

    def add(self, a: Ct, b: Ct, sign: int = 1) -> Ct:
        self._check_pair(a, b)
        if a.npolys != b.npolys:
            raise OracleError("NOT_RELINEARIZED", "poly count mismatch")
        out = np.zeros_like(a.data)
        f = self.lib.orc_add if sign > 0 else self.lib.orc_sub
        f(self.ctx, np.ascontiguousarray(a.data), np.ascontiguousarray(b.data), a.npolys, a.level, out)
        return Ct(out, a.level, a.scale)

    def sub(self, a: Ct, b: Ct) -> Ct:
        return self.add(a, b, -1)

    def add_plain(self, a: Ct, p: Pt, sign: int = 1) -> Ct:
        self._need2(a)
        self._check_pair(a, p)
        out = np.zeros_like(a.data)
        self.lib.orc_add_plain(self.ctx, np.ascontiguousarray(a.data), np.ascontiguousarray(p.data), a.npolys,
                               a.level, sign, out)
        return Ct(out, a.level, a.scale)

    def sub_plain(self, a: Ct, p: Pt) -> Ct:
        return self.add_plain(a, p, -1)

    def add_scalar(self, a: Ct, x: float, sign: int = 1) -> Ct:
        """x encoded at the ciphertext's scale: X = llround(x * scale) (A20)."""
        self._need2(a)
        X = llround(float(x) * a.scale) * sign
        if abs(X) >= 1 << 62:
            raise OracleError("PARAMS", "scalar too large")
        out = np.zeros_like(a.data)
        self.lib.orc_add_scalar_int(self.ctx, np.ascontiguousarray(a.data), X, a.npolys, a.level, out)
        return Ct(out, a.level, a.scale)

    def sub_scalar(self, a: Ct, x: float) -> Ct:
        return self.add_scalar(a, x, -1)

    def mul_plain(self, a: Ct, p: Pt) -> Ct:
        self._need2(a)
        if a.level != p.level:
            raise OracleError("LEVEL_MISMATCH", "")
        out = np.zeros_like(a.data)
        self.lib.orc_mul_plain(self.ctx, np.ascontiguousarray(a.data), np.ascontiguousarray(p.data), a.npolys,
                               a.level, out)
        return Ct(out, a.level, a.scale * p.scale)

    def scalar_int(self, a: Ct, x: float, pt_scale: float = 0.0) -> tuple[int, float]:
        """A8/A20: pt_scale 0 means (double) q_top of the ciphertext."""
        ps = float(self.q[a.level]) if pt_scale == 0.0 else float(pt_scale)
        X = llround(float(x) * ps)
        if abs(X) >= 1 << 62:
            raise OracleError("PARAMS", "scalar too large")
        return X, ps

    def mul_scalar(self, a: Ct, x: float, pt_scale: float = 0.0) -> Ct:
        self._need2(a)
        X, ps = self.scalar_int(a, x, pt_scale)
        out = np.zeros_like(a.data)
        self.lib.orc_mul_scalar_int(self.ctx, np.ascontiguousarray(a.data), X, a.npolys, a.level, out)
        return Ct(out, a.level, a.scale * ps)

    def mul_norelin(self, a: Ct, b: Ct) -> Ct:
        """Relin profile: 3-poly tensor product."""
        self._need2(a)
        self._need2(b)
        if a.level != b.level:
            raise OracleError("LEVEL_MISMATCH", "")
        out = np.zeros((3, a.level + 1, self.N), dtype=np.uint64)
        self.lib.orc_tensor(self.ctx, np.ascontiguousarray(a.data), np.ascontiguousarray(b.data), a.level, out)
        return Ct(out, a.level, a.scale * b.scale)

    def relinearize(self, a: Ct) -> Ct:
        if a.npolys == 2:
            return self.copy(a)
        if self.rlk is None:
            raise OracleError("NO_KEY", "relinearisation key")
        out = np.zeros((2, a.level + 1, self.N), dtype=np.uint64)
        self.lib.orc_relinearize(self.ctx, np.ascontiguousarray(a.data), a.level, self.rlk, out)
        return Ct(out, a.level, a.scale)

    def mul(self, a: Ct, b: Ct) -> Ct:
        return self.relinearize(self.mul_norelin(a, b))

    def keyswitch(self, d: np.ndarray, level: int, key: np.ndarray) -> np.ndarray:
        out = np.zeros((2, level + 1, self.N), dtype=np.uint64)
        self.lib.orc_keyswitch(self.ctx, np.ascontiguousarray(d, dtype=np.uint64), level, key, out)
        return out

    def rot_left(self, a: Ct, k: int) -> Ct:
        """P:478-487 / A15: out[i] = in[(i + k) mod s]; k = 0 is a copy."""
        self._need2(a)
        kk = self.norm_rot(k)
        if kk == 0:
            return self.copy(a)
        if kk not in self.rot_keys:
            raise OracleError("NO_KEY", f"rotation {kk}")
        out = np.zeros_like(a.data)
        self.lib.orc_rotate(self.ctx, np.ascontiguousarray(a.data), a.level, kk, self.rot_keys[kk], out)
        return Ct(out, a.level, a.scale)

    def rot_right(self, a: Ct, k: int) -> Ct:
        """right rotations are left rotations by s - k."""
        return self.rot_left(a, self.slots - self.norm_rot(k))

    # ---------------------------------------------------------------- division profile
    def max_scalar_div(self, a: Ct, ub: int) -> int:
        """A18: q_top if q_top <= ub else 1."""
        qt = self.q[a.level]
        return qt if qt <= ub else 1

    def div_scalar(self, a: Ct, d: int) -> Ct:
        if d == 1:
            return self.copy(a)
        if a.level == 0:
            raise OracleError("MODULUS_EXHAUSTED", "")
        if d != self.q[a.level]:
            raise OracleError("INVALID_DIVISOR", str(d))
        return self.rescale(a)

    def rescale(self, a: Ct) -> Ct:
        if a.level == 0:
            raise OracleError("MODULUS_EXHAUSTED", "")
        out = np.zeros((a.npolys, a.level, self.N), dtype=np.uint64)
        self.lib.orc_rescale(self.ctx, np.ascontiguousarray(a.data), a.npolys, a.level, out)
        return Ct(out, a.level - 1, a.scale / float(self.q[a.level]))

    def mod_switch(self, a: Ct, drop: int = 1) -> Ct:
        """A19: drop the top limb(s), scale unchanged."""
        if drop < 0 or a.level - drop < 0:
            raise OracleError("MODULUS_EXHAUSTED", "")
        return Ct(a.data[:, : a.level + 1 - drop].copy(), a.level - drop, a.scale)

    def bootstrap(self, a: Ct):
        raise OracleError("UNSUPPORTED_PROFILE", "bootstrap (P:292-293)")

    # ---------------------------------------------------------------- bench inputs (A11 tag BENCH)
    def bench_ct(self, b: int, level: int, npolys: int = 2) -> Ct:
        """Uniform residues (not a valid encryption): limb (b, poly, i) from stream index
        b<<32 | poly<<16 | i, tag BENCH (config 2)."""
        out = np.zeros((npolys, level + 1, self.N), dtype=np.uint64)
        for p in range(npolys):
            for i in range(level + 1):
                self.lib.orc_sample_uniform(self.ctx, self.seed, TAG_BENCH, (b << 32) | (p << 16) | i, self.q[i],
                                            out[p, i])
        return Ct(out, level, 2.0 ** 40)

    def bench_pt(self, b: int, level: int) -> Pt:
        """Uniform plaintext residues: stream index b<<32 | 0xFFFF<<16 | i."""
        out = np.zeros((level + 1, self.N), dtype=np.uint64)
        for i in range(level + 1):
            self.lib.orc_sample_uniform(self.ctx, self.seed, TAG_BENCH, (b << 32) | (0xFFFF << 16) | i, self.q[i],
                                        out[i])
        return Pt(out, level, 2.0 ** 40)
