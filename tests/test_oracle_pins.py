"""Pins for the CPU oracle (-m "not gpu").

Each test fixes the oracle to something other than itself: a mathematical definition evaluated
with Python big integers at tiny N, a closed form, an invariant, a library routine, or a value
printed in the paper/spec (tests/golden, cited).  See DESIGN.md "Pins".
"""
import json
from fractions import Fraction
import math
import os

import numpy as np
import pytest

from oracle import ckks
from oracle.ckks import Oracle, OracleError
from tests import bigint_defs as D

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def small_oracle(log_n=4, q_bits=(30, 28, 28), p_bits=31, seed=7):
    o = Oracle(log_n, list(q_bits), p_bits, seed=seed, nthreads=2)
    return o


# ------------------------------------------------------------------------- primes and roots
CONFIG_PARAMS = {
    "config1": (13, [60, 40, 40], 60),
    "config2_13": (13, [50] * 3, 60),
    "config2_14": (14, [50] * 8, 60),
    "config2_15": (15, [50] * 16, 60),
    "config2_16": (16, [50] * 24, 60),
    "config3": (14, [60] + [40] * 6, 60),
    "config4": (15, [60] + [40] * 13, 60),
    "config5": (16, [60] + [40] * 23, 60),
}


def _expected_primes(log_n, q_bits, p_bits):
    """A3 written as a brute-force scan with an independent primality test."""
    two_n = 2 << (log_n - 1) << 0
    two_n = 1 << (log_n + 1)
    cursors = {}

    def take(b):
        k = cursors.get(b, ((1 << b) - 2) // two_n)
        while True:
            q = k * two_n + 1
            k -= 1
            if D.is_prime(q):
                cursors[b] = k
                return q

    p = take(p_bits)
    qs = [take(b) for b in q_bits]
    return qs + [p]


@pytest.mark.parametrize("name", sorted(CONFIG_PARAMS))
def test_primes_rule_and_golden(name):
    log_n, qb, pb = CONFIG_PARAMS[name]
    o = Oracle(log_n, qb, pb, nthreads=2)
    two_n = 1 << (log_n + 1)
    for m, b in zip(o.moduli, qb + [pb]):
        assert D.is_prime(m) and m % two_n == 1 and m < (1 << b) and m > (1 << (b - 1))
    assert len(set(o.moduli)) == len(o.moduli)
    assert o.moduli == _expected_primes(log_n, qb, pb)
    gold = json.load(open(os.path.join(GOLD, "moduli.json")))
    assert o.moduli == gold[name]["moduli"]


def _min_root_independent(q, N):
    # a different generator search (largest non-residue below 1000 instead of smallest)
    g = max(x for x in range(2, 1000) if pow(x, (q - 1) // 2, q) == q - 1)
    r0 = pow(g, (q - 1) // (2 * N), q)
    best, cur, sq = r0, r0, r0 * r0 % q
    for _ in range(N - 1):
        cur = cur * sq % q
        best = min(best, cur)
    return best


@pytest.mark.parametrize("log_n,qb,pb", [(4, [20, 20], 22), (10, [40, 30], 50), (13, [60, 40], 60)])
def test_roots(log_n, qb, pb):
    o = Oracle(log_n, qb, pb, nthreads=2)
    N = o.N
    for q, psi in zip(o.moduli, o.psi):
        assert pow(psi, N, q) == q - 1 and pow(psi, 2 * N, q) == 1
        assert psi == _min_root_independent(q, N)
    if log_n == 4:  # brute-force minimality on a tiny prime
        q, psi = o.moduli[0], o.psi[0]
        assert all(pow(x, N, q) != q - 1 for x in range(2, psi))


# ------------------------------------------------------------------------- NTT (a1, a2)
@pytest.mark.parametrize("log_n,qb,pb", [(4, [30, 28], 31), (6, [50, 40], 60), (8, [60], 60)])
def test_ntt_matches_definition(log_n, qb, pb):
    o = Oracle(log_n, qb, pb, nthreads=2)
    rng = np.random.default_rng(log_n)
    for midx, q in enumerate(o.moduli):
        a = [int(x) for x in rng.integers(0, q, size=o.N, dtype=np.uint64)]
        want = D.ntt_direct(a, q, o.psi[midx])
        got = o.ntt(np.array([a], dtype=np.uint64), midx0=midx)[0]
        assert [int(x) for x in got] == want
        back = o.intt(np.array([want], dtype=np.uint64), midx0=midx)[0]
        assert [int(x) for x in back] == a


@pytest.mark.parametrize("log_n", [6, 8])
def test_negacyclic_product(log_n):
    o = Oracle(log_n, [60, 50], 40, nthreads=2)
    rng = np.random.default_rng(3)
    for midx, q in enumerate(o.moduli):
        a = rng.integers(0, q, size=o.N, dtype=np.uint64)
        b = rng.integers(0, q, size=o.N, dtype=np.uint64)
        A = o.ntt(a[None], midx)[0]
        B = o.ntt(b[None], midx)[0]
        prod = np.array([int(x) * int(y) % q for x, y in zip(A, B)], dtype=np.uint64)
        got = o.intt(prod[None], midx)[0]
        assert [int(x) for x in got] == D.negacyclic_mul(a, b, q)


def test_ntt_roundtrip_large():
    o = Oracle(13, [60, 40, 40], 60, nthreads=4)
    rng = np.random.default_rng(0)
    a = np.stack([rng.integers(0, q, size=o.N, dtype=np.uint64) for q in o.moduli])
    assert (o.intt(o.ntt(a)) == a).all()


# ------------------------------------------------------------------------- ChaCha20 + samplers (A9-A11)
def _lib_keystream(key: bytes, counter: int, nonce: bytes, nbytes: int) -> bytes:
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    return Cipher(algorithms.ChaCha20(key, counter.to_bytes(4, "little") + nonce), mode=None).encryptor().update(
        b"\0" * nbytes)


def _orc_block(key: bytes, counter: int, nonce: bytes) -> bytes:
    out = np.zeros(16, dtype=np.uint32)
    ckks.lib().orc_chacha20_block(np.frombuffer(key, dtype="<u4").astype(np.uint32).copy(), counter,
                                  np.frombuffer(nonce, dtype="<u4").astype(np.uint32).copy(), out)
    return out.astype("<u4").tobytes()


def test_chacha20_rfc8439_vector():
    g = json.load(open(os.path.join(GOLD, "chacha20_rfc8439.json")))
    key, nonce = bytes.fromhex(g["key_hex"]), bytes.fromhex(g["nonce_hex"])
    assert _orc_block(key, g["counter"], nonce).hex() == g["serialized_block_hex"]
    assert _lib_keystream(key, g["counter"], nonce, 64).hex() == g["serialized_block_hex"]


def test_chacha20_vs_library_random():
    rng = np.random.default_rng(11)
    for _ in range(20):
        key = rng.bytes(32)
        nonce = rng.bytes(12)
        ctr = int(rng.integers(0, 2 ** 32 - 4))
        assert _orc_block(key, ctr, nonce) == _lib_keystream(key, ctr, nonce, 64)


def test_stream_layout_matches_library():
    """A11: key = seed LE in bytes 0..7, nonce = (tag, index lo, index hi), word64 n at u32 2n,2n+1."""
    seed, tag, index = 0x0123456789ABCDEF, 7, (5 << 32) | (3 << 16) | 2
    out = np.zeros(40, dtype=np.uint64)
    ckks.lib().orc_stream_u64(seed, tag, index, 0, 40, out)
    key = seed.to_bytes(8, "little") + b"\0" * 24
    nonce = tag.to_bytes(4, "little") + index.to_bytes(8, "little")
    ks = _lib_keystream(key, 0, nonce, 40 * 8)
    assert out.astype("<u8").tobytes() == ks


def test_sampler_moments():
    o = Oracle(14, [50], 60, nthreads=2)
    t = np.zeros(o.N, dtype=np.int64)
    ckks.lib().orc_sample_ternary(o.ctx, 1, 1, 0, t)
    assert set(np.unique(t)) <= {-1, 0, 1}
    for v in (-1, 0, 1):
        assert abs((t == v).mean() - 1 / 3) < 0.02
    e = np.zeros(o.N, dtype=np.int64)
    ckks.lib().orc_sample_cbd(o.ctx, 1, 3, 0, e)
    assert np.abs(e).max() <= 21 and abs(e.mean()) < 0.1 and abs(e.var() - 10.5) < 0.5
    u = np.zeros(o.N, dtype=np.uint64)
    q = o.q[0]
    ckks.lib().orc_sample_uniform(o.ctx, 1, 2, 0, q, u)
    assert int(u.max()) < q
    hist = np.bincount((u.astype(np.float64) / q * 16).astype(int), minlength=16)
    chi2 = ((hist - o.N / 16) ** 2 / (o.N / 16)).sum()
    assert chi2 < 50  # 15 dof, p ~ 1e-5
    # uniform residue = (w[2t+1] * 2^64 + w[2t]) mod q (A11 fixed-position extraction)
    w = np.zeros(2 * o.N, dtype=np.uint64)
    ckks.lib().orc_stream_u64(1, 2, 0, 0, 2 * o.N, w)
    for tt in (0, 1, 777, o.N - 1):
        assert int(u[tt]) == ((int(w[2 * tt + 1]) << 64) | int(w[2 * tt])) % q


# ------------------------------------------------------------------------- encode / decode (a13)
def test_encode_constant_closed_form_and_spec_examples():
    o = Oracle(10, [60, 40], 60, nthreads=2)
    g = json.load(open(os.path.join(GOLD, "encode_examples.json")))
    for case in g["cases"]:
        m = o.encode_coeffs(np.full(o.slots, case["value"]), case["scale"])
        assert m[0] == case["constant_coeff"] and (m[1:] == 0).all()
    for c in (0.123456789, -2.5, 1.0, -0.3):
        m = o.encode_coeffs(np.full(o.slots, c), 2.0 ** 40)
        # P-ENC-1 closed form, rounded exactly (A7): round-half-away(c Delta) of the exact real
        assert m[0] == D.round_half_away(Fraction(c) * 2 ** 40) and (m[1:] == 0).all()


def test_llround_ties_literal():
    """A20: scalars are X = llround(x scale), round half AWAY from zero of the double, exactly
    (the classic floor(x + 0.5) bugs at 0.49999999999999994 and 2^52 + 1 included)."""
    cases = {2.5: 3, -2.5: -3, 0.5: 1, -0.5: -1, 1.5: 2, -1.5: -2, 0.49999999999999994: 0,
             -0.49999999999999994: 0, 4503599627370497.0: 4503599627370497, 2.0 ** 61 + 0.0: 2 ** 61,
             1099511627775.5: 1099511627776, -1099511627775.5: -1099511627776, 7.0: 7}
    for x, want in cases.items():
        assert ckks.llround(x) == want, x


def test_encode_exact_ties_closed_form():
    """A7 exact ties: a constant slot vector c at scale 1 encodes to the constant polynomial with
    m_0 = c exactly (P-ENC-1: the t = 0 sum has only exact terms), so c = k + 1/2 is an exact
    tie -- rounded half away from zero, every other coefficient 0."""
    o = Oracle(10, [60, 40], 60, nthreads=2)
    for c, want in ((2.5, 3), (-3.5, -4), (0.5, 1), (-0.5, -1), (1234567.5, 1234568), (-7.5, -8)):
        m = o.encode_coeffs(np.full(o.slots, c), 1.0)
        assert m[0] == want and (m[1:] == 0).all(), (c, m[:4])


def test_encode_near_ties_match_exact_real_rounding():
    """A7 near ties: at N = 16, slot vectors tuned (through z_0) so that a chosen coefficient lies
    within 2^-14 .. 2^-34 of a half-integer, above and below it, for positive and negative
    values; EVERY coefficient must equal round-half-away of the exact real v_t (Decimal sums to
    ~85 digits, tests/bigint_defs.py) -- this exercises the oracle's binary128 recomputation
    window (2^-12) and its long-double path on the same vectors."""
    from decimal import Decimal, localcontext
    o = Oracle(4, [60], 60, nthreads=1)
    N, s = o.N, o.slots
    rng = np.random.default_rng(11)
    pi = D.dec_pi()
    in_window = set()
    for case, (t, K, delta) in enumerate([(1, 1000, 2.0 ** -14), (3, -2000, -2.0 ** -20), (5, 777777, 2.0 ** -30),
                                          (2, -31, 2.0 ** -34), (7, 123456, -2.0 ** -26), (6, -500000, 2.0 ** -16)]):
        z = rng.uniform(-1, 1, s)
        scale = 2.0 ** 20
        with localcontext() as ctx:
            ctx.prec = 90
            rest = D.encode_values_exact(np.r_[0.0, z[1:]], scale, N)[t]
            coef = Decimal(float(scale)) / N * 2 * D.dec_cos(pi * t / N)      # d v_t / d z_0
            target = Decimal(K) + (Decimal("0.5") if K >= 0 else Decimal("-0.5")) + Decimal(delta)
            z[0] = float((target - rest) / coef)
        v = D.encode_values_exact(z, scale, N)
        want = [D.round_half_away(x) for x in v]
        got = o.encode_coeffs(z, scale)
        assert [int(x) for x in got] == want, case
        frac = abs(v[t]) - int(abs(v[t]))
        if abs(frac - Decimal("0.5")) < Decimal(2) ** -12:
            in_window.add((v[t] > 0, frac > Decimal("0.5")))
    assert in_window == {(True, True), (True, False), (False, True), (False, False)}


def test_encode_matches_canonical_embedding():
    """Evaluate the encoded polynomial at zeta^(5^j) with numpy complex128: ~ Delta z_j."""
    o = Oracle(8, [60], 60, nthreads=2)
    rng = np.random.default_rng(5)
    z = rng.uniform(-1, 1, o.slots)
    delta = 2.0 ** 30
    m = o.encode_coeffs(z, delta).astype(np.float64)
    N = o.N
    t = np.arange(N)
    for j in range(o.slots):
        k = pow(5, j, 2 * N)
        val = np.sum(m * np.exp(1j * np.pi * k * t / N))
        assert abs(val.real / delta - z[j]) < 1e-6 and abs(val.imag / delta) < 1e-6


def test_decode_monomial_closed_form():
    """P-ENC-2: decode of Delta X^t is cos(pi 5^j t / N) (real part of zeta^(5^j t))."""
    o = Oracle(8, [60], 60, nthreads=2)
    delta = 2.0 ** 40
    for t in (0, 1, 5, 77, o.N - 1):
        m = np.zeros(o.N, dtype=np.int64)
        m[t] = int(delta)
        pt = o.pt_from_int_coeffs(m, delta, 0)
        z = o.decode(pt)
        want = np.array([math.cos(math.pi * ((pow(5, j, 2 * o.N) * t) % (2 * o.N)) / o.N) for j in range(o.slots)])
        assert np.abs(z - want).max() < 1e-12


def test_encode_decode_roundtrip_error_bound():
    """encoding error O(sqrt N)/Delta."""
    o = Oracle(12, [60, 40], 60, nthreads=4)
    z = np.random.default_rng(2).uniform(0, 1, o.slots)
    pt = o.encode(z, 2.0 ** 40)
    err = np.abs(o.decode(pt) - z).max()
    assert err < 4 * math.sqrt(o.N) / 2.0 ** 40
    with pytest.raises(OracleError) as ei:
        o.encode(np.zeros(o.slots + 1), 2.0 ** 40)
    assert ei.value.code == "CAPACITY"


# ------------------------------------------------------------------------- keys, encrypt, decrypt (a14)
def _coeffs(o, limb_ntt, midx):
    return [D.centered(int(x), o.moduli[midx]) for x in o.intt(limb_ntt[None], midx)[0]]


def _sample(o, kind, tag, index):
    x = np.zeros(o.N, dtype=np.int64)
    getattr(ckks.lib(), f"orc_sample_{kind}")(o.ctx, o.seed, tag, index, x)
    return [int(v) for v in x]


def test_public_key_exact():
    o = small_oracle(log_n=5)
    o.keygen()
    e = _sample(o, "cbd", ckks.TAG_PK_E, 0)
    s = [int(v) for v in o.s_int]
    assert _coeffs(o, o.s_ntt[0], 0) == s
    for i, q in enumerate(o.q):
        b = o.intt(o.pk[0, i][None], i)[0]
        a = o.intt(o.pk[1, i][None], i)[0]
        as_ = D.negacyclic_mul(a, s, q)
        assert [D.centered(int(x) + y, q) for x, y in zip(b, as_)] == e


def test_ksk_exact():
    o = small_oracle(log_n=4)
    o.keygen(rot_amounts=[3])
    s = [int(v) for v in o.s_int]
    P = o.p
    targets = {0: D.negacyclic_mul(s, s), 3: None}
    g = o.galois(3)
    sg = [0] * o.N
    for t, v in enumerate(s):
        idx = g * t % (2 * o.N)
        if idx < o.N:
            sg[idx] += v
        else:
            sg[idx - o.N] -= v
    targets[3] = sg
    for keyid, key in ((0, o.rlk), (3, o.rot_keys[3])):
        for j in range(o.L):
            e = _sample(o, "cbd", ckks.TAG_KSK_E, (keyid << 32) | j)
            for r, q in enumerate(o.moduli):
                b = o.intt(key[j, 0, r][None], r)[0]
                a = o.intt(key[j, 1, r][None], r)[0]
                as_ = D.negacyclic_mul(a, s, q)
                lhs = [(int(x) + y) % q for x, y in zip(b, as_)]
                gad = [(P * v) % q if r == j else 0 for v in targets[keyid]]
                assert [D.centered(x - y, q) for x, y in zip(lhs, gad)] == e


def test_encrypt_decrypt_exact_error():
    """c0 + c1 s - m = v e_pk + e0 + e1 s exactly (integer polynomials, A12)."""
    o = small_oracle(log_n=5)
    o.keygen()
    z = np.linspace(0, 1, o.slots)
    pt = o.encode(z, 2.0 ** 20)
    ct = o.encrypt(pt)
    v = _sample(o, "ternary", ckks.TAG_ENC_V, 0)
    e0 = _sample(o, "cbd", ckks.TAG_ENC_E0, 0)
    e1 = _sample(o, "cbd", ckks.TAG_ENC_E1, 0)
    epk = _sample(o, "cbd", ckks.TAG_PK_E, 0)
    s = [int(x) for x in o.s_int]
    want = [a + b + c for a, b, c in zip(D.negacyclic_mul(v, epk), e0, D.negacyclic_mul(e1, s))]
    dec = o.decrypt(ct)
    m = [int(x) for x in o.encode_coeffs(z, 2.0 ** 20)]
    for i, q in enumerate(o.q):
        got = _coeffs(o, dec.data[i], i)
        assert [D.centered(x - y, q) for x, y in zip(got, m)] == want
    assert o.enc_counter == 1


def test_encrypt_decrypt_semantics():
    o = Oracle(11, [60, 40, 40], 60, seed=3, nthreads=4)
    o.keygen()
    z = np.random.default_rng(0).uniform(0, 1, o.slots)
    out = o.decode(o.decrypt(o.encrypt(o.encode(z, 2.0 ** 40))))
    assert np.abs(out - z).max() < 2.0 ** -20


# ------------------------------------------------------------------------- key switching (a5) by big integers
def _crt_poly(o, limbs_ntt, midxs):
    """NTT-form limbs -> integer coefficients in [0, prod) by INTT per limb + CRT."""
    coeffs = [o.intt(l[None], m)[0] for l, m in zip(limbs_ntt, midxs)]
    mods = [o.moduli[m] for m in midxs]
    return [D.crt([int(c[t]) for c in coeffs], mods) for t in range(o.N)], mods


@pytest.mark.parametrize("level", [2, 1, 0])
def test_keyswitch_bigint_definition(level):
    """out = (A - [A]_{p,c}) / p mod Q_l with A = sum_j x_j (b_j, a_j) mod p Q_l (A14)."""
    o = small_oracle(log_n=4, q_bits=(30, 28, 28), p_bits=31)
    o.keygen(rot_amounts=[1])
    key = o.rot_keys[1]
    l1 = level + 1
    rng = np.random.default_rng(level)
    d = np.stack([rng.integers(0, o.q[i], size=o.N, dtype=np.uint64) for i in range(l1)])
    out = o.keyswitch(d, level, key)
    midxs = list(range(l1)) + [o.L]
    PQ = 1
    for m in midxs:
        PQ *= o.moduli[m]
    A = [[0] * o.N, [0] * o.N]
    for j in range(l1):
        xj = _coeffs(o, d[j], j)                      # centered lift of digit j
        for k in range(2):
            kj, _ = _crt_poly(o, [key[j, k, m] for m in midxs], midxs)
            prod = D.negacyclic_mul(xj, kj, PQ)
            A[k] = [(u + v) % PQ for u, v in zip(A[k], prod)]
    p = o.p
    for k in range(2):
        want = [(a - D.centered(a, p)) // p for a in A[k]]
        for i in range(l1):
            got = [int(x) for x in o.intt(out[k, i][None], i)[0]]
            assert got == [w % o.q[i] for w in want]


def test_rescale_bigint_definition():
    """A18: rescale = round(u / q_l) mod Q_{l-1} for the representative u in [0, Q_l)."""
    o = small_oracle(log_n=4, q_bits=(30, 28, 28, 26), p_bits=31)
    rng = np.random.default_rng(1)
    level = 3
    data = np.stack([np.stack([rng.integers(0, o.q[i], size=o.N, dtype=np.uint64) for i in range(level + 1)])
                     for _ in range(2)])
    ct = ckks.Ct(data, level, 2.0 ** 40)
    out = o.rescale(ct)
    assert out.level == level - 1 and out.scale == 2.0 ** 40 / o.q[level]
    ql = o.q[level]
    for k in range(2):
        u, _ = _crt_poly(o, list(data[k]), list(range(level + 1)))
        want = [D.round_div(x, ql) for x in u]
        for i in range(level):
            got = [int(x) for x in o.intt(out.data[k, i][None], i)[0]]
            assert got == [w % o.q[i] for w in want]


def test_tensor_is_negacyclic_product():
    o = small_oracle(log_n=4)
    rng = np.random.default_rng(9)
    lv = 2
    a = np.stack([np.stack([rng.integers(0, q, size=o.N, dtype=np.uint64) for q in o.q]) for _ in range(2)])
    b = np.stack([np.stack([rng.integers(0, q, size=o.N, dtype=np.uint64) for q in o.q]) for _ in range(2)])
    out = o.mul_norelin(ckks.Ct(a, lv, 1.0), ckks.Ct(b, lv, 1.0))
    for i, q in enumerate(o.q):
        ca = [o.intt(a[k, i][None], i)[0] for k in range(2)]
        cb = [o.intt(b[k, i][None], i)[0] for k in range(2)]
        want = [D.negacyclic_mul(ca[0], cb[0], q),
                [(x + y) % q for x, y in zip(D.negacyclic_mul(ca[0], cb[1], q), D.negacyclic_mul(ca[1], cb[0], q))],
                D.negacyclic_mul(ca[1], cb[1], q)]
        for k in range(3):
            assert [int(x) for x in o.intt(out.data[k, i][None], i)[0]] == want[k]


# ------------------------------------------------------------------------- automorphism / rotation (a7)
@pytest.mark.parametrize("log_n", [4, 8])
def test_automorphism_ntt_permutation_closed_form(log_n):
    """NTT-domain psi_g = index permutation perm[j] = brv(((2 brv(j)+1) g mod 2N - 1)/2) (K6)."""
    o = Oracle(log_n, [40], 40, nthreads=2)
    N, bits = o.N, log_n
    rng = np.random.default_rng(0)
    a = rng.integers(0, o.q[0], size=N, dtype=np.uint64)
    for k in (1, 3, N // 2 - 1):
        g = o.galois(k)
        out = np.zeros(N, dtype=np.uint64)
        ckks.lib().orc_automorphism_ntt_limb(o.ctx, 0, g, a, out)
        perm = [D.brv((((2 * D.brv(j, bits) + 1) * g) % (2 * N) - 1) // 2, bits) for j in range(N)]
        assert [int(x) for x in out] == [int(a[perm[j]]) for j in range(N)]


def test_rotation_semantics():
    o = Oracle(10, [60, 40, 40], 60, seed=1, nthreads=4)
    ks = [1, 2, 5, 100, o.slots - 1]
    o.keygen(rot_amounts=ks)
    z = np.random.default_rng(4).uniform(0, 1, o.slots)
    ct = o.encrypt(o.encode(z, 2.0 ** 40))
    for k in ks:
        r = o.decode(o.decrypt(o.rot_left(ct, k)))
        assert np.abs(r - np.roll(z, -k)).max() < 1e-6
    # rotRight(c, k) == rotLeft(c, s - k) bit-exactly
    assert (o.rot_right(ct, 1).data == o.rot_left(ct, o.slots - 1).data).all()
    assert (o.rot_left(ct, 0).data == ct.data).all()
    with pytest.raises(OracleError) as ei:
        o.rot_left(ct, 3)
    assert ei.value.code == "NO_KEY"


def test_mul_relin_rescale_semantics():
    o = Oracle(10, [60, 40, 40], 60, seed=2, nthreads=4)
    o.keygen()
    rng = np.random.default_rng(6)
    x, y = rng.uniform(0, 1, o.slots), rng.uniform(-1, 1, o.slots)
    cx, cy = o.encrypt(o.encode(x, 2.0 ** 40)), o.encrypt(o.encode(y, 2.0 ** 40))
    c3 = o.mul_norelin(cx, cy)
    # scale 2^80 > q_0/2: limb-0 decode (A13) needs the rescale first
    c3r = o.rescale(c3)
    assert c3r.npolys == 3 and np.abs(o.decode(o.decrypt(c3r)) - x * y).max() < 1e-6
    r = o.rescale(o.relinearize(c3))
    assert r.npolys == 2 and r.level == 1
    assert np.abs(o.decode(o.decrypt(r)) - x * y).max() < 1e-6
    # plaintext / scalar ops
    w = rng.uniform(-1, 1, o.slots)
    pw = o.encode(w, float(o.q[2]))
    r2 = o.rescale(o.mul_plain(cx, pw))
    assert np.abs(o.decode(o.decrypt(r2)) - x * w).max() < 1e-6
    r3 = o.rescale(o.mul_scalar(cx, -0.75))
    assert abs(r3.scale - 2.0 ** 40) / 2.0 ** 40 < 1e-4
    assert np.abs(o.decode(o.decrypt(r3)) - (-0.75 * x)).max() < 1e-6
    r4 = o.add_scalar(cx, 0.5)
    assert np.abs(o.decode(o.decrypt(r4)) - (x + 0.5)).max() < 1e-6
    r5 = o.sub(o.add(cx, cy), cy)
    assert np.abs(o.decode(o.decrypt(r5)) - x).max() < 1e-6


def test_depth_example_consumes_two_levels():
    """beta * (gamma*gamma + a + lambda) has multiplicative depth 2."""
    o = Oracle(10, [60, 40, 40, 40], 60, seed=5, nthreads=4)
    o.keygen()
    rng = np.random.default_rng(8)
    b, g, lam, a = (rng.uniform(0, 1, o.slots) for _ in range(4))
    top = o.L - 1
    cb, cg, cl = (o.encrypt(o.encode(v, 2.0 ** 40)) for v in (b, g, lam))
    gg = o.rescale(o.mul(cg, cg))
    s = o.add_plain(gg, o.encode(a, gg.scale, gg.level))
    s = o.add(s, o.mod_switch(ckks.Ct(cl.data, cl.level, gg.scale), 1))
    res = o.rescale(o.mul(o.mod_switch(ckks.Ct(cb.data, cb.level, s.scale), 1), s))
    assert res.level == top - 2
    want = b * (g * g + a + lam)
    # lambda / beta were re-labelled with the drifted scale; tolerance covers |1 - q/2^40|
    assert np.abs(o.decode(o.decrypt(res)) - want).max() < 1e-3


def test_error_contract_and_division_profile():
    o = Oracle(10, [60, 40, 40], 60, seed=2, nthreads=4)
    o.keygen()
    c = o.encrypt(o.encode([0.5], 2.0 ** 40))
    with pytest.raises(OracleError) as ei:
        o.add(c, o.mod_switch(c))
    assert ei.value.code == "LEVEL_MISMATCH"
    with pytest.raises(OracleError) as ei:
        o.add(c, ckks.Ct(c.data, c.level, 2.0 ** 41))
    assert ei.value.code == "SCALE_MISMATCH"
    with pytest.raises(OracleError) as ei:
        o.bootstrap(c)
    assert ei.value.code == "UNSUPPORTED_PROFILE"
    assert o.max_scalar_div(c, 2 ** 41) == o.q[2]
    assert o.max_scalar_div(c, 2 ** 39) == 1
    with pytest.raises(OracleError) as ei:
        o.div_scalar(c, 3)
    assert ei.value.code == "INVALID_DIVISOR"
    # with L limbs, L-1 rescales succeed and the next is MODULUS_EXHAUSTED (S:177 analogue)
    x = c
    for _ in range(o.L - 1):
        x = o.div_scalar(x, o.max_scalar_div(x, 2 ** 62))
    with pytest.raises(OracleError) as ei:
        o.div_scalar(x, o.q[0])
    assert ei.value.code == "MODULUS_EXHAUSTED"
    with pytest.raises(OracleError) as ei:
        o.mul_norelin(o.mul_norelin(c, c), c)
    assert ei.value.code == "NOT_RELINEARIZED"


def test_determinism():
    outs = []
    for _ in range(2):
        o = Oracle(9, [60, 40], 60, seed=42, nthreads=3)
        o.keygen(rot_amounts=[2])
        c = o.encrypt(o.encode(np.linspace(0, 1, o.slots), 2.0 ** 40))
        outs.append(o.rot_left(c, 2).data.copy())
    assert (outs[0] == outs[1]).all()
