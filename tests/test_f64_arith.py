"""The exact-FP64 modular primitives of csrc/ntt_f64.cuh, emulated on the host with IEEE binary64
(Python floats) and an exact FMA (integer arithmetic, one rounding): exactness (t == a w mod q)
and the magnitude bounds the butterfly engines rely on, for q up to 2^50 and adversarial operands.
"""
import random
from fractions import Fraction

import pytest


def fma(a: float, b: float, c: float) -> float:
    """fl(a*b + c) with a single rounding (round-half-even): exact rational, then float()."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def redd(v: float, q: float, qinv: float) -> float:
    return fma(-float(round(v * qinv)), q, v)


def mulred(a: float, w: float, q: float, qinv: float) -> float:
    h = a * w
    l = fma(a, w, -h)
    qt = float(round(h * qinv))
    return fma(-qt, q, h) + l


def _primes_near_2_50():
    # q = 1 mod 2^17 (N = 2^16), the largest below 2^50 (config 2's 50-bit limbs), and 2^40-ish
    out = []
    for bits in (50, 40):
        k = ((1 << bits) - 2) // (1 << 17)
        while len([q for q in out if q.bit_length() == bits]) < 2:
            q = k * (1 << 17) + 1
            if all(q % p for p in range(3, 2000, 2)) and pow(3, q - 1, q) == 1:
                out.append(q)
            k -= 1
    return out


@pytest.mark.parametrize("q", _primes_near_2_50())
def test_mulred_exact_and_bounded(q):
    rng = random.Random(q)
    qf, qinv = float(q), 1.0 / float(q)
    for B in (0.5, 1.0, 2.0):                      # the engines' input bounds (|a| <= B q)
        amax = int(B * q)
        cases = [(amax, q - 1), (-amax, q - 1), (amax, 1), (0, q - 1), (amax - 1, (q - 1) // 2)]
        cases += [(rng.randint(-amax, amax), rng.randrange(q)) for _ in range(4000)]
        worst = 0.0
        for a, w in cases:
            t = mulred(float(a), float(w), qf, qinv)
            assert t == int(t) and abs(t) < 2 ** 53
            assert (int(t) - a * w) % q == 0, (a, w)
            worst = max(worst, abs(t) / q)
        assert worst <= 0.5 + 0.5 * B + 1e-9, (B, worst)   # ntt_f64.cuh: |t| <= (0.5 + 0.5 B) q


@pytest.mark.parametrize("q", _primes_near_2_50())
def test_butterfly_fixed_points(q):
    """Forward CT (X, Y) -> (red X + t, red X - t) stays <= 2q over many stages; inverse GS
    (X, Y) -> (red(X + Y), mulred(red(X - Y), W)) stays <= 0.75 q."""
    rng = random.Random(q + 1)
    qf, qinv = float(q), 1.0 / float(q)
    for _ in range(300):
        x, y = float(rng.randrange(q)), float(rng.randrange(q))
        for _stage in range(16):
            w = float(rng.randrange(q))
            xr = redd(x, qf, qinv)
            t = mulred(y, w, qf, qinv)
            x, y = xr + t, xr - t
            assert abs(x) <= 2 * q and abs(y) <= 2 * q
        a, b = float(rng.randrange(q)), float(rng.randrange(q))
        for _stage in range(16):
            w = float(rng.randrange(q))
            s = redd(a + b, qf, qinv)
            d = mulred(redd(a - b, qf, qinv), w, qf, qinv)
            assert (int(d) - ((int(a) - int(b)) % q) * int(w)) % q == 0
            a, b = s, d
            assert abs(a) <= 0.5 * q * (1 + 2 ** -40) and abs(b) <= 0.75 * q


def test_bit_conversions():
    """u2d / d2u bit tricks: x < 2^52 <-> double exactly (used at every load / store)."""
    import struct
    for x in (0, 1, (1 << 50) - 1, (1 << 52) - 1, 123456789012345):
        bits = x | 0x4330000000000000
        d = struct.unpack("<d", struct.pack("<Q", bits))[0] - 4503599627370496.0
        assert d == float(x) and int(d) == x
        back = struct.unpack("<Q", struct.pack("<d", d + 4503599627370496.0))[0] & ((1 << 52) - 1)
        assert back == x


def _full_stage(u: int, log_m: int, last_full: bool = True) -> bool:
    """ntt_f64.cuh full_stage: X is re-centred at stages u % 3 == 0 and at the pass's last stage
    (full_stage_cols, last_full=False: column passes, whose outputs feed a row pass, skip the
    latter)."""
    return u % 3 == 0 or (last_full and u == log_m - 1)


def _bound_recurrence(log_m: int, b_in: float, last_full: bool = True):
    """The header's worst-case magnitude bounds (units of q) per stage, centred twiddles:
    full stage B' = 1 + 3/16 B (+ eps), lazy stage B' = 19/16 B + 1/2."""
    out, b = [], b_in
    for u in range(log_m):
        b = (1.0 + 0.1875 * b) if _full_stage(u, log_m, last_full) else (1.1875 * b + 0.5)
        out.append(b * (1 + 2 ** -40))
    return out


@pytest.mark.parametrize("q", _primes_near_2_50())
@pytest.mark.parametrize("log_m", [2, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("row_last_full", [True, False])
def test_lazy_forward_schedule_exact_and_bounded(q, log_m, row_last_full):
    """The forward engines' lazy schedule (centred twiddles |W| <= q/2, X left unreduced except at
    full stages) over two chained passes: every value is an exact integer < 2^53 congruent to the
    textbook butterfly's, magnitudes stay within the header's recurrence, and each pass's output is
    <= 2q (the key inner product's d_rep4 precondition).  Operands: random, plus a greedy adversary
    that picks the twiddle maximising |t| among extreme candidates at every butterfly."""
    rng = random.Random(q * 7 + log_m)
    qf, qinv = float(q), 1.0 / float(q)
    M = 1 << log_m
    half = (q - 1) // 2
    cands = [half, -half, half - 1, -(half - 1), 1, -1]
    for trial in range(6):
        adversary = trial % 2 == 1
        x = [float(rng.randrange(q)) for _ in range(M)]          # canonical input, B <= 1
        xi = [int(v) % q for v in x]
        b_in = 1.0
        for _pass in range(2):
            # pass 0 = a column pass (full_stage_cols); pass 1 = a row pass: full last stage
            # (K4, whose d_rep4 needs <= 2q) or lazy (the register-direct rows, canonicalised)
            last_full = _pass == 1 and row_last_full
            bounds = _bound_recurrence(log_m, b_in, last_full)
            for u in range(log_m):
                dist = M >> (u + 1)
                full = _full_stage(u, log_m, last_full)
                for blk in range(0, M, 2 * dist):
                    w = rng.choice(cands) if not adversary else None
                    for e in range(blk, blk + dist):
                        X = redd(x[e], qf, qinv) if full else x[e]
                        if adversary:   # the twiddle maximising |t| for this operand
                            ts = [(abs(mulred(x[e + dist], float(c), qf, qinv)), c) for c in cands[:2]]
                            w = max(ts)[1]
                        t = mulred(x[e + dist], float(w), qf, qinv)
                        assert t == int(t) and abs(t) < 2 ** 53
                        ti = (xi[e + dist] * w) % q
                        assert (int(t) - ti) % q == 0
                        x[e], x[e + dist] = X + t, X - t
                        xi[e], xi[e + dist] = (xi[e] + ti) % q, (xi[e] - ti) % q
                top = max(abs(v) for v in x)
                assert top < 2 ** 52.6 and top <= bounds[u] * q, (u, top / q, bounds[u])
            assert all((int(v) - vi) % q == 0 for v, vi in zip(x, xi))
            assert max(abs(v) for v in x) <= (2 * q if last_full else 2.5 * q)
            b_in = max(abs(v) for v in x) / q


def test_lazy_schedule_accepts_wide_lift():
    """ModUp lifts a 50-bit source residue (|v| < 2^49, centred) into a 40-bit target without a
    separate reduction: the first (full) stage re-centres X and mulred's bound is absolute,
    |t| <= q/2 + 0.75 2^-52 |a| q."""
    q = [p for p in _primes_near_2_50() if p.bit_length() == 40][0]
    qf, qinv = float(q), 1.0 / float(q)
    rng = random.Random(5)
    for _ in range(2000):
        a = float(rng.randint(-(1 << 49), 1 << 49))
        w = rng.randint(-((q - 1) // 2), (q - 1) // 2)
        t = mulred(a, float(w), qf, qinv)
        assert t == int(t) and (int(t) - int(a) * w) % q == 0
        assert abs(t) <= q / 2 + 0.75 * 2 ** -52 * abs(a) * q + 1
        assert abs(redd(a, qf, qinv)) <= 0.5 * q + 1


@pytest.mark.parametrize("q", _primes_near_2_50())
def test_k4_row_schedule(q):
    """K4 v6 (ks_kernels.cu k4_full): the 8-stage row pass re-centres X at stages 0, 4, 7 only.  From
    a column-pass output (|v| <= 2.41 q, also driven by the greedy twiddle adversary) every value is
    an exact integer congruent to the textbook butterfly's, magnitudes stay <= 4.3 q (< 2^52.1), the
    output is <= 1.7 q, and the MAC that consumes it (a key word |K| <= q/2, the internal key
    format) stays <= 0.82 q, so eight of them sum below 7.1 q < 2^53."""
    rng = random.Random(q * 11)
    qf, qinv = float(q), 1.0 / float(q)
    M = 256
    half = (q - 1) // 2
    cands = [half, -half, half - 1, -(half - 1), 1, -1]
    full = {0, 4, 7}
    for trial in range(4):
        adversary = trial % 2 == 1
        # a column-pass output: the lazy column schedule from canonical inputs (<= 2.41 q)
        x = [float(rng.randrange(-int(2.41 * q), int(2.41 * q))) for _ in range(M)]
        xi = [int(v) % q for v in x]
        top_all = 0.0
        for u in range(8):
            dist = M >> (u + 1)
            for blk in range(0, M, 2 * dist):
                w = rng.choice(cands) if not adversary else None
                for e in range(blk, blk + dist):
                    X = redd(x[e], qf, qinv) if u in full else x[e]
                    if adversary:
                        w = max((abs(mulred(x[e + dist], float(c), qf, qinv)), c) for c in cands[:2])[1]
                    t = mulred(x[e + dist], float(w), qf, qinv)
                    assert t == int(t) and abs(t) < 2 ** 53
                    ti = (xi[e + dist] * w) % q
                    assert (int(t) - ti) % q == 0
                    x[e], x[e + dist] = X + t, X - t
                    xi[e], xi[e + dist] = (xi[e] + ti) % q, (xi[e] - ti) % q
            top = max(abs(v) for v in x)
            top_all = max(top_all, top)
            assert top < 2 ** 52.1 and top <= 4.3 * q, (u, top / q)
        assert all((int(v) - vi) % q == 0 for v, vi in zip(x, xi))
        assert max(abs(v) for v in x) <= 1.7 * q
        for d in x[:64]:
            for k in (half, -half, 0, 1):
                m = mulred(d, float(k), qf, qinv)
                assert (int(m) - int(d) * k) % q == 0 and abs(m) <= 0.82 * q
