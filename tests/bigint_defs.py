"""Plain big-integer definitions used to PIN the oracle (tests only).

Nothing here calls the oracle's arithmetic; each function is the textbook/mathematical
definition written with Python integers, usable only at tiny N.
"""
from __future__ import annotations


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin for n < 3.3e24 (first 13 prime bases)."""
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for p in small:
        if n % p == 0:
            return n == p
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def brv(j: int, bits: int) -> int:
    return int(format(j, f"0{bits}b")[::-1], 2) if bits else 0


def ntt_direct(a, q: int, psi: int):
    """Definition (A5): ahat[j] = sum_t a_t psi^((2 brv(j) + 1) t) mod q."""
    N = len(a)
    bits = N.bit_length() - 1
    out = []
    for j in range(N):
        e = 2 * brv(j, bits) + 1
        w = pow(psi, e, q)
        acc, wt = 0, 1
        for t in range(N):
            acc += int(a[t]) * wt
            wt = wt * w % q
        out.append(acc % q)
    return out


def negacyclic_mul(a, b, mod: int | None = None):
    """Schoolbook product in Z[X]/(X^N + 1) (optionally mod `mod`)."""
    N = len(a)
    out = [0] * N
    for i in range(N):
        ai = int(a[i])
        if ai == 0:
            continue
        for j in range(N):
            k = i + j
            if k < N:
                out[k] += ai * int(b[j])
            else:
                out[k - N] -= ai * int(b[j])
    if mod is not None:
        out = [x % mod for x in out]
    return out


def crt(residues, moduli) -> int:
    """Chinese remaindering to [0, prod moduli)."""
    M = 1
    for m in moduli:
        M *= m
    x = 0
    for r, m in zip(residues, moduli):
        Mi = M // m
        x += int(r) * Mi * pow(Mi, -1, m)
    return x % M


def centered(x: int, m: int) -> int:
    x %= m
    return x - m if x > m // 2 else x


def round_div(a: int, d: int) -> int:
    """round(a / d) for odd d (no ties), exact integers."""
    return (2 * a + d) // (2 * d)


# ---------------------------------------------------------------- exact encoding (A7) at tiny N
from decimal import Decimal, localcontext  # noqa: E402
from fractions import Fraction  # noqa: E402

_DEC_PREC = 90


def _atan_inv(n: int) -> Decimal:
    """atan(1/n) by its Taylor series (|1/n| <= 1/5), at the current Decimal precision."""
    x = Decimal(1) / n
    x2 = x * x
    term, acc, k = x, x, 1
    eps = Decimal(10) ** (-_DEC_PREC - 5)
    while abs(term) > eps:
        term = -term * x2
        acc += term / (2 * k + 1)
        k += 1
    return acc


def dec_pi() -> Decimal:
    """Machin: pi = 16 atan(1/5) - 4 atan(1/239)."""
    with localcontext() as ctx:
        ctx.prec = _DEC_PREC + 10
        return +(16 * _atan_inv(5) - 4 * _atan_inv(239))


def dec_cos(x: Decimal) -> Decimal:
    """cos(x) by its Taylor series, |x| <= 2 pi, ~90 significant digits."""
    with localcontext() as ctx:
        ctx.prec = _DEC_PREC + 20
        x2 = x * x
        term, acc, k = Decimal(1), Decimal(1), 0
        eps = Decimal(10) ** (-_DEC_PREC - 10)
        while abs(term) > eps or k < 4:
            term = -term * x2 / ((2 * k + 1) * (2 * k + 2))
            acc += term
            k += 1
        return +acc


def encode_values_exact(z, scale: float, N: int):
    """A7's real values v_t = (Delta/N) sum_{j<n} 2 z_j cos(pi (5^j t mod 2N) / N), t < N, to ~85
    significant digits (every double z_j and the scale enter exactly)."""
    pi = dec_pi()
    cos_tab = {}
    out = []
    with localcontext() as ctx:
        ctx.prec = _DEC_PREC
        for t in range(N):
            acc = Decimal(0)
            for j, zj in enumerate(z):
                if zj == 0.0:
                    continue
                e = (pow(5, j, 2 * N) * t) % (2 * N)
                if e not in cos_tab:
                    cos_tab[e] = dec_cos(pi * e / N)
                acc += 2 * Decimal(float(zj)) * cos_tab[e]
            out.append(acc * Decimal(float(scale)) / N)
    return out


def round_half_away(v) -> int:
    """round half away from zero of an exact Decimal / Fraction / int."""
    f = Fraction(v)
    h = abs(f) + Fraction(1, 2)
    r = h.numerator // h.denominator          # floor(|v| + 1/2)
    return r if f >= 0 else -r
