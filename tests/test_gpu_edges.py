"""Edge cases of the C-ABI path (GPU): empty batches, level-0 ciphertexts (a key switch with a
single digit), the smallest ring (N = 2^8), a large key-switch (N = 2^16, L = 40 limbs: 40 digits,
3.4 GB key) sampled against the oracle, ragged slot counts, in-place forms and handle reuse."""
import numpy as np
import pytest

from oracle.ckks import Oracle

pytestmark = pytest.mark.gpu

H = pytest.importorskip("paper_1810_00845_b200.hisa")


def _pair(log_n, qb, pb, rots, seed=21, arena=4 << 30):
    g = H.Context(log_n, qb, pb, seed=seed, arena_bytes=arena)
    o = Oracle(log_n, qb, pb, seed=seed)
    g.keygen(rots, True)
    o.keygen(rot_amounts=rots)
    return g, o


def test_empty_batches_are_noops():
    g, o = _pair(10, [60, 40], 60, [1])
    assert g.rot_left_batch([], 1) == []
    assert g.rot_left_hoisted_batch([], [1, 2]) == []
    assert g.rescale_batch([]) == []
    assert g.mul_batch([], []) == []
    assert g.rot_add_batch([], 1) == []
    a = g.ct_random(1, 1)
    assert g.rot_left_hoisted(a, []) == []
    assert g.encode_batch(np.zeros((0, 4)), 2.0 ** 40) == []
    with pytest.raises(H.HisaError) as ei:           # more values than slots
        g.encode_batch(np.zeros((2, g.slots + 1)), 2.0 ** 40)
    assert ei.value.code == "CAPACITY"
    g.close()


def test_level_zero_keyswitch_and_smallest_ring():
    """N = 2^8 (the smallest supported ring) and level 0: one digit, the key switch is
    ModUp to {q_0, p}, inner product, ModDown."""
    g, o = _pair(8, [60, 40, 40], 60, [1, 5])
    a = g.ct_random(3, 0)
    oa = o.bench_ct(3, 0)
    for k in (1, 5):
        assert (g.ct_export(g.rot_left(a, k)) == o.rot_left(oa, k).data).all()
    t = g.mul_norelin(a, a)
    g.relinearize(t)
    assert (g.ct_export(t) == o.relinearize(o.mul_norelin(oa, oa)).data).all()
    with pytest.raises(H.HisaError) as ei:
        g.rescale(a)
    assert ei.value.code == "MODULUS_EXHAUSTED"
    hz = g.rot_left_hoisted(a, [1, 5, 0])
    assert (g.ct_export(hz[1]) == o.rot_left(oa, 5).data).all()
    assert (g.ct_export(hz[2]) == oa.data).all()
    g.close()


def test_ragged_and_full_slot_counts():
    g, o = _pair(11, [60, 40], 60, [])
    for n in (1, 3, 1023, 1024):
        z = np.random.default_rng(n).uniform(-1, 1, n)
        hp = g.encode(z, 2.0 ** 30)
        assert (g.pt_export(hp) == o.encode(z, 2.0 ** 30).data).all()
        assert np.abs(g.decode(hp, n) - z).max() < 1e-6
    g.close()


def test_inplace_forms_and_handle_reuse():
    g, o = _pair(10, [60, 40, 40], 60, [2])
    a, b = g.ct_random(4, 2), g.ct_random(5, 2)
    oa, ob = o.bench_ct(4, 2), o.bench_ct(5, 2)
    h = g.copy(a)
    assert g.add(h, b, inplace=True) == h
    assert (g.ct_export(h) == o.add(oa, ob).data).all()
    g.rot_left(h, 2, inplace=True)
    assert (g.ct_export(h) == o.rot_left(o.add(oa, ob), 2).data).all()
    g.free(h)
    for _ in range(50):            # slot reuse: generations make stale handles detectable
        x = g.copy(a)
        g.free(x)
        with pytest.raises(H.HisaError) as ei:
            g.ct_info(x)
        assert ei.value.code == "INVALID_HANDLE"
    g.close()


@pytest.mark.slow
def test_large_keyswitch_sampled():
    """N = 2^16 with 40 x 50-bit limbs (dnum = 40): a 40-digit key switch, 3.4 GB key, bit-exact
    with the oracle on one ciphertext; hoisted and batched paths agree with it."""
    L = 40
    g, o = _pair(16, [50] * L, 60, [7, 11], seed=2, arena=40 << 30)
    a = g.ct_random(9, L - 1)
    oa = o.bench_ct(9, L - 1)
    want = o.rot_left(oa, 7).data
    assert (g.ct_export(g.rot_left(a, 7)) == want).all()
    hz = g.rot_left_hoisted(a, [7, 11])
    assert (g.ct_export(hz[0]) == want).all()
    assert (g.ct_export(g.rot_left_batch([a, a], 7)[1]) == want).all()
    g.close()


def test_gpu_encode_exact_ties():
    """NEXT-4 GPU encode: exact half-integer coefficients (a constant vector z = k + 1/2 at scale 1
    encodes to the constant polynomial, P-ENC-1) fall in the near-tie window, are recomputed
    exactly in binary128 and rounded half away from zero (A7) -- equal to the oracle."""
    g, o = _pair(12, [60, 40], 60, [])
    for c in (2.5, -3.5, 0.5, 1234567.5):
        z = np.full(g.slots, c)
        h = g.encode(z, 1.0)
        want = o.encode(z, 1.0)
        assert (g.pt_export(h) == want.data).all(), c
        coeffs = o.intt(want.data[0:1].copy(), 0)[0]
        q0 = o.q[0]
        m0 = int(coeffs[0]) if coeffs[0] <= q0 // 2 else int(coeffs[0]) - q0
        assert m0 == (int(abs(c) + 0.5) * (1 if c > 0 else -1))
    hs = g.encode_batch(np.stack([np.full(g.slots, 2.5), np.linspace(-1, 1, g.slots)]), 2.0 ** 40)
    assert (g.pt_export(hs[0]) == o.encode(np.full(g.slots, 2.5), 2.0 ** 40).data).all()
    assert (g.pt_export(hs[1]) == o.encode(np.linspace(-1, 1, g.slots), 2.0 ** 40).data).all()
    g.close()


def test_gpu_encode_near_ties_match_exact_real_rounding():
    """A7 near ties on the GPU encoder (double-double FFT + host binary128 recomputation inside
    its tie window): sparse slot vectors at N = 2^8 tuned through z_0 so that chosen
    coefficients lie 2^-14 .. 2^-34 above / below half-integers of both signs; every coefficient
    equals round-half-away of the exact real v_t (Decimal, tests/bigint_defs.py) and the oracle's."""
    from decimal import Decimal, localcontext
    from tests import bigint_defs as D
    g, o = _pair(8, [60], 60, [])
    N, s = g.N, g.slots
    rng = np.random.default_rng(17)
    pi = D.dec_pi()
    q0 = o.q[0]
    for case, (t, K, delta) in enumerate([(1, 1000, 2.0 ** -14), (3, -2000, -2.0 ** -20), (9, 777777, 2.0 ** -30),
                                          (2, -31, 2.0 ** -34), (77, 123456, -2.0 ** -26)]):
        z = np.zeros(s)
        nz = rng.choice(np.arange(1, s), 6, replace=False)
        z[nz] = rng.uniform(-1, 1, 6)
        scale = 2.0 ** 20
        with localcontext() as ctx:
            ctx.prec = 90
            rest = D.encode_values_exact(np.r_[0.0, z[1:]], scale, N)[t]
            coef = Decimal(float(scale)) / N * 2 * D.dec_cos(pi * t / N)
            target = Decimal(K) + (Decimal("0.5") if K >= 0 else Decimal("-0.5")) + Decimal(delta)
            z[0] = float((target - rest) / coef)
        want = [D.round_half_away(x) for x in D.encode_values_exact(z, scale, N)]
        pt = g.encode(z, scale)
        coeffs = o.intt(g.pt_export(pt)[0:1].copy(), 0)[0]
        got = [int(c) if c <= q0 // 2 else int(c) - q0 for c in coeffs]
        assert got == want, case
        assert (g.pt_export(pt) == o.encode(z, scale).data).all(), case
    g.close()


_ENGINE_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1810_00845_b200 import hisa as H
g = H.Context(16, [60, 50, 40], 60, seed=4, arena_bytes=8 << 30)
rng = np.random.default_rng(2)
T, OC = 45, 19                      # ragged chunk (32 + 13) and output tile (16 + 3)
hs = [g.ct_random(t, 2) for t in range(T)]
W = rng.normal(0, 0.3, (OC, T))
W[0, :] = -W[1, :]                  # negative residues (all byte planes set)
outs = g.conv_accumulate(hs, W.ravel(), 2.0 ** 30)
np.save(sys.argv[1], np.stack([g.ct_export(h) for h in outs]))
"""


def test_conv_engines_bit_identical(tmp_path):
    """K8 on the tensor cores (default) and on the CUDA cores (HISA_CONV_TC=0, read once per
    process) give the same words, at N = 2^16 with 60 / 50 / 40-bit limbs (8 / 7 / 5 byte planes),
    a ragged input chunk and a ragged output tile; the tensor-core result also equals the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    # "small": the tensor-core kernel with shared memory for ONE K-chunk per super-chunk, so the
    # second (ragged) chunk goes through the add-onto-stored-outputs path on every limb
    for tc, extra in (("1", {}), ("0", {}), ("small", {"HISA_CONV_TC": "1", "HISA_CONV_TC_SMEM": str(8 * 4608)})):
        out = tmp_path / f"conv_{tc}.npy"
        env = dict(os.environ, HISA_CONV_TC=tc)
        env.update(extra)
        subprocess.run([sys.executable, "-c", _ENGINE_SCRIPT % root, str(out)], env=env, check=True, timeout=600)
        res[tc] = np.load(out)
    assert res["1"].shape == res["0"].shape and (res["1"] == res["0"]).all()
    assert (res["small"] == res["1"]).all()
    o = Oracle(16, [60, 50, 40], 60, seed=4)
    rng = np.random.default_rng(2)
    T, OC = 45, 19
    W = rng.normal(0, 0.3, (OC, T))
    W[0, :] = -W[1, :]
    cts = [o.bench_ct(t, 2) for t in range(T)]
    for oc in (0, 7, 18):
        acc = None
        for t in range(T):
            term = o.mul_scalar(cts[t], float(W[oc, t]), 2.0 ** 30)
            acc = term if acc is None else o.add(acc, term)
        assert (res["1"][oc] == acc.data).all(), oc


def test_truncated_rotation_keys():
    """hisa_keygen(max_level): a rotation key stored for levels <= m holds exactly the words of
    the full key's digits j <= m on q_0..q_m and p (checked against the oracle's full key);
    rotations at levels <= m are bit-exact with the oracle's (full-key) rotation, the rotation at
    level m + 1 fails with NO_KEY, and a later request at a higher level regenerates the key."""
    qb = [60, 40, 40, 40, 40]
    L = len(qb)
    g, o = _pair(11, qb, 60, [], seed=5)
    N = g.N
    m = 2
    g.keygen([7, 300], False, m)
    o.keygen(rot_amounts=[7, 300])
    kL = m + 1
    for k in (7, 300):
        got = g.key_export(k, kL * 2 * (kL + 1) * N).reshape(kL, 2, kL + 1, N)
        full = o.rot_keys[k]
        assert (got[:, :, :kL] == full[:kL, :, :kL]).all()
        assert (got[:, :, kL] == full[:kL, :, L]).all()          # the special prime's limb
    for lv in (0, 1, 2):
        a = g.ct_random(40 + lv, lv)
        oa = o.bench_ct(40 + lv, lv)
        assert (g.ct_export(g.rot_left(a, 7)) == o.rot_left(oa, 7).data).all()
        hs = g.rot_left_hoisted(a, [7, 300])                   # K7 with truncated keys
        assert (g.ct_export(hs[1]) == o.rot_left(oa, 300).data).all()
    hi = g.ct_random(50, 3)
    with pytest.raises(H.HisaError) as ei:
        g.rot_left(hi, 7)
    assert ei.value.code == "NO_KEY"
    with pytest.raises(H.HisaError) as ei:
        g.keygen([9], False, L)
    assert ei.value.code == "PARAMS"
    g.keygen([7], False, 3)                                     # regenerated at level 3
    assert (g.ct_export(g.rot_left(hi, 7)) == o.rot_left(o.bench_ct(50, 3), 7).data).all()
    g.keygen([7], False, 1)                                     # lower request keeps level 3
    assert g.key_export(7, 4 * 2 * 5 * N).size == 4 * 2 * 5 * N
    g.close()


def test_conv_tc_squeezenet_shape_sampled():
    """K8 at the shape the bench's config-5 leg spends its conv time in (N = 2^16, a 60-bit q_0 +
    15 x 40-bit limbs, T = 144 inputs = 16 channels x 9 taps, OC = 64: one super-chunk of five
    K-chunks per CTA, two CTAs per SM, four output tiles) -- three sampled output channels against
    the oracle's mulScalar + add chain, all words."""
    qb = [60] + [40] * 15
    g = H.Context(16, qb, 60, seed=6, arena_bytes=24 << 30)
    o = Oracle(16, qb, 60, seed=6)
    T, OC = 144, 64
    lvl = len(qb) - 1
    hs = [g.ct_random(t, lvl) for t in range(T)]
    W = np.random.default_rng(12).normal(0, 0.05, (OC, T))
    outs = g.conv_accumulate(hs, W.ravel())
    cts = [o.bench_ct(t, lvl) for t in range(T)]
    for oc in (0, 37, 63):
        acc = None
        for t in range(T):
            term = o.mul_scalar(cts[t], float(W[oc, t]))
            acc = term if acc is None else o.add(acc, term)
        assert (g.ct_export(outs[oc]) == acc.data).all(), oc
    g.close()


def test_conv_tc_all_plane_counts():
    """Every byte-plane specialisation of the tensor-core K8: 45-bit (P = 6), 30-bit (P = 4) and
    24 / 22-bit limbs (P = 3, run as 4 with a zero plane) beside the 60 / 50 / 40-bit ones of the
    other conv tests (P = 8 / 7 / 5); ragged chunk and output tile, negative weights."""
    qb = [45, 30, 24, 22]
    g = H.Context(12, qb, 60, seed=8, arena_bytes=2 << 30)
    o = Oracle(12, qb, 60, seed=8)
    T, OC = 40, 5
    lvl = len(qb) - 1
    hs = [g.ct_random(t, lvl) for t in range(T)]
    W = np.random.default_rng(13).normal(0, 0.4, (OC, T))
    outs = g.conv_accumulate(hs, W.ravel(), 2.0 ** 20)
    cts = [o.bench_ct(t, lvl) for t in range(T)]
    for oc in range(OC):
        acc = None
        for t in range(T):
            term = o.mul_scalar(cts[t], float(W[oc, t]), 2.0 ** 20)
            acc = term if acc is None else o.add(acc, term)
        assert (g.ct_export(outs[oc]) == acc.data).all(), oc
    g.close()
