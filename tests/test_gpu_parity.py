"""GPU parity: libhisa (sm_100a, via the C-ABI binding) vs the CPU oracle, bit for bit.

Every case feeds identical seeded inputs to both sides: ChaCha20 streams (keys, encryption
randomness, BENCH residues) are generated independently on each side from the same seed (A11);
float inputs come from synth/.  Ciphertexts are compared word by word after canonical export.
"""
import numpy as np
import pytest

from oracle.ckks import Ct, Oracle, Pt

pytestmark = pytest.mark.gpu

H = pytest.importorskip("paper_1810_00845_b200.hisa")

# (log_n, q_bits, p_bits): several tiles per pass and odd log N splits (M1 != M2)
PARAMS = {
    "n10": (10, [60, 40, 40], 60),
    "n11_odd": (11, [50] * 5, 60),
    "c1_n13": (13, [60, 40, 40], 60),
    "c2_n14": (14, [50] * 8, 60),
    "n15_odd": (15, [60, 40, 40, 40], 60),
    # N = 2^16 runs the register-direct M = 256 kernels (k_fwd_cols_r16 / k_fwd_rows_r16 / K4
    # k_ks_ip5); mixed 60 / 50 / 40-bit moduli: integer-engine rows and wide FP64 lifts
    "n16_mixed": (16, [60, 50, 40, 50], 60),
}
SEED = 1234


class Pair:
    def __init__(self, log_n, qb, pb, rots=(1, 3)):
        self.g = H.Context(log_n, qb, pb, seed=SEED, arena_bytes=3 << 30)
        self.o = Oracle(log_n, qb, pb, seed=SEED)
        assert self.g.moduli == self.o.moduli
        self.rots = list(rots)
        self.g.keygen(self.rots, True)
        self.o.keygen(rot_amounts=self.rots)

    def ct(self, b, level=None, npolys=2):
        level = self.o.L - 1 if level is None else level
        h = self.g.ct_random(b, level, npolys)
        oc = self.o.bench_ct(b, level, npolys)
        assert (self.g.ct_export(h) == oc.data).all(), "BENCH sampler mismatch"
        return h, oc

    def pt(self, b, level=None):
        level = self.o.L - 1 if level is None else level
        h = self.g.pt_random(b, level)
        op = self.o.bench_pt(b, level)
        assert (self.g.pt_export(h) == op.data).all()
        return h, op

    def same(self, h, oc: Ct):
        got = self.g.ct_export(h)
        lv, npl, sc = self.g.ct_info(h)
        assert (lv, npl) == (oc.level, oc.npolys)
        assert sc == oc.scale
        if not (got == oc.data).all():
            bad = np.argwhere(got != oc.data)
            raise AssertionError(f"{len(bad)} words differ, first at {bad[0].tolist()}")


@pytest.fixture(scope="module", params=sorted(PARAMS))
def pair(request):
    log_n, qb, pb = PARAMS[request.param]
    p = Pair(log_n, qb, pb, rots=(1, 3, (1 << (log_n - 1)) - 1))
    yield p
    p.g.close()


def test_keys_bit_exact(pair):
    g, o = pair.g, pair.o
    N, L = o.N, o.L
    assert (g.key_export(-2, (L + 1) * N).reshape(L + 1, N) == o.s_ntt).all()
    assert (g.key_export(-1, 2 * L * N).reshape(2, L, N) == o.pk).all()
    kw = L * 2 * (L + 1) * N
    assert (g.key_export(0, kw).reshape(o.rlk.shape) == o.rlk).all()
    for k in pair.rots:
        assert (g.key_export(k, kw).reshape(o.rlk.shape) == o.rot_keys[k]).all()


def test_ntt_intt_bit_exact(pair):
    h, oc = pair.ct(11)
    pair.g.ntt(h, False)
    want = np.stack([pair.o.ntt(oc.data[p], 0) for p in range(2)])
    assert (pair.g.ct_export(h) == want).all()
    pair.g.ntt(h, True)
    assert (pair.g.ct_export(h) == oc.data).all()


def test_elementwise_bit_exact(pair):
    g, o = pair.g, pair.o
    a, oa = pair.ct(1)
    b, ob = pair.ct(2)
    p, op = pair.pt(3)
    pair.same(g.add(a, b), o.add(oa, ob))
    pair.same(g.sub(a, b), o.sub(oa, ob))
    pair.same(g.add_plain(a, p), o.add_plain(oa, op))
    pair.same(g.sub_plain(a, p), o.sub_plain(oa, op))
    pair.same(g.mul_plain(a, p), o.mul_plain(oa, op))
    for x in (0.5, -1.25, 3.0e-3):
        pair.same(g.mul_scalar(a, x), o.mul_scalar(oa, x))
        pair.same(g.mul_scalar(a, x, 2.0 ** 30), o.mul_scalar(oa, x, 2.0 ** 30))
        pair.same(g.add_scalar(a, x), o.add_scalar(oa, x))
        pair.same(g.sub_scalar(a, x), o.sub_scalar(oa, x))
    pair.same(g.mul_norelin(a, b), o.mul_norelin(oa, ob))
    pair.same(g.mul_norelin(a, a), o.mul_norelin(oa, oa))
    pair.same(g.mod_switch(a, 1), o.mod_switch(oa, 1))


def test_rescale_bit_exact(pair):
    g, o = pair.g, pair.o
    for npolys in (2, 3):
        a, oa = pair.ct(4, npolys=npolys)
        r, orr = g.rescale(a), o.rescale(oa)
        pair.same(r, orr)
        if orr.level > 0:
            pair.same(g.div_scalar(r, o.q[orr.level]), o.div_scalar(orr, o.q[orr.level]))


def test_relinearize_bit_exact(pair):
    g, o = pair.g, pair.o
    a, oa = pair.ct(5, npolys=3)
    g.relinearize(a)
    pair.same(a, o.relinearize(oa))
    b, ob = pair.ct(6)
    c, oc = pair.ct(7)
    pair.same(g.mul(b, c), o.mul(ob, oc))


def test_rotation_bit_exact(pair):
    g, o = pair.g, pair.o
    a, oa = pair.ct(8)
    for k in pair.rots:
        pair.same(g.rot_left(a, k), o.rot_left(oa, k))
    k = pair.rots[0]
    pair.same(g.rot_right(a, o.slots - k), o.rot_left(oa, k))
    pair.same(g.rot_left(a, 0), oa)
    # lower level: keys truncated to the active limbs
    lo = g.mod_switch(a, 1)
    pair.same(g.rot_left(lo, 3), o.rot_left(o.mod_switch(oa, 1), 3))
    # in-place (Assign) form reuses the handle
    h = g.copy(a)
    assert g.rot_left(h, 1, inplace=True) == h
    pair.same(h, o.rot_left(oa, 1))


def test_rotation_batch_and_hoisted_bit_exact(pair):
    g, o = pair.g, pair.o
    hs, os_ = zip(*[pair.ct(20 + i) for i in range(3)])
    outs = g.rot_left_batch(list(hs), 3)
    for h, oc in zip(outs, os_):
        pair.same(h, o.rot_left(oc, 3))
    outs = g.rot_left_hoisted(hs[0], pair.rots)
    for h, k in zip(outs, pair.rots):
        pair.same(h, o.rot_left(os_[0], k))


def test_encode_encrypt_decrypt_bit_exact(pair):
    g, o = pair.g, pair.o
    rng = np.random.default_rng(0)
    for n in (o.slots, 37):      # full and ragged slot counts
        z = rng.uniform(0, 1, n)
        hp = g.encode(z, 2.0 ** 40)
        op = o.encode(z, 2.0 ** 40)
        assert (g.pt_export(hp) == op.data).all()
        hc = g.encrypt(hp)
        oc = o.encrypt(op)
        pair.same(hc, oc)
        hd = g.decrypt(hc)
        od = o.decrypt(oc)
        assert (g.pt_export(hd) == od.data).all()
        # fresh-encryption noise in a slot grows ~ N (sqrt(N) coefficient noise x sqrt(N) slot sum;
        # measured 1.1e-6 at N = 2^16, scale 2^40): 2^-20 up to N = 2^15, x N / 2^15 beyond
        assert np.abs(g.decode(hd, n) - z).max() < 2.0 ** -20 * max(1, o.N >> 15)
        assert np.abs(g.decode(hd, n) - o.decode(od, n)).max() < 1e-12


def test_conv_accumulate_bit_exact(pair):
    g, o = pair.g, pair.o
    T, OC = 5, 3
    hs, os_ = zip(*[pair.ct(40 + i) for i in range(T)])
    W = np.random.default_rng(3).normal(0, 0.1, (OC, T))
    outs = g.conv_accumulate(list(hs), W.ravel())
    for oi in range(OC):
        acc = None
        for t in range(T):
            term = o.mul_scalar(os_[t], float(W[oi, t]))
            acc = term if acc is None else o.add(acc, term)
        pair.same(outs[oi], acc)


def test_semantics_rotation_mul(pair):
    g, o = pair.g, pair.o
    z = np.random.default_rng(1).uniform(0, 1, o.slots)
    c = g.encrypt(g.encode(z, 2.0 ** 40))
    grow = max(1, o.N >> 15)          # slot noise ~ N (see test_encode_encrypt_decrypt_bit_exact)
    for k in pair.rots:
        r = g.decode(g.decrypt(g.rot_left(c, k)), o.slots)
        assert np.abs(r - np.roll(z, -k)).max() < 1e-6 * grow
    if o.L >= 2:
        sq = g.rescale(g.mul(c, c))
        _, _, sc = g.ct_info(sq)
        # fresh-noise bound ~ N sigma ||s|| / scale; with 50-bit primes the rescaled scale is 2^30
        tol = 1e-5 * max(1.0, 2.0 ** 40 / sc) * grow
        assert np.abs(g.decode(g.decrypt(sq), o.slots) - z * z).max() < tol


def test_error_contract(pair):
    g, o = pair.g, pair.o
    a, _ = pair.ct(50)
    with pytest.raises(H.HisaError) as ei:
        g.add(a, g.mod_switch(a, 1))
    assert ei.value.code == "LEVEL_MISMATCH"
    with pytest.raises(H.HisaError) as ei:
        g.rot_left(a, 2)
    assert ei.value.code == "NO_KEY"
    with pytest.raises(H.HisaError) as ei:
        g.bootstrap(a)
    assert ei.value.code == "UNSUPPORTED_PROFILE"
    with pytest.raises(H.HisaError) as ei:
        g.div_scalar(a, 12345)
    assert ei.value.code == "INVALID_DIVISOR"
    with pytest.raises(H.HisaError) as ei:
        g.encode(np.zeros(o.slots + 1), 2.0 ** 40)
    assert ei.value.code == "CAPACITY"
    t = g.mul_norelin(a, a)
    with pytest.raises(H.HisaError) as ei:
        g.rot_left(t, 1)
    assert ei.value.code == "NOT_RELINEARIZED"
    x = g.copy(a)
    g.free(x)
    with pytest.raises(H.HisaError) as ei:
        g.add(x, a)
    assert ei.value.code == "INVALID_HANDLE"
    lo = g.mod_switch(a, o.L - 1)
    with pytest.raises(H.HisaError) as ei:
        g.rescale(lo)
    assert ei.value.code == "MODULUS_EXHAUSTED"
    assert g.max_scalar_div(a, 2 ** 62) == o.q[o.L - 1]
    assert g.max_scalar_div(a, 2) == 1
    assert not g.supports(H.PROFILE_BOOTSTRAP) and g.supports(H.PROFILE_RELIN)


def test_hoisted_many_amounts_and_levels(pair):
    """K7 chunking (> 8 amounts), zero amounts (copies), and a lower level (truncated keys)."""
    g, o = pair.g, pair.o
    s = o.slots
    extra = [5, 7, 9, 11, 13, 17, 19, 23, 29, 31]
    g.keygen(extra, False)
    for k in extra:
        o.add_rot_key(k)
    a, oa = pair.ct(60)
    ks = [0] + extra + [1, s + 3]           # s + 3 normalises to 3
    outs = g.rot_left_hoisted(a, ks)
    for h, k in zip(outs, ks):
        pair.same(h, o.rot_left(oa, k))
    if o.L >= 2:
        lo, olo = g.mod_switch(a, 1), o.mod_switch(oa, 1)
        for h, k in zip(g.rot_left_hoisted(lo, extra[:3]), extra[:3]):
            pair.same(h, o.rot_left(olo, k))


def test_exchange_fixups(pair):
    """a15 device steps: conv accumulation into caller memory + adoption of int64 sums."""
    import torch
    g, o = pair.g, pair.o
    T, OC = 3, 2
    hs, os_ = zip(*[pair.ct(70 + i) for i in range(T)])
    W = np.random.default_rng(5).normal(0, 0.1, (OC, T))
    l1 = o.L
    buf = torch.zeros((OC, 2, l1, o.N), dtype=torch.int64, device="cuda")
    g.conv_accumulate_dev(list(hs), W.ravel(), buf.data_ptr())
    ref = [o.add(o.add(o.mul_scalar(os_[0], W[i, 0]), o.mul_scalar(os_[1], W[i, 1])), o.mul_scalar(os_[2], W[i, 2]))
           for i in range(OC)]
    for i in range(OC):
        assert (buf[i].cpu().numpy().view(np.uint64) == ref[i].data).all()
    # int64 sum of up to 8 reduced residue arrays -> residues (exact, < 2^63)
    s8 = buf[0] * 8
    h = g.ct_adopt_sum(s8.data_ptr(), o.L - 1, 2, ref[0].scale)
    want = ref[0].data
    for _ in range(7):
        want = o.add(Ct(want, ref[0].level, ref[0].scale), ref[0]).data
    assert (g.ct_export(h) == want).all()


@pytest.mark.slow
def test_full_size_bench_config_rotation():
    """BASELINE.json config 2 top point at full size (N = 2^16, L = 24, dnum = L), in the launch
    configuration bench.py times (batched K4 path, B = 8 ciphertexts, one key), sampled: two of
    the eight outputs are compared word for word with the oracle; plus one hoisted pair."""
    import synth
    log_n, L = 16, 24
    k = synth.rot_amount(0, log_n, L)
    g = H.Context(log_n, [50] * L, 60, seed=0)
    o = Oracle(log_n, [50] * L, 60, seed=0)
    assert g.moduli == o.moduli
    g.keygen([k, 1], False)
    o.keygen(rot_amounts=[k, 1], relin=False)
    cts = [g.ct_random(b, L - 1) for b in range(8)]
    outs = g.rot_left_batch(cts, k)
    for b in (0, 7):
        oc = o.bench_ct(b, L - 1)
        assert (g.ct_export(outs[b]) == o.rot_left(oc, k).data).all(), f"ct {b}"
    oc0 = o.bench_ct(0, L - 1)
    hz = g.rot_left_hoisted(cts[0], [k, 1])
    assert (g.ct_export(hz[1]) == o.rot_left(oc0, 1).data).all()
    g.close()


@pytest.mark.parametrize("fill", ["max", "half", "alt", "zero_one"])
def test_extreme_residues_ntt_and_keyswitch(pair, fill):
    """Adversarial residues for the lazy-reduction bounds of both engines (the FP64 engine runs
    every modulus < 2^50, ntt_f64.cuh; the 60-bit moduli run the integer one): every word q-1,
    (q-1)/2, alternating q-1 / 0, or 0 / 1.  NTT, INTT, rotation (ModUp + ModDown) and rescale
    must equal the oracle bit for bit."""
    g, o = pair.g, pair.o
    L, N = o.L, o.N
    data = np.zeros((2, L, N), dtype=np.uint64)
    for i in range(L):
        q = o.q[i]
        if fill == "max":
            data[:, i, :] = q - 1
        elif fill == "half":
            data[:, i, :] = (q - 1) // 2
        elif fill == "alt":
            data[:, i, 0::2] = q - 1
        else:
            data[:, i, 1::2] = 1
    h = g.ct_import(data, L - 1, 2, 2.0 ** 40)
    oc = Ct(data.copy(), L - 1, 2.0 ** 40)
    pair.same(g.rot_left(h, pair.rots[0]), o.rot_left(oc, pair.rots[0]))
    if L >= 2:
        pair.same(g.rescale(h), o.rescale(oc))
    g.ntt(h, False)
    want = np.stack([o.ntt(data[p], 0) for p in range(2)])
    assert (g.ct_export(h) == want).all()
    g.ntt(h, True)
    assert (g.ct_export(h) == data).all()


def test_conv_accumulate_large_t_worst_case(pair):
    """K8 across weight tiles (T > 256) and past the 128-bit headroom of 60-bit moduli (partial
    reductions every 2^127 / q^2 terms): inputs all q - 1 and weights with residue q - 1
    (X = -1), plus random weights; OC not a multiple of the 8-output register tile."""
    g, o = pair.g, pair.o
    L, N = o.L, o.N
    T, OC = 300, 11
    data = np.zeros((2, L, N), dtype=np.uint64)
    for i in range(L):
        data[:, i, :] = o.q[i] - 1
    h = g.ct_import(data, L - 1, 2, 2.0 ** 40)
    oc = Ct(data.copy(), L - 1, 2.0 ** 40)
    ps = float(o.q[L - 1])
    W = np.full((OC, T), -1.0 / ps)
    W[5:] = np.random.default_rng(9).normal(0, 0.3, (OC - 5, T))
    outs = g.conv_accumulate([h] * T, W.ravel())
    for oi in (0, 4, 5, OC - 1):
        acc = None
        for t in range(T):
            term = o.mul_scalar(oc, float(W[oi, t]))
            acc = term if acc is None else o.add(acc, term)
        pair.same(outs[oi], acc)


def test_fused_rot_add_and_mulplain_accumulate(pair):
    """The fused driver kernels equal their HISA definitions bit for bit: rot_add_batch =
    add(x, rotLeft(x, k)); mul_plain_accumulate = sum_c mulPlain(x_c, p_{j,c})."""
    g, o = pair.g, pair.o
    hs, os_ = zip(*[pair.ct(80 + i) for i in range(3)])
    k = pair.rots[1]
    for h, oc in zip(g.rot_add_batch(list(hs), k), os_):
        pair.same(h, o.add(oc, o.rot_left(oc, k)))
    C, J = 3, 5
    pts = [pair.pt(90 + i) for i in range(C * J)]
    outs = g.mul_plain_accumulate(list(hs), [p[0] for p in pts], J)
    for j in range(J):
        acc = None
        for c in range(C):
            term = o.mul_plain(os_[c], pts[j * C + c][1])
            acc = term if acc is None else o.add(acc, term)
        pair.same(outs[j], acc)


def test_batched_mul_and_rescale(pair):
    """hisa_mul_batch / hisa_rescale_batch == the per-ciphertext hisa_mul / hisa_rescale."""
    g, o = pair.g, pair.o
    hs, os_ = zip(*[pair.ct(100 + i) for i in range(3)])
    outs = g.mul_batch([hs[0], hs[1], hs[2]], [hs[0], hs[2], hs[2]])
    pair.same(outs[0], o.mul(os_[0], os_[0]))
    pair.same(outs[1], o.mul(os_[1], os_[2]))
    pair.same(outs[2], o.mul(os_[2], os_[2]))
    if o.L >= 2:
        for h, oc in zip(g.rescale_batch(list(hs)), os_):
            pair.same(h, o.rescale(oc))


def test_hoisted_batch_many_cts(pair):
    """hisa_rot_left_hoisted_batch: 5 ciphertexts (K7 groups of 4 + 1) x 6 amounts (key chunks
    of 4 + 2) incl. a zero amount, == per-ciphertext rotLeft bit for bit."""
    g, o = pair.g, pair.o
    extra = [5, 7, 9, 11, 13]
    g.keygen(extra, False)
    for k in extra:
        o.add_rot_key(k)
    hs, os_ = zip(*[pair.ct(110 + i) for i in range(5)])
    ks = [5, 0, 7, 9, 11, 13]
    outs = g.rot_left_hoisted_batch(list(hs), ks)
    for i in (0, 3, 4):
        for r, k in enumerate(ks):
            pair.same(outs[i][r], o.rot_left(os_[i], k))


def test_encode_batch_bit_exact(pair):
    """hisa_encode_batch (host threads + batched GPU NTT) == the oracle's exact encoder (A7),
    including sparse weight-like vectors and a ragged slot count."""
    g, o = pair.g, pair.o
    rng = np.random.default_rng(11)
    vs = rng.normal(0, 0.1, (5, 40))
    vs[1, ::3] = 0.0
    vs[2, :] = 0.0
    lv = o.L - 1
    hs = g.encode_batch(vs, float(o.q[lv]), lv)
    for h, v in zip(hs, vs):
        assert (g.pt_export(h) == o.encode(v, float(o.q[lv]), lv).data).all()


@pytest.mark.parametrize("nz", [1, 2, 4, 5, 7, 8, 11])
def test_k4_batch_shapes_and_long_digit_chains(nz):
    """K4 at M = 256 (N = 2^15) in every CTA shape (ciphertexts x rows per CTA: 8x1, 4x1, 2x2,
    1x4; a batch is split into groups of 8k / 4 / 2 / 1: 5 = 4 + 1, 7 = 4 + 2 + 1, 11 = 8 + 2 + 1)
    with 13 digits (the FP64 accumulators are re-centred every 6
    products): a batched rotation of nz ciphertexts, one of them all (q - 1) residues (the
    largest lifted digits and MAC operands), equal to the oracle word for word."""
    log_n, qb = 15, [60] + [50] * 12
    g = H.Context(log_n, qb, 60, seed=7, arena_bytes=8 << 30)
    o = Oracle(log_n, qb, 60, seed=7)
    L = len(qb)
    g.keygen([5], False)
    o.keygen(rot_amounts=[5], relin=False)
    hs, ocs = [], []
    for b in range(nz):
        if b == nz - 1:
            data = np.stack([np.stack([np.full(o.N, q - 1, dtype=np.uint64) for q in o.q[:L]])] * 2)
            hs.append(g.ct_import(data, L - 1, 2, 2.0 ** 40))
            ocs.append(Ct(data.copy(), L - 1, 2.0 ** 40))
        else:
            hs.append(g.ct_random(300 + b, L - 1))
            ocs.append(o.bench_ct(300 + b, L - 1))
    outs = g.rot_left_batch(hs, 5)
    for b, (h, oc) in enumerate(zip(outs, ocs)):
        want = o.rot_left(oc, 5).data
        got = g.ct_export(h)
        assert (got == want).all(), f"ct {b}: {int((got != want).sum())} words differ"
    g.close()


def test_gpu_decode_batch(pair):
    """NEXT-4: decode on the GPU (INTT of limb 0, centred lift, twist, double FFT, gather).  A batch
    of plaintexts (fresh encodings at two scales and a decrypted product) decodes within 1e-12 of the
    oracle's long-double decode (decode is approximate by definition), equal to
    one-at-a-time decoding, and an empty batch / n = 0 are no-ops."""
    g, o = pair.g, pair.o
    rng = np.random.default_rng(99)
    n = o.slots
    zs = [rng.uniform(-1, 1, n), rng.uniform(0, 1, n // 3), np.linspace(-2, 2, n)]
    hs, ods = [], []
    for z, sc in zip(zs, (2.0 ** 40, 2.0 ** 30, 2.0 ** 40)):
        hs.append(g.encode(z, sc))
        ods.append(o.encode(z, sc))
    got = g.decode_batch(hs, n)
    for i, (h, od) in enumerate(zip(hs, ods)):
        ref = o.decode(od, n)
        assert np.abs(got[i] - ref).max() < 1e-12 * max(1.0, np.abs(ref).max()), f"pt {i}"
        assert (got[i] == g.decode(h, n)).all()
    assert g.decode_batch([], n).shape == (0, n)
    assert g.decode_batch(hs[:1], 0).shape == (1, 0)


def test_mul_plain_batch(pair):
    """hisa_mul_plain_batch: n mulPlains in one launch equal the per-pair oracle products; mixed
    levels are refused; an empty batch is a no-op."""
    g, o = pair.g, pair.o
    hs, ocs = zip(*[pair.ct(500 + i) for i in range(3)])
    ps, ops = zip(*[pair.pt(600 + i) for i in range(3)])
    for h, oc, op in zip(g.mul_plain_batch(list(hs), list(ps)), ocs, ops):
        pair.same(h, o.mul_plain(oc, op))
    assert g.mul_plain_batch([], []) == []
    if o.L > 1:
        lo = g.mod_switch(hs[0], 1)
        with pytest.raises(H.HisaError) as ei:
            g.mul_plain_batch([lo, hs[1]], [ps[0], ps[1]])
        assert ei.value.code == "LEVEL_MISMATCH"
