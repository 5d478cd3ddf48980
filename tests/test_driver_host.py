"""Host-side driver logic (no GPU): the symbolic planner (the paper's analysers),
the compile-time folding (A25, A26), the oracle's lowering pinned to the float64 definition on
small networks that exercise every branch, and the multi-rank path over gloo (world size 2)."""
import math
import os
import socket

import numpy as np
import pytest

from synth import nets as SN


def _moduli(net):
    from oracle.ckks import Oracle
    return Oracle(net["log_n"], net["q_bits"], net["p_bits"]).moduli


# every lowering branch: padded first conv, act, avgpool, SAME conv on a pooled (unclean)
# input -> mask, FC from the HW layout (mulPlain + rotate-and-sum), FC from slot 0
MINI = dict(log_n=11, q_bits=[60] + [40] * 8, p_bits=60, scale=2.0 ** 40, input=(2, 8, 8),
            layers=[("conv", 2, 3, 1, 1), ("act",), ("avgpool",), ("conv", 2, 3, 1, 1), ("act",),
                    ("fc", 3), ("act",), ("fc", 2)], sigma=[0.3, 0.3, 0.3, 0.3])


# replica FC (A27): pooled 3x3 plane (span 37 -> block 64), R = 4 neurons per ciphertext, then
# an FC reading the replica layout
MINI_REP = dict(log_n=11, q_bits=[60] + [40] * 6, p_bits=60, scale=2.0 ** 40, input=(2, 6, 6),
                layers=[("conv", 2, 3, 1, 1), ("act",), ("avgpool",), ("fc", 6, 4), ("act",), ("fc", 3)],
                sigma=[0.3, 0.3, 0.3])


def _mini_rep_weights():
    shapes = [(2, 2, 3, 3), (6, 2 * 3 * 3), (3, 6)]
    return [SN._weights(91 + i, s, 0.3) for i, s in enumerate(shapes)]


# SqueezeNet-shaped (config 5 layer kinds): padded 3x3 conv, pools, two fire modules (squeeze,
# mask, fused 1x1 || 3x3 SAME expand), final 1x1 conv, global average pool; compile-time gains
MINI_SQ = dict(log_n=11, q_bits=[60] + [40] * 13, p_bits=60, scale=2.0 ** 40, input=(3, 8, 8),
               layers=[("conv", 4, 3, 1, 1), ("act",), ("avgpool",), ("fire", 2, 2, 2), ("avgpool",),
                       ("fire", 2, 3, 1), ("conv", 3, 1, 1, 0), ("gap",)], sigma=[0.5] * 8,
               act_gains=[4.0, 16.0, 64.0, 4.0 ** 4, 4.0 ** 4])     # A41 gains on every fire path


def _mini_sq_weights():
    from synth import nets as _n
    saved = _n.NETS.get("_mini_sq")
    _n.NETS["_mini_sq"] = MINI_SQ
    try:
        shapes = _n.linear_shapes("_mini_sq")
    finally:
        if saved is None:
            del _n.NETS["_mini_sq"]
    return [SN._weights(31 + i, s, 0.5) for i, s in enumerate(shapes)]


# CHW-tiled second conv (NEXT-1): pooled 4x4 planes (hS 20, wS 2), SAME 3x3 -> block stride 128,
# 8 channels per ciphertext (4 channels -> one packed ciphertext), then FC
MINI_CHW = dict(log_n=11, q_bits=[60] + [40] * 6, p_bits=60, scale=2.0 ** 40, input=(2, 8, 8),
                layers=[("conv", 4, 3, 1, 1), ("act",), ("avgpool",), ("conv", 3, 3, 1, 1, "chw"), ("act",),
                        ("fc", 2)], sigma=[0.3, 0.3, 0.3])


def _mini_chw_weights():
    shapes = [(4, 2, 3, 3), (3, 4, 3, 3), (2, 3 * 4 * 4)]
    return [SN._weights(51 + i, s, 0.3) for i, s in enumerate(shapes)]


# CHW-tiled FC (NEXT-1, the paper's "CHW-fc" layouts): pooled 4x4 planes (span 67 -> block 128),
# 3 channels -> one packed ciphertext (G = 4), 3 neurons from one mulPlain each, then slot-0 FC
MINI_CHWFC = dict(log_n=11, q_bits=[60] + [40] * 7, p_bits=60, scale=2.0 ** 40, input=(2, 8, 8),
                  layers=[("conv", 3, 3, 1, 1), ("act",), ("avgpool",), ("fc", 3, 1, "chw"), ("act",),
                          ("fc", 2)], sigma=[0.3, 0.3, 0.3])


def _mini_chwfc_weights():
    shapes = [(3, 2, 3, 3), (3, 3 * 4 * 4), (2, 3)]
    return [SN._weights(61 + i, s, 0.3) for i, s in enumerate(shapes)]


def _mini_weights():
    shapes = [(2, 2, 3, 3), (2, 2, 3, 3), (3, 2 * 4 * 4), (2, 3)]
    return [SN._weights(77 + i, s, 0.3) for i, s in enumerate(shapes)]


def test_plan_tiny_rotation_set_and_levels():
    from paper_1810_00845_b200.driver import EncryptedNet
    net = SN.NETS["tiny"]
    pl = EncryptedNet.plan(net, SN.net_weights("tiny"), SN.ACT_COEFFS, _moduli(net))
    # 3x3 taps on an 8-wide channel: fh*8 + fw
    assert pl["rotations"] == [1, 2, 8, 9, 10, 16, 17, 18]
    assert pl["levels_used"] == 2 and pl["final_level"] == 0        # A28: 2 of 2
    assert pl["counts"]["rot_hoisted"] == 8                          # IC * (K^2 - 1)


def test_plan_spec_example_rotation_set():
    """a 3x3 filter on a 5x5 channel with hS = 5 needs left rotations
    {1, 2, 5, 6, 7, 10, 11, 12}; rotations counted IC * (K^2 - 1), independent of OC."""
    from paper_1810_00845_b200.driver import EncryptedNet
    for oc in (1, 4):
        net = dict(log_n=10, q_bits=[60, 40], p_bits=60, scale=2.0 ** 40, input=(3, 5, 5),
                   layers=[("conv", oc, 3, 1, 0)], sigma=[0.1])
        w = [SN._weights(1, (oc, 3, 3, 3), 0.1)]
        pl = EncryptedNet.plan(net, w, SN.ACT_COEFFS, _moduli(net))
        assert pl["rotations"] == [1, 2, 5, 6, 7, 10, 11, 12]
        assert pl["counts"]["rot_hoisted"] == 3 * 8
        assert pl["counts"]["scalar_mac_ct"] == oc * 3 * 9


def test_plan_lenet_small_levels():
    from paper_1810_00845_b200.driver import EncryptedNet
    import copy
    net = SN.NETS["lenet_small"]
    pl = EncryptedNet.plan(net, SN.net_weights("lenet_small"), SN.ACT_COEFFS, _moduli(net))
    assert pl["levels_used"] == 6                                    # FC1 with R = 8: mask + 5 = 6 of 6
    assert pl["counts"]["rot_hoisted"] == 24
    # R = 8: replicate 5 channels (3 rotations each), 13 groups x 10 rotate-and-sum steps inside
    # the 1024-slot blocks, FC2 reads the replica layout: 10 outputs x 3 cross-block steps
    assert pl["counts"]["rot"] == 5 * 3 + 13 * 10 + 10 * 3
    r1 = copy.deepcopy(net)
    r1["layers"][2] = ("fc", 100)
    pl1 = EncryptedNet.plan(r1, SN.net_weights("lenet_small"), SN.ACT_COEFFS, _moduli(net))
    assert pl1["levels_used"] == 5                                   # A28 with R = 1: 5 of 6
    # FC1 rotate-and-sum: 100 neurons x ceil(log2(12*60 + 12*2 + 1)) = 10 steps
    assert pl1["counts"]["rot"] == 100 * 10


def test_fold_identity():
    """A25 (+ A41 gain G): G (a2 x^2 + a1 x + a0) == (r x + beta)^2 + gamma (one level)."""
    from paper_1810_00845_b200.driver import act_fold
    x = np.linspace(-3, 3, 101)
    for coeffs in (SN.ACT_COEFFS, (0.1, -0.7, 2.0), (1.0, 0.0, 0.5)):
        for G in (1.0, 4.0, 4.0 ** 7):
            r, beta, gamma = act_fold(coeffs, G)
            a0, a1, a2 = coeffs
            assert np.allclose((r * x + beta) ** 2 + gamma, G * (a0 + a1 * x + a2 * x * x), rtol=1e-12, atol=1e-12 * G)


def test_compile_weights_pool_and_act_factors():
    from paper_1810_00845_b200.driver import compile_weights
    w = _mini_weights()
    folded, gammas, gains = compile_weights(MINI, w, SN.ACT_COEFFS)
    r = math.sqrt(SN.ACT_COEFFS[2])
    assert np.allclose(folded[0][0], w[0] * r) and folded[0][1] == pytest.approx(0.5)   # act after
    assert np.allclose(folded[1][0], w[1] * 0.25 * r)                                    # pool before
    assert np.allclose(folded[3][0], w[3]) and folded[3][1] == 0.0                       # last layer
    assert gammas == [pytest.approx(-0.25)] * 3
    assert [g for g, _o in gains] == [r, 1.0, 4.0, r, 1.0, r, 1.0, 1.0]      # the pool holds 4 x its mean


def test_compile_weights_gains():
    """A41: with activation gains G_n every encrypted tensor holds G x its value: the linear layer
    before activation n is scaled by sqrt(a2 G_n) / G_(n-1), its bias is sqrt(a2 G_n) a1 / (2 a2),
    gamma_n = G_n gamma; other linear layers keep the gain (the output is decoded / G_last)."""
    import copy
    from paper_1810_00845_b200.driver import compile_weights
    net = copy.deepcopy(MINI)
    net["act_gains"] = [16.0, 4.0 ** 5, 4.0]
    w = _mini_weights()
    folded, gammas, gains = compile_weights(net, w, SN.ACT_COEFFS)
    a0, a1, a2 = SN.ACT_COEFFS
    assert np.array_equal(folded[0][0], w[0] * math.sqrt(a2 * 16))
    assert np.array_equal(folded[1][0], w[1] * 0.25 * math.sqrt(a2 * 4 ** 5) / 16)
    assert np.array_equal(folded[2][0], w[2] * math.sqrt(a2 * 4) / 4 ** 5)
    assert np.array_equal(folded[3][0], w[3])
    assert folded[1][1] == math.sqrt(a2 * 4 ** 5) * a1 / (2 * a2)
    assert gammas == [16 * -0.25, 4 ** 5 * -0.25, 4 * -0.25]
    r1, r2, r3 = (math.sqrt(a2 * G) for G in (16, 4 ** 5, 4))
    assert gains == [(r1, r1), (16.0, 0.0), (64.0, 0.0), (r2, r2), (4.0 ** 5, 0.0), (r3, r3), (4.0, 0.0),
                     (4.0, 0.0)]           # (gain, offset) of each layer's output; beta = r here
    with pytest.raises(ValueError):
        net["act_gains"] = [2.0, 4.0, 4.0]          # not a power of 4
        compile_weights(net, w, SN.ACT_COEFFS)


def test_act_gains_follow_calibration_rule():
    """The stored act_gains (synth/nets.py) are what tools/calibrate_gains.py's rule gives
    (floor(log4(16 / max|act|)) on the float64 network, calibration image seed 1007), and every
    gained activation output peaks in (4, 16] (bounds |x'^2| = G/4 . (...) well inside the
    modulus, A41)."""
    from tools import calibrate_gains as CG
    for name in ("lenet_small", "lenet_large", "lenet_large_chw", "squeezenet"):
        net = SN.NETS[name]
        img = SN._image(CG.CALIB_SEED, net["input"])
        base = "lenet_large" if name == "lenet_large_chw" else name
        W = SN.net_weights(base)
        assert CG.gains_for(net, W, img) == net["act_gains"], name
        for g, m in zip(net["act_gains"], CG.act_maxima(net, W, img, SN.ACT_COEFFS)):
            assert 4.0 < g * m <= 16.0 or g == 1.0


def test_oracle_net_tiny_matches_float64():
    from oracle import plain
    from oracle.nets import OracleNet
    net = SN.NETS["tiny"]
    W = SN.net_weights("tiny")
    img = SN.net_image("tiny", 3)
    on = OracleNet(net, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(net, img, W, SN.ACT_COEFFS)
    assert got.shape == (2, 6, 6)
    assert np.abs(got - ref).max() <= 1e-3
    assert out[0].level == 0


def test_oracle_net_every_branch_matches_float64():
    """Pins the oracle's lowering (mask, SAME padding through wrap-around, pools, both FC
    forms, folded activations) to the float64 definition of the network."""
    from oracle import plain
    from oracle.nets import OracleNet
    W = _mini_weights()
    img = SN._image(5, MINI["input"])
    on = OracleNet(MINI, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(MINI, img, W, SN.ACT_COEFFS)
    assert got.shape == ref.shape == (2,)
    assert np.abs(got - ref).max() <= 1e-3, (got, ref)


def test_oracle_net_replica_fc_matches_float64():
    """Pins the oracle's replica FC lowering (mask, log R replication, block rotate-and-sum,
    FC from the replica layout) to the float64 network."""
    from oracle import plain
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet
    W = _mini_rep_weights()
    img = SN._image(6, MINI_REP["input"])
    on = OracleNet(MINI_REP, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(MINI_REP, img, W, SN.ACT_COEFFS)
    assert got.shape == ref.shape == (3,)
    assert np.abs(got - ref).max() <= 1e-3, (got, ref)
    pl = EncryptedNet.plan(MINI_REP, W, SN.ACT_COEFFS, on.o.moduli)
    assert pl["rotations"] == on.amounts
    assert pl["levels_used"] == 6


def test_plan_lenet_large_replicas():
    """Config 4 with FC1 at R = 16 (A27): 2048 weight plaintexts instead of 32768, 9 of 13
    levels (SURVEY A.4 plans 8-11)."""
    from paper_1810_00845_b200.driver import EncryptedNet
    net = SN.NETS["lenet_large"]
    pl = EncryptedNet.plan(net, SN.net_weights("lenet_large"), SN.ACT_COEFFS, _moduli(net))
    assert pl["levels_used"] == 9
    assert pl["counts"]["rot_hoisted"] == 24 + 32 * 3 + 32 * 24 + 64 * 3
    fc_pts = pl["counts"]["encode"] - 2          # minus the two mask plaintexts
    assert fc_pts == 32 * 64 + 10 * 32


def test_oracle_net_squeezenet_kinds_match_float64():
    """Pins the oracle's fire-module and global-average-pool lowering to the float64 net."""
    from oracle import plain
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet
    W = _mini_sq_weights()
    img = SN._image(8, MINI_SQ["input"])
    on = OracleNet(MINI_SQ, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(MINI_SQ, img, W, SN.ACT_COEFFS)
    assert got.shape == ref.shape == (3,)
    assert np.abs(got - ref).max() <= 1e-3, (got, ref)
    pl = EncryptedNet.plan(MINI_SQ, W, SN.ACT_COEFFS, on.o.moduli)
    assert pl["rotations"] == on.amounts
    assert pl["levels_used"] == 13 and pl["final_level"] == 0


def test_plan_squeezenet_levels():
    """Config 5 (A33): 1 + 4 x 5 + 1 + 1 = 23 of 23 levels with masked fire expands (A24)."""
    from paper_1810_00845_b200.driver import EncryptedNet
    net = SN.NETS["squeezenet"]
    pl = EncryptedNet.plan(net, SN.net_weights("squeezenet"), SN.ACT_COEFFS, _moduli(net))
    assert pl["levels_used"] == 23 and pl["final_level"] == 0
    # hoisted rotations: conv1 3 x 8, fire expands 16,16,32,32 input channels x 8, pools 64 x 3 x 2
    assert pl["counts"]["rot_hoisted"] == 3 * 8 + (16 + 16 + 32 + 32) * 8 + 64 * 3 * 2


def test_plan_matches_oracle_rotation_selection():
    """The product planner and the oracle's own walk select the same key set (independent
    implementations of the same lowering)."""
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet
    W = _mini_weights()
    on = OracleNet(MINI, W, SN.ACT_COEFFS)
    pl = EncryptedNet.plan(MINI, W, SN.ACT_COEFFS, on.o.moduli)
    assert pl["rotations"] == on.amounts
    assert pl["levels_used"] == 8


# ------------------------------------------------------------------------------ gloo, world 2 / 4 / 8
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_1810_00845_b200 import parallel
        from paper_1810_00845_b200.driver import EncryptedNet, Symbolic, input_layout
        res = {}
        # (1) the numeric exchange: int64 SUM reduce-scatter of reduced residues
        qm = (1 << 60) - 93
        rng = np.random.default_rng(100 + rank)
        per = 3
        parts = torch.from_numpy(rng.integers(0, qm, size=(world * per, 5), dtype=np.int64))
        res["parts"] = parts.numpy().copy()
        res["block"] = parallel.exchange(parts, per, None).numpy()
        # (2) the sharded driver on the symbolic backend (metadata + real collectives), both
        # conv partitions
        net = SN.NETS["lenet_small"]
        from oracle.ckks import Oracle
        mod = Oracle(net["log_n"], net["q_bits"], net["p_bits"]).moduli
        for part in ("ic", "oc"):
            sym = Symbolic(net["log_n"], mod)
            en = EncryptedNet(sym, net, SN.net_weights("lenet_small"), SN.ACT_COEFFS, group=dist.group.WORLD,
                              partition=part)
            lay = input_layout(net)
            cts = en.shard_input([sym.fresh(len(mod) - 2, net["scale"]) for _ in range(lay.C)])
            out, ol = en.forward_gathered(cts, lay)
            res[part] = dict(n_out=len(out), final_level=sym.cts[out[0]][0], counts=sym.counts,
                             rotations=sorted(sym.rotations))
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multirank_gloo(world):
    """Exchange numerics and the sharded plan at world 2 / 4 / 8 (lenet_small: 5 conv channels ->
    uneven shards, idle ranks at world 8).  "ic": the (ic, tap) rotations and scalar MACs are
    partitioned (they sum to the single-GPU counts); "oc": every rank repeats the conv's
    rotations and owns its output channels.  FC layers (8e plan): mulPlains partitioned."""
    import torch.multiprocessing as mp
    from oracle.ckks import Oracle
    from paper_1810_00845_b200.driver import EncryptedNet
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # exchange: rank r's block = rows [3r, 3r+3) summed over ranks (< 2^63, exact)
    total = sum(got[r]["parts"] for r in range(world))
    for r in range(world):
        assert (got[r]["block"] == total[3 * r:3 * r + 3]).all()
    net = SN.NETS["lenet_small"]
    single = EncryptedNet.plan(net, SN.net_weights("lenet_small"), SN.ACT_COEFFS,
                               Oracle(net["log_n"], net["q_bits"], net["p_bits"]).moduli)
    for part in ("ic", "oc"):
        for r in range(world):
            g = got[r][part]
            assert g["n_out"] == 10 and g["final_level"] == single["final_level"]
            assert set(g["rotations"]) <= set(single["rotations"])
        total = {k: sum(got[r][part]["counts"].get(k, 0) for r in range(world))
                 for k in ("scalar_mac_ct", "rot_hoisted", "mul_plain")}
        assert total["scalar_mac_ct"] == single["counts"]["scalar_mac_ct"]
        assert total["mul_plain"] == single["counts"]["mul_plain"]
        want_h = single["counts"]["rot_hoisted"] * (world if part == "oc" else 1)
        assert total["rot_hoisted"] == want_h


def test_oracle_pow2_policy_matches_float64_and_planner():
    """NEXT-2 pin: the oracle's power-of-two composition (signed-binary digits) decrypts within
    1e-3 of the float64 network on every lowering branch, its key set is powers of two (left or
    right), and the product planner selects the same keys."""
    from oracle import plain
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet
    W = _mini_weights()
    img = SN._image(5, MINI["input"])
    on = OracleNet(MINI, W, SN.ACT_COEFFS, rot_policy="pow2")
    s = on.o.slots
    assert all((k & (k - 1)) == 0 or ((s - k) & (s - k - 1)) == 0 for k in on.amounts)
    # composition is exact in Z_s: the steps of every amount sum to it
    for k in (1, 3, 7, 13, 31, s - 3, s // 2 + 5):
        assert sum(on._steps(k)) % s == k % s
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(MINI, img, W, SN.ACT_COEFFS)
    assert np.abs(got - ref).max() <= 1e-3
    pl = EncryptedNet.plan(MINI, W, SN.ACT_COEFFS, on.o.moduli, rot_policy="pow2")
    assert pl["rotations"] == on.amounts


def test_oracle_chw_conv_matches_float64_and_planner():
    """NEXT-1 pin: the oracle's CHW-tiled conv (packing, per-block mulPlain, cross-block
    rotate-and-sum) decrypts within 1e-3 of the float64 network; the planner agrees on keys."""
    from oracle import plain
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet
    W = _mini_chw_weights()
    img = SN._image(12, MINI_CHW["input"])
    on = OracleNet(MINI_CHW, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(MINI_CHW, img, W, SN.ACT_COEFFS)
    assert got.shape == ref.shape == (2,)
    assert np.abs(got - ref).max() <= 1e-3, (got, ref)
    pl = EncryptedNet.plan(MINI_CHW, W, SN.ACT_COEFFS, on.o.moduli)
    assert pl["rotations"] == on.amounts
    assert pl["levels_used"] == 6


def test_oracle_chw_fc_matches_float64_and_planner():
    """NEXT-1 pin: the oracle's CHW-tiled FC (mask, pack G channels per ciphertext, one mulPlain
    per (neuron, packed ciphertext), rotate-and-sum over G blocks) decrypts within 1e-3 of the
    float64 network, and the product planner selects the same keys and levels."""
    from oracle import plain
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet
    W = _mini_chwfc_weights()
    img = SN._image(13, MINI_CHWFC["input"])
    on = OracleNet(MINI_CHWFC, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    ref = plain.forward(MINI_CHWFC, img, W, SN.ACT_COEFFS)
    assert got.shape == ref.shape == (2,)
    assert np.abs(got - ref).max() <= 1e-3, (got, ref)
    pl = EncryptedNet.plan(MINI_CHWFC, W, SN.ACT_COEFFS, on.o.moduli)
    assert pl["rotations"] == on.amounts
    assert pl["levels_used"] == 6          # conv, act, mask, FC, act, FC


def test_plain_reference_ops_match_torch():
    """Pins oracle/plain.py (the float64 definition the decrypted outputs are held to) against an
    independent library routine: torch.nn.functional conv2d / avg_pool2d / linear in float64,
    including strided, padded and multi-channel cases."""
    import torch
    import torch.nn.functional as F
    from oracle import plain
    rng = np.random.default_rng(3)
    for (c, h, w, oc, k, s, p) in [(1, 8, 8, 2, 3, 1, 0), (1, 28, 28, 5, 5, 2, 1), (3, 9, 7, 4, 3, 1, 1),
                                   (2, 6, 6, 3, 1, 1, 0)]:
        x = rng.normal(size=(c, h, w))
        wt = rng.normal(size=(oc, c, k, k))
        want = F.conv2d(torch.from_numpy(x)[None], torch.from_numpy(wt), stride=s, padding=p)[0].numpy()
        assert np.allclose(plain.conv2d(x, wt, s, p), want, atol=1e-12)
    x = rng.normal(size=(4, 14, 14))
    assert np.allclose(plain.avgpool2(x), F.avg_pool2d(torch.from_numpy(x)[None], 2)[0].numpy(), atol=1e-14)
    net = dict(layers=[("conv", 2, 3, 1, 1), ("act",), ("avgpool",), ("fc", 3)], input=(1, 6, 6))
    W = [rng.normal(size=(2, 1, 3, 3)), rng.normal(size=(3, 18))]
    img = rng.uniform(size=(1, 6, 6))
    y = F.conv2d(torch.from_numpy(img)[None], torch.from_numpy(W[0]), padding=1)
    y = 0.0 + 0.5 * y + 0.25 * y * y
    y = F.avg_pool2d(y, 2).reshape(-1)
    want = F.linear(y, torch.from_numpy(W[1])).numpy()
    assert np.allclose(plain.forward(net, img, W, SN.ACT_COEFFS), want, atol=1e-12)


@pytest.mark.slow
def test_oracle_squeezenet_shape_relative_error_n4096():
    """Config 5's network (A33 shapes, its N(0, 0.05) weights, its act_gains) on the oracle at
    N = 2^12 (24 x 40-bit limbs; the 32 x 32 planes fit 2048 slots): decrypted logits within
    1e-4 RELATIVE to the float64 network (max |ref| ~ 3e-7, so an absolute bound alone would
    pass an all-zero output).  Measured: 1.4e-7 with the gains, 0.16 without them (same N, same
    image) -- the CKKS error floor is what the gains (A41) keep the signal above."""
    import copy
    from oracle import plain
    from oracle.nets import OracleNet
    net = copy.deepcopy(SN.NETS["squeezenet"])
    net["log_n"] = 12
    W, img = SN.net_weights("squeezenet"), SN.net_image("squeezenet", 0)
    ref = plain.forward(net, img, W, SN.ACT_COEFFS)
    on = OracleNet(net, W, SN.ACT_COEFFS)
    cts, lay = on.encrypt_image(img)
    out, ol = on.forward(cts, lay)
    got = on.decrypt_output(out, ol)
    rel = np.abs(got - ref).max() / np.abs(ref).max()
    assert rel <= 1e-4, rel
    assert np.abs(got - ref).max() <= 1e-3


def test_golden_plain_outputs_are_the_float64_network():
    """tests/golden/plain_outputs.json (bench.py's accuracy reference) = oracle/plain.py on the
    stated weights and images (spot check: first and last image of two nets)."""
    import json
    from oracle import plain
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "plain_outputs.json")))
    assert gold["images"] == 20
    for name in ("tiny", "lenet_small"):
        W = SN.net_weights(name)
        for s in (0, 19):
            ref = plain.forward(SN.NETS[name], SN.net_image(name, s), W, SN.ACT_COEFFS).ravel()
            assert np.array_equal(np.asarray(gold["outputs"][name][s]), ref)
