"""Encrypted CNN driver (rows a9-a12): GPU driver vs the oracle's independent Alg. 1 lowering,
bit for bit after every layer, and decrypted outputs vs the float64 plaintext network
(max-abs <= 1e-3, BASELINE.json north star / A36)."""
import numpy as np
import pytest

from synth import nets as SN

pytestmark = pytest.mark.gpu

H = pytest.importorskip("paper_1810_00845_b200.hisa")


def _run_pair(name, image_seed=0):
    from oracle import plain
    from oracle.nets import OracleNet
    from paper_1810_00845_b200.driver import EncryptedNet

    net = SN.NETS[name]
    W = SN.net_weights(name)
    img = SN.net_image(name, image_seed)
    ref = plain.forward(net, img, W, SN.ACT_COEFFS)

    on = OracleNet(net, W, SN.ACT_COEFFS, seed=0)
    ocs, olay = on.encrypt_image(img)
    otrace = []
    ocs_out, olay_out = on.forward(ocs, olay, trace=otrace)

    g = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=0, arena_bytes=8 << 30)
    assert g.moduli == on.o.moduli
    plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, g.moduli)
    assert plan["rotations"] == on.amounts          # the compiler's key selection
    g.keygen(plan["rotations"], True)
    en = EncryptedNet(g, net, W, SN.ACT_COEFFS)
    cts, lay = en.encrypt_image(img)
    for h, oc in zip(cts, ocs):
        assert (g.ct_export(h) == oc.data).all(), "input encryption parity"
    gtrace = []
    out, lay_out = en.forward(cts, lay, trace=lambda li, hs, ly: gtrace.append((li, [g.ct_export(h) for h in hs],
                                                                               [g.ct_info(h) for h in hs])))
    for (li, gd, gi), (oli, octs) in zip(gtrace, otrace):
        assert li == oli and len(gd) == len(octs)
        for c, (d, info, oc) in enumerate(zip(gd, gi, octs)):
            assert info[0] == oc.level and info[2] == oc.scale, f"layer {li} ch {c}: level/scale"
            if not (d == oc.data).all():
                raise AssertionError(f"layer {li} {net['layers'][li]} channel {c}: "
                                     f"{int((d != oc.data).sum())} words differ")
    got = en.decrypt_output(out, lay_out)
    ogot = on.decrypt_output(ocs_out, olay_out)
    g.close()
    return got, ogot, ref


@pytest.mark.parametrize("name", ["tiny", "lenet_small"])
def test_driver_bit_exact_and_accurate(name):
    got, ogot, ref = _run_pair(name)
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 1e-3, np.abs(got - ref).max()
    assert np.abs(got - ogot).max() < 1e-9
