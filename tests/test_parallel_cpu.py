"""Multi-rank encrypted inference on CPU: the product driver and its exchange
code (paper_1810_00845_b200/parallel.py) run over gloo at world 2, 4 and 8 -- one process per
"GPU" -- on the oracle test double (tests/oracle_backend.py), with real ciphertexts.  Both conv
partitions (input channels + int64 reduce-scatter; the north star's output channels + all-gather)
and the FC plan (inputs all-gathered, neurons / R-groups partitioned) must give final ciphertexts
bit-identical to the one-rank run, including uneven shards (5 channels over 4 ranks: 2, 2, 1, 0;
over 8 ranks: ranks 5-7 own nothing)."""
import os
import socket

import numpy as np
import pytest

from synth import nets as SN

# conv 3 -> 5 (padded), act, pool, SAME conv 5 -> 5 after the pool (mask), act, FC with R = 2
# replicas (6 neurons -> 3 R-groups), act, FC from the replica layout (4), act, FC from slot 0 (3)
NET_A = dict(log_n=11, q_bits=[60] + [40] * 12, p_bits=60, scale=2.0 ** 40, input=(3, 6, 6),
             layers=[("conv", 5, 3, 1, 1), ("act",), ("avgpool",), ("conv", 5, 3, 1, 1), ("act",),
                     ("fc", 6, 2), ("act",), ("fc", 4), ("act",), ("fc", 3)],
             sigma=[0.4] * 5, act_gains=[4.0, 16.0, 4.0, 16.0])
# fire modules + global average pool, 5 channels into the first fire, FC-free
NET_B = dict(log_n=11, q_bits=[60] + [40] * 13, p_bits=60, scale=2.0 ** 40, input=(2, 8, 8),
             layers=[("conv", 5, 3, 1, 1), ("act",), ("avgpool",), ("fire", 3, 2, 3), ("avgpool",),
                     ("fire", 2, 3, 2), ("conv", 3, 1, 1, 0), ("gap",)], sigma=[0.5] * 8,
             act_gains=[4.0, 16.0, 64.0, 4.0 ** 4, 4.0 ** 4])


def _weights(net, seed):
    SN.NETS["_par"] = net
    try:
        shapes = SN.linear_shapes("_par")
    finally:
        del SN.NETS["_par"]
    return [SN._weights(seed + i, s, net["sigma"][i]) for i, s in enumerate(shapes)]


CASES = [("A", NET_A, 401), ("B", NET_B, 501)]


def _run(net, W, img, group=None, partition="ic"):
    from tests.oracle_backend import OracleBackend
    from paper_1810_00845_b200.driver import EncryptedNet
    b = OracleBackend(net["log_n"], net["q_bits"], net["p_bits"], seed=3)
    plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, b.moduli)
    EncryptedNet.keygen(b, plan)
    en = EncryptedNet(b, net, W, SN.ACT_COEFFS, group=group, partition=partition)
    cts, lay = en.encrypt_image(img)
    if group is not None:
        cts = en.shard_input(cts)
    out, lo = en.forward_gathered(cts, lay)
    data = [b.objs[h].data.copy() for h in out]
    dec = en.decrypt_output(out, lo)
    return data, dec


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
        res = {}
        for name, net, seed in CASES:
            W = _weights(net, seed)
            img = SN._image(seed, net["input"])
            for part in ("ic", "oc"):
                res[(name, part)] = _run(net, W, img, group=dist.group.WORLD, partition=part)
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


_REF = {}


def _reference():
    """One-rank runs (computed once per session), checked against the float64 networks."""
    from oracle import plain
    if not _REF:
        for name, net, seed in CASES:
            W = _weights(net, seed)
            img = SN._image(seed, net["input"])
            _REF[name] = _run(net, W, img)
            want = plain.forward(net, img, W, SN.ACT_COEFFS)
            err = np.abs(_REF[name][1] - want).max()
            assert err <= 1e-4 * np.abs(want).max(), (name, err)
    return _REF


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_inference_bit_identical(world):
    import torch.multiprocessing as mp
    ref = _reference()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        for name, _net, _s in CASES:
            for part in ("ic", "oc"):
                data, dec = got[r][(name, part)]
                rdata, rdec = ref[name]
                assert len(data) == len(rdata), (r, name, part)
                for a, b in zip(data, rdata):
                    assert np.array_equal(a, b), (world, r, name, part)
                assert np.array_equal(dec, rdec)
