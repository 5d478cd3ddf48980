"""Row a15 end to end on one B200: two processes (ranks) share the GPU, each with its own libhisa
context, and run the input-channel-sharded network with the real exchange code path
(conv_accumulate_dev -> reduce-scatter of int64 partial sums -> hisa_ct_adopt_sum, final
all-gather).  The collectives use gloo staged through host memory (NCCL refuses two ranks on one
device; no kernel waits on another rank).  SURVEY 8e: the sharded outputs must be bit-identical to
the single-GPU run."""
import os
import socket

import numpy as np
import pytest

from synth import nets as SN

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1810_00845_b200 import hisa as H
        from paper_1810_00845_b200.driver import EncryptedNet
        net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 1)
        g = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=5, device=0, arena_bytes=12 << 30)
        plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, g.moduli)
        EncryptedNet.keygen(g, plan)
        en = EncryptedNet(g, net, W, SN.ACT_COEFFS, group=dist.group.WORLD)
        cts, lay = en.encrypt_image(img)
        mine = en.shard_input(cts)
        out, lo = en.forward_gathered(mine, lay)
        res = [g.ct_export(h) for h in out] if rank == 0 else None
        q.put((rank, res))
        g.close()
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["tiny", "lenet_small"])
def test_sharded_network_bit_identical(name):
    import torch.multiprocessing as mp
    from paper_1810_00845_b200 import hisa as H
    from paper_1810_00845_b200.driver import EncryptedNet
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=900) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # the single-GPU reference (same seed -> same keys and encryptions)
    net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 1)
    g = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=5, arena_bytes=12 << 30)
    plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, g.moduli)
    EncryptedNet.keygen(g, plan)
    en = EncryptedNet(g, net, W, SN.ACT_COEFFS)
    cts, lay = en.encrypt_image(img)
    out, _ = en.forward(cts, lay)
    ref = [g.ct_export(h) for h in out]
    g.close()
    assert len(got[0]) == len(ref)
    for a, b in zip(got[0], ref):
        assert a.shape == b.shape and (a == b).all()
