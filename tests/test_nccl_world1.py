"""Rows a15 / (e) on NCCL: the box has one GPU, so the only NCCL group that can exist is a
one-rank group -- but it drives the production data plane end to end: int64 partial sums written
by hisa_conv_accumulate_dev into a torch device buffer, `reduce_scatter_tensor` / 
`all_gather_into_tensor` on the NCCL communicator (device tensors, zero-copy views of libhisa
memory), hisa_ct_adopt_sum, the final gather.  Both partitionings (SURVEY 8e input-channel
reduce-scatter, north-star output-channel all-gather) must reproduce the plain single-GPU
ciphertexts bit for bit.  (World 2/4/8 with uneven shards: gloo tests in test_parallel_cpu.py /
test_driver_host.py / test_multigpu_emulated.py.)"""
import os
import socket

import pytest

from synth import nets as SN

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(port, name, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    try:
        from paper_1810_00845_b200 import hisa as H
        from paper_1810_00845_b200.driver import EncryptedNet
        net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 1)
        g = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=5, device=0, arena_bytes=12 << 30)
        plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, g.moduli)
        EncryptedNet.keygen(g, plan)
        plain = EncryptedNet(g, net, W, SN.ACT_COEFFS)
        cts, lay = plain.encrypt_image(img)
        ref, _ = plain.forward([g.copy(h) for h in cts], lay)
        ref = [g.ct_export(h) for h in ref]
        res = {"backend": dist.get_backend(), "launch_calls": {}}
        for part in ("ic", "oc"):
            en = EncryptedNet(g, net, W, SN.ACT_COEFFS, group=dist.group.WORLD, partition=part,
                              exchange_at_world1=True)
            assert en.sharded and en.world == 1
            mine = en.shard_input([g.copy(h) for h in cts])
            out, _ = en.forward_gathered(mine, lay)
            got = [g.ct_export(h) for h in out]
            res[part] = len(got) == len(ref) and all((a == b).all() for a, b in zip(got, ref))
        g.close()
        torch.cuda.synchronize()
        q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["tiny", "lenet_small"])
def test_nccl_data_plane_world1_bit_identical(name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_run, args=(_free_port(), name, q))
    p.start()
    res = q.get(timeout=900)
    p.join(timeout=120)
    assert p.exitcode == 0
    assert res["backend"] == "nccl"
    assert res["ic"] and res["oc"]
