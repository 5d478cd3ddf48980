"""Multi-GPU exchange of the encrypted CNN driver.

One process per GPU (torch.distributed, NCCL over NVLink / NVSwitch).  Between layers every
rank holds its own block of channels (EncryptedNet.owned).  Convolutions (partition "ic", the
default): every conv's input channels are partitioned across ranks: rank r hoists the rotations
of ITS input channels only, and accumulates partial sums for ALL outputs; the exchange is one
reduce-scatter per conv of those partials as int64 (SUM):

  * exact -- each partial word is a fully reduced residue < q_i < 2^60 and world <= 8, so every
    sum is < 2^63; hisa_ct_adopt_sum reduces it back into [0, q_i) on the device;
  * the scattered block of rank r is exactly its owned output channels, which are its input
    shard of the next layer -- so no all-gather is needed between layers;
  * ModDown / rescale run only after the complete sum, so the outputs at 1 / 2 / 4 / 8 ranks
    are bit-identical to the single-GPU result (modular addition is order independent).

Partition "oc" (the north star's output-channel split, kept as the measured baseline) and every
FC layer (SURVEY 8e's FC plan): the layer's input channels are all-gathered (gather_outputs) and
each rank computes its own output channels / neurons / R-groups from all of them -- no partial
sums cross ranks, so the outputs are bit-identical by construction; the cost is that every rank
repeats the inputs' rotations.

The partial buffers are torch int64 tensors (PyTorch owns device memory); libhisa writes the
partial sums into them directly (hisa_conv_accumulate_dev) or they are copied from ciphertext
device views, and the reduced blocks are adopted back as ciphertexts (hisa_ct_adopt_sum).
"""
from __future__ import annotations

import numpy as np


class _DevArray:
    """A raw device pointer as a CUDA-array-interface object (for torch.as_tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False), "version": 3}


def _words(ptr: int, n: int, dev):
    """n int64 words at `ptr` as a tensor on `dev` (zero-copy): a libhisa device view, or -- for a
    host-memory backend (the CPU test double of tests/test_parallel_cpu.py) -- host memory."""
    import torch
    if dev.type == "cuda":
        return torch.as_tensor(_DevArray(ptr, n), device=dev)
    import ctypes
    return torch.from_numpy(np.ctypeslib.as_array((ctypes.c_int64 * n).from_address(ptr)))


def _host_staged(t, group) -> bool:
    """gloo cannot reduce CUDA tensors: stage through host memory (transport only; used by the
    multi-process emulation of several GPUs on one device in tests/test_multigpu_emulated.py --
    NCCL, the production transport, takes device tensors directly)."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def exchange(buf, per: int, group):
    """Reduce-scatter (int64 SUM) of a [world * per, ...] partial buffer: returns this rank's
    [per, ...] block (the NCCL step of a15)."""
    import torch
    import torch.distributed as dist
    if _host_staged(buf, group):
        torch.cuda.current_stream().synchronize()
        out = exchange(buf.cpu(), per, group)
        return out.to(buf.device)
    out = torch.empty((per,) + tuple(buf.shape[1:]), dtype=buf.dtype, device=buf.device)
    dist.reduce_scatter_tensor(out, buf, op=dist.ReduceOp.SUM, group=group)
    return out


def _all_gather(out, inp, group):
    import torch
    import torch.distributed as dist
    if _host_staged(inp, group):
        torch.cuda.current_stream().synchronize()
        o = torch.empty(out.shape, dtype=out.dtype)
        dist.all_gather_into_tensor(o, inp.cpu(), group=group)
        out.copy_(o)
        return
    dist.all_gather_into_tensor(out, inp, group=group)


def _all_reduce_max(t, group):
    import torch
    import torch.distributed as dist
    if _host_staged(t, group):
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX, group=group)
        t.copy_(c)
        return
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)


def layer_meta(en, handles, device):
    """(level, scale) of a layer's ciphertexts agreed by all ranks: ranks that own no input
    channel contribute (-1, 0).  All data-holding ranks already agree (deterministic plan)."""
    import torch
    import torch.distributed as dist
    if handles:
        lv, _np, sc = en.b.ct_info(handles[0])
    else:
        lv, sc = -1, 0.0
    t = torch.tensor([float(lv), float(sc)], dtype=torch.float64, device=device)
    _all_reduce_max(t, en.group)
    return int(t[0].item()), float(t[1].item())


def _device(en):
    import torch
    from .driver import Symbolic
    if isinstance(en.b, Symbolic) or getattr(en.b, "host_memory", False):
        return torch.device("cpu")
    return torch.device("cuda", torch.cuda.current_device())


def _per(en, n_out):
    return -(-n_out // en.world)


def reduce_scatter_partials(en, rotated, wmat: np.ndarray, n_out: int):
    """Scalar-MAC partial sums (conv taps, slot-0 FC) for all n_out outputs over this rank's
    inputs -> reduce-scatter -> this rank's owned outputs (pre-rescale ciphertexts)."""
    import torch
    from .driver import Symbolic
    dev = _device(en)
    lv, sc_in = layer_meta(en, rotated, dev)
    ps = float(en.q[lv])
    per = _per(en, n_out)
    own = en.owned(n_out)
    if isinstance(en.b, Symbolic):
        en.b._count("scalar_mac_ct", int(wmat.size))
        buf = torch.zeros((en.world * per, 1), dtype=torch.int64)
        exchange(buf, per, en.group)
        return [en.b.fresh(lv, sc_in * ps) for _ in own]
    N = 2 * en.slots
    buf = torch.zeros((en.world * per, 2, lv + 1, N), dtype=torch.int64, device=dev)
    if rotated:
        en.b.conv_accumulate_dev(rotated, np.ascontiguousarray(wmat).ravel(), buf.data_ptr())
    blk = exchange(buf, per, en.group)
    return [en.b.ct_adopt_sum(blk[i].data_ptr(), lv, 2, sc_in * ps) for i in range(len(own))]


def gather_outputs(en, cts, n_out: int):
    """All-gather the final layer's owned outputs so every rank (rank 0 decrypts) holds all
    n_out ciphertexts (all-gather at the end)."""
    import torch
    import torch.distributed as dist
    from .driver import Symbolic
    dev = _device(en)
    lv, sc = layer_meta(en, cts, dev)
    per = _per(en, n_out)
    if isinstance(en.b, Symbolic):
        buf = torch.zeros((per, 1), dtype=torch.int64)
        allb = torch.zeros((en.world * per, 1), dtype=torch.int64)
        _all_gather(allb, buf, en.group)
        return [en.b.fresh(lv, sc) for _ in range(n_out)]
    N = 2 * en.slots
    words = 2 * (lv + 1) * N
    buf = torch.zeros((per, words), dtype=torch.int64, device=dev)
    for i, h in enumerate(cts):
        ptr, w = en.b.ct_device_view(h)
        buf[i].copy_(_words(ptr, w, dev))
    allb = torch.empty((en.world * per, words), dtype=torch.int64, device=dev)
    _all_gather(allb, buf, en.group)
    return [en.b.ct_adopt_device(allb[j].data_ptr(), lv, 2, sc) for j in range(n_out)]
