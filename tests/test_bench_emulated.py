"""bench.py's N > 1 code path (torchrun launch, barriers, max-over-ranks timing, sharded inference
in both partitionings) on the one GPU of the box: two ranks share the device
(HISA_BENCH_SHARED_DEVICE) and the collectives run on gloo (NCCL refuses two ranks on one
device).  The numbers are meaningless (two ranks time-slice one GPU); the JSON contract and the
absence of errors are what is checked."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_bench_two_ranks_one_gpu():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, HISA_BENCH_SHARED_DEVICE="1", HISA_BENCH_BACKEND="gloo", HISA_BENCH_ARENA_GB="24")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(root, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--nets", "tiny,lenet_small",
           "--no-cpu-baseline", "--no-e2e", "--no-hoisted"]
    r = subprocess.run(cmd, env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["global_batch"] == 2 * d["config"]["batch_per_gpu"]
    inf = d["inference"]
    assert {(e["config"], e["partition"]) for e in inf} == {(n, p) for n in ("tiny", "lenet_small") for p in ("ic", "oc")}
    for e in inf:
        assert "error" not in e, e
        assert e["latency_s"] > 0
