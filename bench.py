#!/usr/bin/env python
"""bench.py -- key-switch rotations/s at N=2^16 (BASELINE.json metric, config 2 top point).

Workload: RNS-CKKS N = 2^16, L = 24 limbs of 50-bit primes + one
60-bit special prime, dnum = L; B ciphertexts per GPU at the top level with uniform residues
(ChaCha20 tag BENCH, resident in HBM before timing), one rotation amount k (A30).  One step =
hisa_rot_left_batch over the B ciphertexts: automorphism + the full key switch (INTT, ModUp,
key inner product, ModDown) for every ciphertext.  Multi-GPU: each rank rotates its own batch
(independent ciphertexts, no data-path collective) -> "scaling": "weak".

--impl reference times the CPU oracle (oracle/) on this box's host cores on the same metric:
each step is one rotation of one ciphertext at the same parameters (a bounded sample).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "key-switch rotations/s at N=2^16"   # + "inference": encrypted CNN latency (s), configs 1 / 3
UNIT = "rot/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hisa", choices=["hisa", "reference"])
    ap.add_argument("--batch", type=int, default=8, help="ciphertexts per GPU per step")
    ap.add_argument("--log-n", type=int, default=16)
    ap.add_argument("--limbs", type=int, default=24)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-hoisted", action="store_true")
    ap.add_argument("--no-inference", action="store_true")
    ap.add_argument("--hoist-r", type=int, default=8, help="rotation amounts per hoisted ModUp")
    ap.add_argument("--nets", default="tiny,lenet_small,lenet_large,squeezenet",
                    help="encrypted-inference configs to time")
    ap.add_argument("--images", type=int, default=20, help="images averaged per inference config (P:843-844)")
    ap.add_argument("--oracle-nets", default="tiny,lenet_small",
                    help="configs whose oracle inference latency is timed on the host cores (cpu_baseline)")
    ap.add_argument("--tiling", default="lenet_small,lenet_large",
                    help="configs whose four layout strategies (Fig. tilings) are timed ('' = skip)")
    ap.add_argument("--replica-sweep", default="",
                    help="config whose first FC is timed with R = 1, 2, 4, 8 replicas (NEXT-3), e.g. lenet_small")
    ap.add_argument("--policy-net", default="lenet_small",
                    help="config on which exact vs power-of-two rotation keys are compared ('' = skip)")
    return ap.parse_args()


def workload(a):
    return {"workload": f"config2 HISA rotate sweep top point: N=2^{a.log_n}, L={a.limbs} x 50-bit q_i + 60-bit p, "
                        f"dnum=L, uniform-residue ciphertexts at the top level",
            "log_n": a.log_n, "limbs": a.limbs, "q_bits": 50, "p_bits": 60, "dnum": a.limbs}


# ------------------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event reasons sampled DURING the timed region: an NVML thread polling
    every 2 ms (the timed regions are tens of milliseconds -- shorter than nvidia-smi's first
    sample), falling back to `nvidia-smi -lms 100` where NVML is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                device = int(vis.split(",")[device])
            except (ValueError, IndexError):
                pass
        self.device = device
        self.samples = []          # (sm_mhz, max_mhz, set(reasons))
        self.proc = None
        self.thread = None
        self.stop_flag = threading.Event()
        self.source = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            bits = {"hw_slowdown": pynvml.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": pynvml.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": pynvml.nvmlClocksEventReasonSwPowerCap}
            smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))

            def poll():
                while not self.stop_flag.is_set():
                    try:
                        sm = float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((sm, smax, {n for n, b in bits.items() if r & b}))
                    except pynvml.NVMLError:
                        pass
                    time.sleep(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.source = "nvml, 2 ms"
            t0 = time.time()
            while not self.samples and time.time() - t0 < 1.0:   # first sample before the region
                time.sleep(0.001)
            self.samples.clear()
            return
        except Exception:   # noqa: BLE001 -- any NVML failure: nvidia-smi fallback
            self.thread = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.source = "nvidia-smi -lms 100"
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                try:
                    self.samples.append((float(parts[0]), float(parts[1]),
                                         {n for n, v in zip(self.NAMES, parts[3:]) if v.lower().startswith("active")}))
                except ValueError:
                    continue

    def stop(self):
        self.stop_flag.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = sorted(x[0] for x in self.samples)
        reasons = set().union(*[x[2] for x in self.samples]) if self.samples else set()
        smax = self.samples[-1][1] if self.samples else None
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "source": self.source}


# ------------------------------------------------------------------------------ work model
def kernel_units(name: str, log_n: int, l1: int, B: int) -> float:
    """Algorithmic butterflies per step for one kernel class: an NTT pass over one
    limb = (N/2) * log2(M) butterflies.  The key multiply-accumulates of the inner product run on
    another pipe (IMAD) and are counted separately (kernel_macs)."""
    N = 1 << log_n
    m1 = log_n // 2
    m2 = log_n - m1
    hb = N // 2
    per_ct = {
        "ntt_inv_rows": l1 * hb * m2,
        "ntt_inv_cols": l1 * hb * m1,
        "ks_modup_cols": l1 * l1 * hb * m1,                       # (j, r != q_j) pairs, first log M1 stages
        "ks_ip_rows": l1 * l1 * hb * m2,                          # last log M2 stages
        "ks_intt_p_rows": 2 * hb * m2,
        "ks_intt_p_cols": 2 * hb * m1,
        "ks_moddown_cols": 2 * l1 * hb * m1,
        "ks_moddown_rows": 2 * l1 * hb * m2,
    }
    return float(per_ct.get(name, 0)) * B


def kernel_macs(name: str, log_n: int, l1: int, B: int) -> float:
    """Key multiply-accumulates per step: the inner product of K4 multiplies every digit j
    (l1 of them) into the b and a key limbs of every output prime (l1 + 1) -> 2 l1 (l1+1) N."""
    if name != "ks_ip_rows":
        return 0.0
    return float(2 * l1 * (l1 + 1) * (1 << log_n)) * B


def rotation_alg_bytes(log_n: int, l1: int, B: int) -> float:
    """read ct 2(l+1) + key 2 beta (l+2) (once per same-key batch) + write 2(l+1) limbs."""
    limb = 8 * (1 << log_n)
    return (B * 4 * l1 + 2 * l1 * (l1 + 1)) * limb


K7_KEYS_PER_LAUNCH = 4   # hisa.cu rotate_hoisted_multi (RK)


def hoisted_step_bytes(log_n: int, l1: int, nct: int, R: int) -> float:
    """Compulsory HBM bytes of one hoisted step: the R keys once
    (2 l1 (l1+1) limbs each), the nct input ciphertexts (2 l1 limbs) and the nct R outputs."""
    limb = 8 * (1 << log_n)
    return (R * 2 * l1 * (l1 + 1) + nct * 2 * l1 + nct * R * 2 * l1) * limb


def measure_hoisted(ctx, cts, amounts, steps, warmup, log_n, L, stream, batched=True):
    """Hoisted rotations (the conv pattern): every ciphertext rotated by R amounts sharing
    one ModUp.  batched: one hisa_rot_left_hoisted_batch over all ciphertexts (K7 streams each
    key once per group of 4 ciphertexts; K7 of the next key group overlaps the ModDown of the
    current one on a second stream); else one hisa_rot_left_hoisted per ciphertext.  roofline_step
    = compulsory bytes (keys once + inputs + outputs) / step time against measured HBM."""
    import torch
    R = len(amounts)

    def step():
        if batched:
            for row in ctx.rot_left_hoisted_batch(cts, amounts):
                for o in row:
                    ctx.free(o)
        else:
            for h in cts:
                for o in ctx.rot_left_hoisted(h, amounts):
                    ctx.free(o)
    for _ in range(warmup):
        step()
    ctx.sync()
    ctx.profile(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    prof = ctx.profile_read()
    ctx.profile(False)
    ip_ms, ip_n = prof.get("ks_ip_hoisted", (0.0, 0))
    total = sum(v[0] for v in prof.values()) or 1.0
    per_launch = ip_ms / max(ip_n, 1)
    nct = len(cts)
    # K7's algorithmic bytes: per launch (<= 4 ciphertexts x <= 4 keys) D of each ciphertext once,
    # each key once, each accumulator written once
    limb = 8 * (1 << log_n)
    cg = min(4, nct) if batched else 1
    k7_bytes_step = (-(-R // K7_KEYS_PER_LAUNCH)) * nct * L * (L + 1) * limb + \
        (-(-nct // cg)) * R * 2 * L * (L + 1) * limb + nct * R * 2 * (L + 1) * limb
    alg = k7_bytes_step * steps / max(ip_n, 1)
    hbm_peak = _hbm_peak()
    step_bytes = hoisted_step_bytes(log_n, L, nct, R)
    step_gbs = step_bytes * steps / (ms / 1e3) / 1e9
    rot = nct * R * steps
    return {"value": rot / (ms / 1e3), "unit": "rot/s", "amounts_per_modup": R, "ciphertexts": nct,
            "call": "hisa_rot_left_hoisted_batch" if batched else "hisa_rot_left_hoisted per ciphertext",
            "ms_per_step": ms / steps,
            "roofline_step": {"bound": "hbm", "achieved": step_gbs, "peak": hbm_peak, "unit": "GB/s",
                              "frac": step_gbs / hbm_peak, "compulsory_bytes_per_step": step_bytes,
                              "model": "keys once + inputs + outputs (SURVEY 8d); ModUp / ModDown are FP64-bound "
                                       "and overlap the key stream only partly",
                              "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "roofline": {"bound": "hbm", "kernel": "ks_ip_hoisted", "achieved": alg / (per_launch / 1e3) / 1e9,
                         "peak": hbm_peak, "unit": "GB/s", "frac": alg / (per_launch / 1e3) / 1e9 / hbm_peak,
                         "alg_bytes_per_launch": alg, "launch_ms_avg": per_launch, "share_of_step": ip_ms / total,
                         "traffic": _ncu_traffic("ks_ip_hoisted", log_n, L, 8),
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "kernels": {n: {"ms": v[0], "launches": v[1], "share": v[0] / total}
                        for n, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}}


def _net_variant(name, fc_replicas=None):
    """A config with its first HW-input FC lowered with `fc_replicas` replicas (NEXT-3)."""
    from synth import nets as SN
    if fc_replicas is None:
        return name
    import copy
    net = copy.deepcopy(SN.NETS[name])
    for i, layer in enumerate(net["layers"]):
        if layer[0] == "fc":
            net["layers"][i] = ("fc", layer[1], fc_replicas)
            break
    key = f"{name}_fcR{fc_replicas}"
    SN.NETS[key] = net
    SN.NETS.setdefault("_weights_alias", {})[key] = name
    return key


def _golden_outputs(name):
    """float64 outputs of `name` on image seeds 0..19 (tests/golden/plain_outputs.json, written by
    tools/write_golden_plain.py from oracle/plain.py -- a stored reference, no oracle code runs
    here)."""
    path = os.path.join(ROOT, "tests", "golden", "plain_outputs.json")
    try:
        return json.load(open(path))["outputs"].get(name)
    except (OSError, ValueError, KeyError):
        return None


def measure_inference(name, device, images=20, rot_policy="exact"):
    """Encrypted CNN inference latency (BASELINE.json metric, second half): server-side forward
    from encrypted input resident on the GPU to encrypted output, CUDA events + wall clock,
    averaged over `images` synthetic images (seeds 0..images-1; the paper averages 20 images,
    P:843-844); client encode/encrypt and decrypt/decode timed separately; every decrypted output
    compared with the float64 network (max_abs_err, rel_err = max-abs / max |float64|)."""
    import numpy as np
    import torch
    from synth import nets as SN
    from paper_1810_00845_b200 import hisa as H
    from paper_1810_00845_b200.driver import EncryptedNet
    net = SN.NETS[name]
    base = SN.NETS.get("_weights_alias", {}).get(name, name)   # replica variants share the weights
    W = SN.net_weights(base)
    gold = _golden_outputs(base)
    torch.cuda.empty_cache()
    ctx = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=0, device=device, arena_bytes=64 << 30)
    t0 = time.perf_counter()
    plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, ctx.moduli, rot_policy=rot_policy)
    EncryptedNet.keygen(ctx, plan)
    ctx.sync()
    t_keys = time.perf_counter() - t0
    en = EncryptedNet(ctx, net, W, SN.ACT_COEFFS, rot_policy=rot_policy)
    stream = torch.cuda.current_stream(device)
    # warm-up pass: encodes (caches) the weight plaintexts once per model
    t0 = time.perf_counter()
    cts, lay = en.encrypt_image(SN.net_image(base, 0))
    out, ol = en.forward(cts, lay)
    ctx.sync()
    t_first = time.perf_counter() - t0
    for h in out + cts:
        ctx.free(h)
    lat, walls, t_encs, t_decs, errs, rels = [], [], [], [], [], []
    for r in range(images):
        img = SN.net_image(base, r)
        t0 = time.perf_counter()
        cts, lay = en.encrypt_image(img)
        ctx.sync()
        t_encs.append(time.perf_counter() - t0)
        ctx.profile(True)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        ev0.record(stream)
        out, ol = en.forward(cts, lay)
        ev1.record(stream)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - w0)
        lat.append(ev0.elapsed_time(ev1) / 1e3)
        launches = ctx.launch_count()
        prof = ctx.profile_read()
        ctx.profile(False)
        t0 = time.perf_counter()
        got = np.ravel(en.decrypt_output(out, ol))
        t_decs.append(time.perf_counter() - t0)
        if gold is not None and r < len(gold):
            ref = np.asarray(gold[r])
            errs.append(float(np.abs(got - ref).max()))
            rels.append(errs[-1] / float(np.abs(ref).max()))
        for h in out + cts:
            ctx.free(h)
    total = sum(v[0] for v in prof.values()) or 1.0
    top = sorted(prof.items(), key=lambda kv: -kv[1][0])[:6]
    ctx.close()
    ctx = None
    torch.cuda.empty_cache()
    return {"config": name, "rot_policy": rot_policy, "latency_s": float(np.mean(lat)),
            "latency_median_s": float(np.median(lat)), "latency_min_s": float(np.min(lat)),
            "wall_s": float(np.mean(walls)), "unit": "s", "images": images,
            "protocol": "mean over synthetic images seeds 0..%d, batch 1 (P:843-844)" % (images - 1),
            "log_n": net["log_n"], "limbs": len(net["q_bits"]), "gpu_launches": launches,
            "client_encrypt_s": float(np.mean(t_encs)), "client_decrypt_s": float(np.mean(t_decs)), "keygen_s": t_keys,
            "first_pass_incl_weight_encoding_s": t_first, "levels_used": plan["levels_used"],
            "rotation_keys": len(plan["rotations"]), "act_gains": net.get("act_gains"),
            "max_abs_err": max(errs) if errs else None, "rel_err": max(rels) if rels else None,
            "accuracy_ref": "float64 network (tests/golden/plain_outputs.json); rel_err = max over images of "
                            "max|dec - ref| / max|ref|" if errs else "no golden reference",
            "output_head": [float(x) for x in np.ravel(got)[:3]],
            "kernel_share": {n: round(v[0] / total, 4) for n, v in top}}


def measure_inference_sharded(name, local, dist, reps=2, partition="ic"):
    """Encrypted inference over all ranks, latency = max over ranks (CUDA events).
    partition "ic": every conv's input channels sharded, one int64 reduce-scatter per conv;
    "oc" (the north star's split, the baseline): each conv's inputs all-gathered, output channels
    partitioned.  FC layers: inputs all-gathered, neurons / R-groups partitioned; final all-gather."""
    import torch
    from synth import nets as SN
    from paper_1810_00845_b200 import hisa as H
    from paper_1810_00845_b200.driver import EncryptedNet
    net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 0)
    torch.cuda.empty_cache()
    arena = int(float(os.environ.get("HISA_BENCH_ARENA_GB", "64")) * (1 << 30))
    ctx = H.Context(net["log_n"], net["q_bits"], net["p_bits"], seed=0, device=local, arena_bytes=arena)
    plan = EncryptedNet.plan(net, W, SN.ACT_COEFFS, ctx.moduli)
    EncryptedNet.keygen(ctx, plan)
    en = EncryptedNet(ctx, net, W, SN.ACT_COEFFS, group=dist.group.WORLD, partition=partition)
    stream = torch.cuda.current_stream(local)
    lat = []
    for r in range(reps + 1):                    # first pass encodes the weight plaintexts
        cts, lay = en.encrypt_image(img)
        mine = en.shard_input(cts)
        ctx.sync()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out, lo = en.forward_gathered(mine, lay)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=f"cuda:{local}", dtype=torch.float64)
        _allreduce_max(t)
        if r:
            lat.append(float(t.item()))
        for h in out + mine:
            ctx.free(h)
    ctx.close()
    ctx = None
    torch.cuda.empty_cache()
    return {"config": name, "partition": partition, "latency_s": min(lat), "unit": "s",
            "n_gpus": dist.get_world_size(), "reps": reps,
            "sharding": ("convs: input channels sharded, NCCL reduce-scatter of int64 partial sums" if partition == "ic"
                         else "convs: inputs all-gathered, output channels partitioned (north-star baseline)") +
                        "; FCs: inputs all-gathered, neurons / R-groups partitioned; final all-gather (SURVEY 8e)"}


def _allreduce_max(t):
    """MAX all-reduce of a device scalar (NCCL directly; gloo via host memory)."""
    import torch.distributed as dist
    if dist.get_backend() == "gloo" and t.is_cuda:
        c = t.cpu()
        dist.all_reduce(c, op=dist.ReduceOp.MAX)
        t.copy_(c)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)


# the paper's CPU latencies for the same network families (context only: non-RNS HEAAN, different
# parameters, 2x Xeon E5-2667v3 with 16 threads)
PAPER_CPU_S = {"lenet_small": (8.0, "P:852"), "lenet_large": (265.0, "P:854"), "squeezenet": (1342.0, "P:856")}


def oracle_inference(name):
    """cpu_baseline leg for the inference metric: the oracle's encrypted network (oracle/nets.py,
    Alg. 1 written literally) on all host cores, one image, server-side forward only."""
    from synth import nets as SN
    from oracle.nets import OracleNet
    net, W, img = SN.NETS[name], SN.net_weights(name), SN.net_image(name, 0)
    on = OracleNet(net, W, SN.ACT_COEFFS, seed=0)
    cts, lay = on.encrypt_image(img)
    t0 = time.perf_counter()
    on.forward(cts, lay)
    dt = time.perf_counter() - t0
    return {"value": dt, "unit": "s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"one {name} image, the whole encrypted network (server side)"}


def _hbm_peak():
    hbm_peak = 6549.8
    mp = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(mp):
        hbm_peak = json.load(open(mp)).get("hbm_gbs", hbm_peak)
    return hbm_peak


def _ncu_traffic(kernel, log_n, L, B):
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            return json.load(open(tf)).get(f"{kernel}@{log_n}/{L}/B{B}")
        except (ValueError, OSError):
            return None
    return None


# ------------------------------------------------------------------------------ reference arm (oracle)
def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.ckks import Oracle
    cores = os.cpu_count() or 1
    o = Oracle(a.log_n, [50] * a.limbs, 60, seed=a.seed, nthreads=cores)
    import synth
    k = synth.rot_amount(a.seed, a.log_n, a.limbs)
    o.keygen(rot_amounts=[k], relin=False)
    ct = o.bench_ct(0, a.limbs - 1)
    for _ in range(a.warmup):
        o.rot_left(ct, k)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        o.rot_left(ct, k)
    dt = time.perf_counter() - t0
    v = a.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": dt * 1e3 / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic", "config": {**workload(a), "batch_per_gpu": 1,
                                                                                  "k": k},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": "1 top-level rotation of 1 ciphertext per step (oracle/ckks_oracle.c, "
                                       "OpenMP over limbs)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(a, k):
    """The oracle (never tuned) rotating one top-level ciphertext on all host cores, and the same
    on one thread (nproc, the CPU model and a single-thread number)."""
    from oracle.ckks import Oracle
    cores = os.cpu_count() or 1
    o = Oracle(a.log_n, [50] * a.limbs, 60, seed=a.seed, nthreads=cores)
    o.keygen(rot_amounts=[k], relin=False)
    ct = o.bench_ct(0, a.limbs - 1)
    t0 = time.perf_counter()
    o.rot_left(ct, k)
    dt = time.perf_counter() - t0
    o1 = Oracle(a.log_n, [50] * a.limbs, 60, seed=a.seed, nthreads=1)
    o1.rot_keys, o1.s_int, o1.s_ntt, o1.pk = o.rot_keys, o.s_int, o.s_ntt, o.pk
    t0 = time.perf_counter()
    o1.rot_left(ct, k)
    dt1 = time.perf_counter() - t0
    return {"value": 1.0 / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "single_thread": {"value": 1.0 / dt1, "unit": UNIT, "cores": 1},
            "sample": f"1 top-level rotation of 1 ciphertext (N=2^{a.log_n}, L={a.limbs}), "
                      f"keygen excluded, {dt:.1f} s on {cores} threads, {dt1:.1f} s on 1"}


# ------------------------------------------------------------------------------ GPU arm
def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    import torch
    import synth
    from paper_1810_00845_b200 import hisa as H

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("HISA_BENCH_SHARED_DEVICE"):   # emulation on one GPU (tests only)
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        import datetime
        # bounded collectives: a failing sharded-inference run must not hang the whole bench
        backend = os.environ.get("HISA_BENCH_BACKEND", "nccl")   # gloo: one-GPU emulation (tests only)
        # communicator setup (rings / trees / NVLS) logged to stderr for the scaling runs
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group(backend, device_id=torch.device(f"cuda:{local}") if backend == "nccl" else None,
                                timeout=datetime.timedelta(seconds=300))
    B, L, log_n = a.batch, a.limbs, a.log_n
    N = 1 << log_n
    k = synth.rot_amount(a.seed, log_n, L)
    arena = int(float(os.environ["HISA_BENCH_ARENA_GB"]) * (1 << 30)) if os.environ.get("HISA_BENCH_ARENA_GB") else None
    ctx = H.Context(log_n, [50] * L, 60, seed=a.seed, device=local, arena_bytes=arena)
    ctx.keygen([k], False)
    cts = [ctx.ct_random(rank * B + b, L - 1) for b in range(B)]
    ctx.sync()
    stream = torch.cuda.current_stream(local)

    def step():
        outs = ctx.rot_left_batch(cts, k)
        for h in outs:
            ctx.free(h)

    for _ in range(a.warmup):
        step()
    ctx.sync()
    ctx.profile(True)
    clocks = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(a.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ck = clocks.stop()
    if dist:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count()
    prof = ctx.profile_read()
    ctx.profile(False)
    ms_max = ms
    if dist:
        t = torch.tensor([ms], device=f"cuda:{local}")
        _allreduce_max(t)
        ms_max = float(t.item())
    value = world * B * a.steps / (ms_max / 1e3)

    # roofline of the dominant kernel (ALU bound): its butterflies run the
    # FP64-pipe engine for the 50-bit q_i (24 of 25 moduli) -> the denominator is the measured
    # FP64 butterfly peak, the faster of the two engines (the int-engine peak is reported beside it)
    peak_int = ctx.microbench_butterfly(2000)
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    sm_ghz = (ck.get("sm_mhz") or 1965.0) / 1e3
    peak_bfly = max(ctx.microbench_butterfly_f64(2000), peak_int)
    dom = max(prof.items(), key=lambda kv: kv[1][0]) if prof else ("none", (0.0, 0))
    dom_name, (dom_ms, dom_n) = dom
    units = kernel_units(dom_name, log_n, L, B) * a.steps
    achieved = units / (dom_ms / 1e3) if dom_ms > 0 else 0.0
    traffic = _ncu_traffic(dom_name, log_n, L, B)
    hbm_peak = _hbm_peak()
    alg_bytes_step = rotation_alg_bytes(log_n, L, B)
    hbm_gbs = alg_bytes_step * a.steps / (ms / 1e3) / 1e9
    total_ms = sum(v[0] for v in prof.values()) or 1.0
    peak_mac = ctx.microbench_mac(2000)
    macs = kernel_macs(dom_name, log_n, L, B) * a.steps
    mac_rate = macs / (dom_ms / 1e3) if dom_ms > 0 else 0.0
    roofline = {"bound": "alu", "kernel": dom_name, "achieved": achieved / 1e9, "peak": peak_bfly / 1e9,
                "unit": "Gbutterfly/s", "frac": achieved / peak_bfly if peak_bfly else None, "traffic": traffic,
                "counts": "butterflies only; the key MACs of the same kernel (on the FP64 pipe since round 2, "
                          "K4 v6) are in 'macs' and both together in 'fp64_pipe'",
                "macs": {"achieved": mac_rate / 1e9, "unit": "GMAC/s",
                         "peak_fp64": peak_bfly * 9.5 / 8.0 / 1e9,
                         "frac_fp64": mac_rate / (peak_bfly * 9.5 / 8.0) if peak_bfly and macs else None,
                         "peak_int_split_mac": peak_mac / 1e9,
                         "model": "one FP64 MAC = u2d of the key word + exact mulred (6) + add = 8 FP64 ops; "
                                  "peak_int_split_mac = hisa_microbench_mac (the round-1 integer MAC, 4 IMAD.WIDE.U32)"},
                "fp64_pipe": {"model_ops": units * 9.5 + macs * 8.0,
                              "achieved": (units * 9.5 + macs * 8.0) / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else None,
                              "peak": peak_bfly * 9.5 / 1e12, "unit": "T FP64 op/s",
                              "frac": (units * 9.5 + macs * 8.0) / (dom_ms / 1e3) / (peak_bfly * 9.5)
                              if dom_ms > 0 and peak_bfly else None,
                              "note": "K4's modeled FP64 work (9.5 ops per butterfly, 8 per key MAC) against the "
                                      "measured FP64 rate of the butterfly microbenchmark"},
                "peak_source": "measured: hisa_microbench_butterfly_f64 (register-resident exact FP64 butterflies, "
                               "all SMs; the faster engine)", "peak_int_engine": peak_int / 1e9,
                "peak_derived": {"fp64_engine": sm_count * 64 * sm_ghz / 9.5,
                                 "int_engine": sm_count * 64 * sm_ghz / 20.0, "unit": "Gbutterfly/s",
                                 "model": "148 SMs x 64 lanes/clk (FP64 pipe; IMAD on the fma pipe) x SM clock "
                                          "/ 9.5 FP64 ops (lazy schedule, ntt_f64.cuh) or ~20 IMAD per butterfly (DESIGN.md 5)"},
                "launch_ms_avg": dom_ms / max(dom_n, 1), "share_of_step": dom_ms / total_ms,
                "rotation_hbm": {"alg_bytes_per_step": alg_bytes_step, "achieved_gbs": hbm_gbs,
                                 "peak_gbs": hbm_peak, "frac": hbm_gbs / hbm_peak,
                                 "peak_source": "MEASURED_PEAKS.json hbm_gbs"}}
    kernels = {n: {"ms": v[0], "launches": v[1], "share": v[0] / total_ms,
                   "gbutterfly_s": kernel_units(n, log_n, L, B) * a.steps / (v[0] / 1e3) / 1e9 if v[0] else None}
               for n, v in sorted(prof.items(), key=lambda kv: -kv[1][0])}

    # end-to-end through the C-ABI with pinned host buffers: every step copies its B input
    # ciphertexts host -> device and its B results device -> host.  Pipelined over three streams
    # (PyTorch streams / events as plumbing): the H2D of step i+1 and the D2H of step i-1 run
    # while step i key-switches; hisa_ct_adopt_device / hisa_ct_device_view move the words
    # between the torch staging tensors and libhisa's arena (device-to-device, ~50 us per step).
    e2e = None
    if not a.no_e2e:
        words = 2 * L * N
        host_in = [torch.empty(words, dtype=torch.int64, pin_memory=True) for _ in range(B)]
        for b in range(B):
            host_in[b].numpy().view("uint64")[:] = ctx.ct_export(cts[b]).ravel()
        host_out = [torch.empty(words, dtype=torch.int64, pin_memory=True) for _ in range(B)]
        dev = torch.device(f"cuda:{local}")
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        din = [[torch.empty(words, dtype=torch.int64, device=dev) for _ in range(B)] for _ in range(2)]
        dout = [[torch.empty(words, dtype=torch.int64, device=dev) for _ in range(B)] for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]      # H2D of slot done
        ev_used = [torch.cuda.Event() for _ in range(2)]    # compute finished reading din[slot]
        ev_res = [torch.cuda.Event() for _ in range(2)]     # results of slot staged in dout
        ev_out = [torch.cuda.Event() for _ in range(2)]     # D2H of slot done
        for e in ev_used + ev_out:
            e.record(stream)
        from paper_1810_00845_b200.parallel import _DevArray

        def e2e_step(i):
            sl = i % 2
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_used[sl])
                for b in range(B):
                    din[sl][b].copy_(host_in[b], non_blocking=True)
                ev_in[sl].record(s_in)
            stream.wait_event(ev_in[sl])
            ins = [ctx.ct_adopt_device(din[sl][b].data_ptr(), L - 1, 2, 2.0 ** 40) for b in range(B)]
            ev_used[sl].record(stream)
            outs = ctx.rot_left_batch(ins, k)
            stream.wait_event(ev_out[sl])
            for b, h in enumerate(outs):
                ptr, w = ctx.ct_device_view(h)
                dout[sl][b].copy_(torch.as_tensor(_DevArray(ptr, w), device=dev))
            ev_res[sl].record(stream)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_res[sl])
                for b in range(B):
                    host_out[b].copy_(dout[sl][b], non_blocking=True)
                ev_out[sl].record(s_out)
            for h in outs + ins:
                ctx.free(h)

        for i in range(2):
            e2e_step(i)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        n_e2e = max(4, a.steps)
        t0 = time.perf_counter()
        for i in range(n_e2e):
            e2e_step(i)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        # the results that reached the host are the rotation's (checked against a direct call)
        ref = ctx.rot_left_batch(cts[:1], k)[0]
        e2e_ok = bool((host_out[0].numpy().view("uint64") == ctx.ct_export(ref).ravel()).all())
        ctx.free(ref)
        if dist:
            t = torch.tensor([dt], device=f"cuda:{local}", dtype=torch.float64)
            _allreduce_max(t)
            dt = float(t.item())
        e2e = {"value": world * B * n_e2e / dt, "unit": UNIT, "h2d_bytes_per_step": B * words * 8,
               "d2h_bytes_per_step": B * words * 8, "steps": n_e2e,
               "pipeline": "3 streams: H2D(i+1) || key switch(i) || D2H(i-1), pinned host buffers",
               "api": "torch pinned-memory copies + hisa_ct_adopt_device -> hisa_rot_left_batch -> "
                      "hisa_ct_device_view (zero-copy hand-over); NOT the C-ABI's host-buffer calls "
                      "hisa_ct_import / hisa_ct_export, which are synchronous and would serialise the copies",
               "result_check": e2e_ok}

    hoisted = None
    if not a.no_hoisted:
        import synth as _s
        rng = _s.rng(a.seed, 11, log_n, L)
        amounts = sorted({int(x) for x in rng.integers(1, N // 2, size=a.hoist_r)})
        amounts24 = sorted({int(x) for x in rng.integers(1, N // 2, size=24)})
        ctx.keygen(sorted(set(amounts) | set(amounts24)), False)
        hsteps = max(2, a.steps // 2)
        # the conv pattern: all B ciphertexts x R amounts through the batched call (headline),
        # plus one ciphertext by the 3x3 (8) and 5x5 (24) tap counts
        hoisted = measure_hoisted(ctx, cts, amounts, hsteps, a.warmup, log_n, L, stream, batched=True)
        hoisted["single_ct"] = [measure_hoisted(ctx, cts[:1], am, hsteps, a.warmup, log_n, L, stream, batched=False)
                                for am in (amounts, amounts24)]
        for v in hoisted["single_ct"]:
            v.pop("kernels", None)
        if dist:
            t = torch.tensor([hoisted["ms_per_step"]], device=f"cuda:{local}", dtype=torch.float64)
            _allreduce_max(t)
            hoisted["value"] = world * len(cts) * len(amounts) / (float(t.item()) / 1e3)

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a, k)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u64", "data": "synthetic",
                "config": {**workload(a), "batch_per_gpu": B, "global_batch": B * world, "k": k,
                           "parallelism": f"dp{world} (independent ciphertexts)",
                           "l2": "inputs larger than L2 (600 MiB key + B x 24 MiB ciphertexts per step)"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": ck, "kernels": kernels, "hoisted": hoisted}
    ctx.close()
    ctx = None
    torch.cuda.empty_cache()
    sharded = None
    if world > 1 and not a.no_inference:
        sharded = []
        for nm in [n for n in a.nets.split(",") if n]:
            for part in ("ic", "oc"):
                try:
                    sharded.append(measure_inference_sharded(nm, local, dist, partition=part))
                except Exception as exc:   # the rotation line must survive a failing network run
                    sharded.append({"config": nm, "partition": part, "error": f"{type(exc).__name__}: {exc}"[:300]})
    if rank == 0:
        if sharded is not None:
            line["inference"] = sharded
        if not a.no_inference and world == 1:
            line["inference"] = [measure_inference(nm, local, images=a.images) for nm in a.nets.split(",") if nm]
            for inf in line["inference"]:
                if inf["config"] in PAPER_CPU_S:
                    sec, cite = PAPER_CPU_S[inf["config"]]
                    inf["paper_cpu_context"] = {"latency_s": sec, "cite": cite,
                                                "hardware": "2x Xeon E5-2667v3, 16 threads, non-RNS HEAAN"}
                if not a.no_cpu_baseline and inf["config"] in a.oracle_nets.split(","):
                    inf["cpu_baseline"] = oracle_inference(inf["config"])
            # NEXT-1: the paper's four layout strategies (Fig. tilings) on
            # configs 3 and 4, each a lowering of the same network (variants: 3 images each)
            if a.tiling:
                from synth import nets as SN
                alias = SN.NETS.setdefault("_weights_alias", {})
                line["tiling"] = {"figure": "Fig. tilings, P:883-900 (paper: CPU HEAAN latencies in s, context only)",
                                  "nets": {}}
                for base in [b for b in a.tiling.split(",") if b]:
                    hw = next((i for i in line["inference"] if i["config"] == base), None) or \
                        measure_inference(base, local, images=a.images)
                    variants = {"CHW-fc HW-before": base + "_chwfc", "CHW": base + "_chw_all"}
                    res = {"HW": {"config": base, "latency_s": hw["latency_s"], "rel_err": hw["rel_err"]}}
                    for strat, nm in variants.items():
                        if nm not in SN.NETS:
                            nm = base + "_chwfc"     # no stride-1 conv to CHW-tile: CHW = CHW-fc
                        alias[nm] = base
                        r = measure_inference(nm, local, images=3)
                        res[strat] = {"config": nm, "latency_s": r["latency_s"], "rel_err": r["rel_err"],
                                      "levels_used": r["levels_used"], "rotation_keys": r["rotation_keys"]}
                    res["HW-conv CHW-rest"] = dict(res["CHW-fc HW-before"],
                                                   note="same lowering as CHW-fc HW-before in this build: "
                                                        "activations and pools act per channel either way")
                    line["tiling"]["nets"][base] = res
            # NEXT-3: replicas trade mulPlain for rotations
            if a.replica_sweep:
                line["replica_sweep"] = {"config": a.replica_sweep, "latency_s": {
                    f"R{r}": measure_inference(_net_variant(a.replica_sweep, r), local)["latency_s"]
                    for r in (1, 2, 4, 8)}}
            # NEXT-2: CHET's exact rotation keys vs HEAAN's power-of-two keys with
            # composed rotations (the paper's Fig. rotopt: 1.43-2.07x on CPU HEAAN)
            if a.policy_net:
                ex = next((i for i in line["inference"] if i["config"] == a.policy_net), None) or \
                    measure_inference(a.policy_net, local, images=a.images)
                p2 = measure_inference(a.policy_net, local, images=a.images, rot_policy="pow2")
                line["rot_key_policy"] = {"config": a.policy_net, "exact_s": ex["latency_s"], "pow2_s": p2["latency_s"],
                                          "exact_keys": ex["rotation_keys"], "pow2_keys": p2["rotation_keys"],
                                          "speedup_exact_over_pow2": p2["latency_s"] / ex["latency_s"],
                                          "paper_cpu_heaan": "1.43-2.07x (P:902-918), context only"}
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
