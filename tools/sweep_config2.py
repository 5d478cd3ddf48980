"""Config-2 HISA primitive sweep (BASELINE.json configs[1]): N in {2^13, 2^14, 2^15,
2^16} with L = 3 / 8 / 16 / 24 limbs of 50-bit primes (+ a 60-bit special prime, dnum = L), batches
B of 1..256 independent top-level ciphertexts with uniform residues; ops NTT (forward, in place),
INTT, mulPlain, mul + relinearize, rotate by k (A30), rescale.  Each op is timed with CUDA events
on the context stream, L2 flushed (a 512 MiB write) before every timed repetition, median of
`--reps`; reported with its roofline fraction: HBM-bound ops (mulPlain) against the measured HBM
bandwidth on their compulsory bytes, ALU-bound ops (NTT / INTT / rescale / key switching) against
the measured FP64 butterfly peak on their butterflies (SURVEY 8d work model).
Writes one JSON line per (N, L, B, op) to --out and prints a table."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1810_00845_b200 import hisa as H  # noqa: E402

POINTS = [(13, 3), (14, 8), (15, 16), (16, 24)]


def hbm_peak():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        return json.load(open(p)).get("hbm_gbs", 6549.8)
    except OSError:
        return 6549.8


def work(op, log_n, l1, B):
    """(butterflies, compulsory bytes) per call over B ciphertexts at l1 = l + 1 limbs."""
    N = 1 << log_n
    limb = 8 * N
    ntt = (N // 2) * log_n                       # butterflies of one limb NTT
    if op in ("ntt", "intt"):
        return B * 2 * l1 * ntt, B * 2 * l1 * 2 * limb
    if op == "mulplain":
        return 0, B * 5 * l1 * limb
    if op == "rescale":                           # INTT top limb, lift, NTT on l limbs, per poly
        return B * 2 * (1 + (l1 - 1)) * ntt, B * (4 * (l1 - 1) + 2) * limb
    if op in ("rotate", "mul_relin"):             # (l+1) + beta (l+1) + 2 + 2 (l+1) NTTs
        n_ntt = l1 + l1 * l1 + 2 + 2 * l1
        extra = B * 7 * l1 * limb if op == "mul_relin" else 0
        return B * n_ntt * ntt, B * 4 * l1 * limb + 2 * l1 * (l1 + 1) * limb + extra
    raise ValueError(op)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--points", default="13,14,15,16")
    ap.add_argument("--ops", default="ntt,intt,mulplain,mul_relin,rotate,rescale")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-gb", type=float, default=40.0, help="skip (point, B) whose ciphertexts exceed this")
    ap.add_argument("--out", default="gpurun_out/config2_sweep.jsonl")
    a = ap.parse_args()
    dev = torch.device("cuda:0")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    peak_hbm = hbm_peak()
    rows = []
    pts = [p for p in POINTS if str(p[0]) in a.points.split(",")]
    for log_n, L in pts:
        N = 1 << log_n
        ctx = H.Context(log_n, [50] * L, 60, seed=0, arena_bytes=int(100 * (1 << 30)))
        k = synth.rot_amount(0, log_n, L)
        ctx.keygen([k], True)
        peak_bfly = ctx.microbench_butterfly_f64(2000)
        st = torch.cuda.current_stream(dev)
        for B in [int(b) for b in a.batches.split(",")]:
            ct_bytes = 2 * L * N * 8
            if B * ct_bytes * 4 > a.max_gb * (1 << 30):
                continue
            cts = [ctx.ct_random(b, L - 1) for b in range(B)]
            pts_ = [ctx.pt_random(1000 + b, L - 1) for b in range(B)]
            for op in a.ops.split(","):
                def run():
                    outs = []
                    if op == "ntt":
                        ctx.ntt_batch(cts, False)
                    elif op == "intt":
                        ctx.ntt_batch(cts, True)
                    elif op == "mulplain":
                        outs = ctx.mul_plain_batch(cts, pts_)
                    elif op == "mul_relin":
                        outs = ctx.mul_batch(cts, cts)
                    elif op == "rotate":
                        outs = ctx.rot_left_batch(cts, k)
                    elif op == "rescale":
                        outs = ctx.rescale_batch(cts)
                    return outs
                for h in run():   # warm-up
                    ctx.free(h)
                times = []
                for _ in range(a.reps):
                    flush.zero_()
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    outs = run()
                    e1.record(st)
                    torch.cuda.synchronize()
                    times.append(e0.elapsed_time(e1))
                    for h in outs:
                        ctx.free(h)
                ms = float(np.median(times))
                bfly, nbytes = work(op, log_n, L, B)
                row = {"log_n": log_n, "limbs": L, "B": B, "op": op, "ms": ms, "ops_per_s": B / (ms / 1e3),
                       "gbs": nbytes / (ms / 1e3) / 1e9, "hbm_frac": nbytes / (ms / 1e3) / 1e9 / peak_hbm,
                       "gbfly_s": bfly / (ms / 1e3) / 1e9 if bfly else None,
                       "alu_frac": bfly / (ms / 1e3) / peak_bfly if bfly else None,
                       "bound": "hbm" if op == "mulplain" else "alu"}
                rows.append(row)
                print(json.dumps(row), flush=True)
            for h in cts:
                ctx.free(h)
            for p in pts_:
                ctx.free(p)
        ctx.close()
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        for r in rows:
            f.write(json.dumps(r) + "\n")
    print(f"{'N':>6} {'L':>3} {'B':>4} {'op':>10} {'ms':>9} {'ops/s':>10} {'frac':>6} bound")
    for r in rows:
        fr = r["hbm_frac"] if r["bound"] == "hbm" else r["alu_frac"]
        print(f"2^{r['log_n']:<4} {r['limbs']:>3} {r['B']:>4} {r['op']:>10} {r['ms']:9.3f} {r['ops_per_s']:10.0f} "
              f"{fr:6.3f} {r['bound']}")


if __name__ == "__main__":
    main()
