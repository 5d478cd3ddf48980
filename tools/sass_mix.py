"""Aggregate an ncu source page (--page source --csv --print-source sass) by opcode: executed
warp instructions, stall samples and shared-memory excess wavefronts per opcode."""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
agg = defaultdict(lambda: [0, 0, 0])
tot = [0, 0, 0]
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", src)
    if not m:
        continue
    op = m.group(2)
    if len(sys.argv) < 3:
        op = op.split(".")[0]
    ex = int(r[ix["Instructions Executed"]] or 0)
    st = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    bx = int(r[ix["L1 Wavefronts Shared Excessive"]] or 0)
    a = agg[op]
    a[0] += ex; a[1] += st; a[2] += bx
    tot[0] += ex; tot[1] += st; tot[2] += bx
print(f"{'opcode':24s} {'warp inst':>14s} {'share':>7s} {'stall smp':>10s} {'share':>7s} {'smem excess wf':>15s}")
for op, (ex, st, bx) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{op:24s} {ex:14d} {ex / tot[0]:7.3f} {st:10d} {st / max(tot[1], 1):7.3f} {bx:15d}")
print(f"{'total':24s} {tot[0]:14d} {'':7s} {tot[1]:10d} {'':7s} {tot[2]:15d}")
