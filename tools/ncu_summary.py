"""Summarise an ncu --set full report (raw CSV page) into profiles/: per-kernel time, DRAM
traffic, occupancy, pipe utilisation; and the per-launch DRAM bytes bench.py reports as
roofline.traffic (profiles/ncu_traffic.json, keyed kernel@logn/L/B)."""
import csv
import json
import subprocess
import sys

rep, out_txt, key_suffix = sys.argv[1], sys.argv[2], sys.argv[3]   # e.g. 16/24/B8
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
names = {"k_ks_ip_hoisted": "ks_ip_hoisted", "k_ks_ip": "ks_ip_rows", "k_fwd_cols": "fwd_cols", "k_fwd_rows": "fwd_rows",
         "k_inv_rows": "inv_rows", "k_inv_cols": "inv_cols", "k_conv_acc": "conv_acc", "k_mulplain_acc": "mulplain_acc"}
traffic = {}
lines = [f"# ncu --set full --clock-control none summary of {rep}", ""]
for d in data:
    kname = d[ix["Kernel Name"]]
    lines.append(kname[:110])
    for w in want:
        if w in ix:
            lines.append(f"    {w:70s} {d[ix[w]]} {units[ix[w]]}")
    short = next((v for k, v in names.items() if kname.startswith("void hisa::" + k) or k in kname.split("(")[0]), None)
    if short and "dram__bytes_read.sum" in ix:
        def gb(col):
            v = float(d[ix[col]].replace(",", ""))
            u = units[ix[col]]
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic.setdefault(f"{short}@{key_suffix}", gb("dram__bytes_read.sum") + gb("dram__bytes_write.sum"))
open(out_txt, "w").write("\n".join(lines) + "\n")
try:
    old = json.load(open("profiles/ncu_traffic.json"))
except (OSError, ValueError):
    old = {}
old.update(traffic)
json.dump(old, open("profiles/ncu_traffic.json", "w"), indent=1, sort_keys=True)
print(json.dumps(traffic, indent=1))
