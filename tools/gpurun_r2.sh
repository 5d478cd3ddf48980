set -x
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:"k_elem|k_mulplain" -c 4 -o gpurun_out/elem_v1 python tools/prof_elem.py > gpurun_out/ncu_elem.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_ks_ip_hoisted_f64 -c 1 -o gpurun_out/k7_v2 python tools/prof_hoisted.py > gpurun_out/ncu_k7.log 2>&1
timeout 1200 python tools/sweep_config2.py --out gpurun_out/config2_sweep.jsonl > gpurun_out/sweep.log 2>&1
bash tools/sanitize.sh memcheck
