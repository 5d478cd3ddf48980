set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t10.log 2>&1; echo "rc=$?" >> gpurun_out/t10.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1
timeout 900 python bench.py > gpurun_out/b10.json 2> gpurun_out/b10.err
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_fwd_rows_r16 -c 1 -o gpurun_out/mdrows_v1 python tools/prof_ks.py > gpurun_out/ncu_mdrows.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_ks_ip_hoisted_f64 -c 1 -o gpurun_out/k7_v2 python tools/prof_hoisted.py > gpurun_out/ncu_k7.log 2>&1
