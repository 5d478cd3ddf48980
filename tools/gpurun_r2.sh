set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "k4_batch or full_size or rotation or extreme" > gpurun_out/t5.log 2>&1; echo "rc=$?" >> gpurun_out/t5.log
timeout 300 python bench.py --no-inference --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/b5.json 2> gpurun_out/b5.err
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_ks_ip6 -c 1 -o gpurun_out/k4_v6c python tools/prof_ks.py > gpurun_out/ncu_k6c.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_fwd_cols_r16 -c 1 -o gpurun_out/modup_v1 python tools/prof_ks.py > gpurun_out/ncu_modup.log 2>&1
