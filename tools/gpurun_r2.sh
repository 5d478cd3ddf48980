set -x
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_driver.py tests/test_abi.py -x -q -m "gpu and not slow" > gpurun_out/t2.log 2>&1; echo "rc=$?" >> gpurun_out/t2.log
timeout 300 python bench.py --no-inference --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/b2.json 2> gpurun_out/b2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_ks_ip5 -c 1 -o gpurun_out/k4_v1 python tools/prof_ks.py > gpurun_out/ncu_k4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_fwd_cols -c 1 -o gpurun_out/cols_v1 python tools/prof_ks.py > gpurun_out/ncu_cols.log 2>&1
