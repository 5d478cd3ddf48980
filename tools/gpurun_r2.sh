set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_driver.py -x -q -m "gpu and not slow" > gpurun_out/t8.log 2>&1; echo "rc=$?" >> gpurun_out/t8.log
timeout 400 python bench.py --no-inference --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/b8.json 2> gpurun_out/b8.err
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_modup_cols16 -c 1 -o gpurun_out/modup_v4 python tools/prof_ks.py > gpurun_out/ncu_modup4.log 2>&1
