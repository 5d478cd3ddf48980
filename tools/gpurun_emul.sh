mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_bench_emulated.py -x -q > gpurun_out/bench_emul.log 2>&1; echo "rc=$?" >> gpurun_out/bench_emul.log
