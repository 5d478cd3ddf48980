mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_edges.py -x -q -k "all_plane_counts" > gpurun_out/one_test.log 2>&1; echo "rc=$?" >> gpurun_out/one_test.log
