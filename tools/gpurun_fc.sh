mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_driver.py -x -q -k "accumulate or small_nets or lenet" > gpurun_out/fc_tests.log 2>&1; echo "rc=$?" >> gpurun_out/fc_tests.log
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:k_mulplain -o gpurun_out/fc_r2 -f python tools/prof_elem.py > gpurun_out/ncu_fc.log 2>&1
timeout 600 python tools/prof_net.py lenet_large > gpurun_out/prof_net_lenet_large2.txt 2>&1
