# measurement legs: parity of the changed kernels, per-net kernel profile, ncu of the HBM-bound
# elementwise kernels, config-2 sweep
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_driver.py -x -q > gpurun_out/meas_tests.log 2>&1; echo "rc=$?" >> gpurun_out/meas_tests.log
for n in lenet_large squeezenet; do timeout 600 python tools/prof_net.py $n > gpurun_out/prof_net_$n.txt 2>&1; done
timeout 900 ncu --set full --clock-control none --profile-from-start off -o gpurun_out/elem_r2 -f python tools/prof_elem.py > gpurun_out/ncu_elem.log 2>&1
timeout 1800 python tools/sweep_config2.py > gpurun_out/sweep_config2.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_config2.log
