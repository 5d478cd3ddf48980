# K8 iteration: conv parity tests, timing at the SqueezeNet / LeNet shapes, one ncu capture
mkdir -p gpurun_out; rm -f gpurun_out/conv_time.log
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -x -q -k "conv" > gpurun_out/conv_tests.log 2>&1; echo "rc=$?" >> gpurun_out/conv_tests.log
timeout 600 python -m pytest tests/test_driver.py -x -q -k "small_nets_bit_exact" > gpurun_out/conv_driver.log 2>&1; echo "rc=$?" >> gpurun_out/conv_driver.log
for shape in "144 64" "288 128" "27 64" "32 128" "800 64"; do
  timeout 300 python tools/prof_conv_tc.py $shape >> gpurun_out/conv_time.log 2>&1
done
echo "smem 221184:" >> gpurun_out/conv_time.log
for shape in "288 128" "800 64"; do
  HISA_CONV_TC_SMEM=221184 timeout 300 python tools/prof_conv_tc.py $shape >> gpurun_out/conv_time.log 2>&1
done
if grep -q "rc=0" gpurun_out/conv_tests.log; then
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k 'regex:k_conv_tc$' -c 2 -o gpurun_out/conv_tc_r2d -f python tools/prof_conv_tc.py 144 64 > gpurun_out/ncu_conv.log 2>&1
fi
