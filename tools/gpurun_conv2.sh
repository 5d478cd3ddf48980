mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k 'regex:k_conv_tc$' -c 1 -o gpurun_out/conv_tc_r2 -f python tools/prof_conv_tc.py 144 64 > gpurun_out/ncu_conv.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k 'regex:k_conv_tc$' -c 1 -o gpurun_out/conv_tc_r2_288 -f python tools/prof_conv_tc.py 288 128 > gpurun_out/ncu_conv288.log 2>&1
timeout 300 python -m pytest tests/test_nccl_world1.py -x -q > gpurun_out/nccl1.log 2>&1; echo "rc=$?" >> gpurun_out/nccl1.log
timeout 600 python bench.py --nets lenet_large,squeezenet --images 3 --no-cpu-baseline --no-e2e --no-hoisted --tiling "" --policy-net "" --steps 2 > gpurun_out/inf_conv2.json 2> gpurun_out/inf_conv2.err
