set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t14.log 2>&1; echo "rc=$?" >> gpurun_out/t14.log
timeout 400 python bench.py --no-inference --no-e2e --no-cpu-baseline --steps 5 > gpurun_out/b14.json 2> gpurun_out/b14.err
timeout 600 python bench.py --nets lenet_large,squeezenet --images 5 --no-cpu-baseline --no-e2e --no-hoisted --tiling "" --policy-net "" --steps 2 > gpurun_out/b14inf.json 2> gpurun_out/b14inf.err
timeout 600 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:k_ks_ip_hoisted_f64 -c 1 -o gpurun_out/k7_v3 python tools/prof_hoisted.py > gpurun_out/ncu_k7b.log 2>&1
