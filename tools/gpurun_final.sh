# round-end sequence on one box: default bench, torchrun N=1 launch mode, ncu launch list of the bench
mkdir -p gpurun_out
( time timeout 900 python bench.py ) > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-inference --no-e2e --no-cpu-baseline --no-hoisted > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
