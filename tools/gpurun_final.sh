# round-end sequence on one box: full GPU suite, smoke, default bench, torchrun N=1 launch mode,
# config-2 sweep, ncu launch list of the bench
mkdir -p gpurun_out
( time timeout 1800 python -m pytest tests -m gpu -x -q ) > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
( time timeout 900 python bench.py ) > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 3 --warmup 3 --no-inference --no-e2e --no-cpu-baseline --no-hoisted > gpurun_out/bench_torchrun1.json 2> gpurun_out/bench_torchrun1.err
timeout 1800 python tools/sweep_config2.py > gpurun_out/sweep_config2.log 2>&1; echo "rc=$?" >> gpurun_out/sweep_config2.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/ncu_launches.err
