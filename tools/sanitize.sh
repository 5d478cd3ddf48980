# compute-sanitizer over the small-parameter GPU parity tests (one tool per call):
#   bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
# Covers every kernel family at N = 2^10 / 2^11 / 2^13 (config 1) -- NTT passes, elementwise,
# key switch K4 (int + FP64 rows), hoisted K7, conv accumulation (tensor cores: mbarrier / TMEM),
# encode / decode, samplers -- plus the driver on the small nets.
tool=${1:-memcheck}
mkdir -p gpurun_out
export HISA_NO_ARENA=1   # per-buffer allocations: memcheck sees every bound
timeout 2400 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "n10 or n11_odd or c1_n13" \
  > gpurun_out/sanitize_${tool}_parity.log 2>&1
echo "parity rc=$?" >> gpurun_out/sanitize_${tool}_parity.log
timeout 1800 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
  python -m pytest tests/test_driver.py -x -q -k "small_nets_bit_exact and (every_branch or chw)" \
  > gpurun_out/sanitize_${tool}_driver.log 2>&1
echo "driver rc=$?" >> gpurun_out/sanitize_${tool}_driver.log
