# one GPU call: ncu --set full captures (one kernel each) of K4 (FP64 rows), ModUp pass 1, and the
# HBM-bound elementwise kernels; reports under gpurun_out/ (read back with tools/ncu_brief.py)
mkdir -p gpurun_out
T=${TAG:-v1}
NCU="ncu --set full --import-source on --clock-control none --profile-from-start off"
timeout 600 $NCU -k regex:k_ks_ip6 -c 1 -o gpurun_out/k4_$T python tools/prof_ks.py > gpurun_out/ncu_k4_$T.log 2>&1
timeout 600 $NCU -k regex:k_modup_cols16 -c 1 -o gpurun_out/modup_$T python tools/prof_ks.py > gpurun_out/ncu_modup_$T.log 2>&1
if [ -n "$ELEM" ]; then
timeout 600 $NCU -k regex:'k_elem|k_mulplain' -c 8 -o gpurun_out/elem_$T python tools/prof_elem.py > gpurun_out/ncu_elem_$T.log 2>&1
fi
