#!/bin/bash
# Round profiling bundle (run on the GPU box from the repo root): bench, per-config step profile,
# launch list of the timed region, ncu --set full captures of the top kernels.  Outputs in gpurun_out/.
set -x
O=gpurun_out
timeout 600 python bench.py > $O/bench_full.json 2> $O/bench_full.err
timeout 900 python tools/config_profile.py cfg1 cfg2 cfg3 cfg4 cfg5 --steps 20 > $O/cfgprof_all.log 2>&1
B="python bench.py --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_cfg2.csv $B > $O/ncu_launch.log 2>&1
F="ncu --nvtx --nvtx-include timed/ --set full --import-source on --clock-control none -c 1 -s 20"
timeout 600 $F -k regex:k_fused_first_pass -o $O/prof_fused -f $B > $O/ncu_fused.log 2>&1
timeout 600 $F -k regex:k_dense_pass_mma -o $O/prof_pass -f $B > $O/ncu_pass.log 2>&1
G="ncu --set full --import-source on --clock-control none -c 1 -s 200"
timeout 900 $G -k regex:k_csr_apply -o $O/prof_csr -f python tools/config_profile.py cfg3 --steps 3 > $O/ncu_csr.log 2>&1
timeout 900 $G -k regex:k_coop_orth -o $O/prof_orth -f python tools/config_profile.py cfg4 --steps 3 > $O/ncu_orth.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -c 1 -s 2 -k regex:k_rr_wide -o $O/prof_rrwide -f python tools/config_profile.py cfg4 --steps 3 > $O/ncu_rrwide.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -c 1 -s 30 -k regex:k_dense_pass_umma -o $O/prof_umma -f python tools/config_profile.py cfg5 --steps 3 > $O/ncu_umma.log 2>&1
timeout 600 python tools/qm_bench.py > $O/qm_bench.log 2>&1
ls -la $O
