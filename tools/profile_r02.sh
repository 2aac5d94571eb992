#!/bin/bash
# Round-2 profiling bundle (GPU box, repo root): the default bench line, the ncu launch list of the
# headline's timed loop, ncu --set full captures of the top kernels.  Outputs in gpurun_out/r02/.
O=gpurun_out/r02
mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
B="python bench.py --steps 60 --warmup 5 --workloads none --no-cpu-baseline"
timeout 600 $B > $O/plain.log 2>&1 && \
timeout 600 ncu --nvtx --nvtx-include "timed_cfg2/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_cfg2.csv $B > $O/ncu_launch.log 2>&1
F="ncu --nvtx --nvtx-include timed_cfg2/ --set full --import-source on --clock-control none -c 1 -s 30"
timeout 600 $F -k regex:k_dense_pass_mma -o $O/prof_pass -f $B > $O/ncu_pass.log 2>&1
timeout 600 $F -k regex:k_fused_first_pass -o $O/prof_fused -f $B > $O/ncu_fused.log 2>&1
C5="python bench.py --workload cfg5 --steps 20 --warmup 10 --workloads none --no-cpu-baseline"
timeout 600 $C5 > $O/plain5.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "timed_cfg5/" --set full --import-source on --clock-control none -c 1 -s 5 \
  -k regex:k_dense_pass_umma -o $O/prof_umma -f $C5 > $O/ncu_umma.log 2>&1
ls -la $O
