#!/bin/bash
# Round-2 (final) profiling bundle (GPU box, repo root): default bench line, ncu launch lists of the cfg2 and
# cfg3 timed loops, ncu --set full captures of the top kernels.  Outputs in gpurun_out/r02b/.
O=gpurun_out/r02b
mkdir -p $O
timeout 1200 python bench.py > $O/bench_default.json 2> $O/bench_default.err
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
C3="python bench.py --workload cfg3 --steps 3 --warmup 3 --workloads none --no-cpu-baseline"
timeout 600 $C3 > $O/plain3.log 2>&1 && \
timeout 900 ncu --nvtx --nvtx-include "timed_cfg3/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches_cfg3.csv $C3 > $O/ncu_launch3.log 2>&1
G="ncu --nvtx --nvtx-include timed_cfg3/ --set full --import-source on --clock-control none -c 1 -s 20"
timeout 900 $G -k regex:k_csr_apply_panel -o $O/prof_csr -f $C3 > $O/ncu_csr.log 2>&1
timeout 900 $G -k regex:k_coop_orth -o $O/prof_orth -f $C3 > $O/ncu_orth.log 2>&1
timeout 900 $G -k regex:k_rr_wide -o $O/prof_rrwide -f $C3 > $O/ncu_rrwide.log 2>&1
# summaries on the box (the .ncu-rep files exceed the 64 MiB that travels back)
for k in pass fused umma csr orth rrwide; do
  [ -f $O/prof_$k.ncu-rep ] && python tools/summarize_ncu.py $O/prof_$k.ncu-rep $O/ncu_$k.md && \
    (ncu -i $O/prof_$k.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | python tools/source_hotspots.py 15 > $O/hotspots_$k.txt 2>&1 || true)
done
python tools/launch_summary.py $O/launches_cfg2.csv > $O/launches_cfg2_summary.txt 2>&1
python tools/launch_summary.py $O/launches_cfg3.csv > $O/launches_cfg3_summary.txt 2>&1
rm -f $O/*.ncu-rep
gzip -f $O/launches_cfg3.csv
ls -la $O
