#!/bin/bash
# Experiments: a metrics-only ncu pass over the wave launches of one C5 call (3 launches).
mkdir -p gpurun_out/prof
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:k_mpk_wave --launch-skip 3 --launch-count 3 --csv \
  --log-file gpurun_out/prof/c5_m.csv python tools/profile_case.py --config ${1:-c5} --launches 1 > gpurun_out/prof/c5_m.log 2>&1
python - <<PY
import csv
rows=[r for r in csv.reader(open("gpurun_out/prof/c5_m.csv")) if len(r)>10]
for r in rows[1:]:
    print(r[0], r[-3], r[-2], r[-1])
PY
