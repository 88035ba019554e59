#!/bin/bash
# Round-2 ncu evidence for the C5 wave schedule: the launch list (time + DRAM bytes) of bench.py's
# timed region and one --set full capture of k_mpk_wave (run only after the same commands exited 0).
mkdir -p gpurun_out/prof
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
CFG=${1:-c5}
timeout 900 ncu --metrics $M --clock-control none --nvtx --nvtx-include "mpk_timed/" --csv \
  --log-file gpurun_out/prof/${CFG}_launches.csv python bench.py --config $CFG --steps 1 --warmup 3 \
  --no-cpu-baseline --no-e2e > gpurun_out/prof/${CFG}_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_mpk_wave --launch-skip 3 \
  --launch-count 1 -o gpurun_out/prof/${CFG}_wave_full python tools/profile_case.py --config $CFG \
  --launches 1 > gpurun_out/prof/${CFG}_f.log 2>&1
