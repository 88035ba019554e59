#!/bin/bash
# ncu evidence for the configs whose kernels changed: launch lists (time + DRAM) of bench.py's timed
# region and one --set full capture of the dominant kernel.
mkdir -p gpurun_out/prof
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none --nvtx --nvtx-include "mpk_timed/" --csv --log-file gpurun_out/prof/c3_launches.csv python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/c3_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_long_rows_bitwise --launch-skip 3 --launch-count 1 -o gpurun_out/prof/c3_long_full python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/c3_f.log 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:"k_dots|k_update|k_tsqr|k_accum|k_sign" --csv --log-file gpurun_out/prof/c4ortho_launches.csv python bench.py --config c4ortho --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/o_l.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_update_dots|k_tsqr_factor" --launch-skip 2 --launch-count 2 -o gpurun_out/prof/c4ortho_full python bench.py --config c4ortho --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/prof/o_f.log 2>&1
