#!/bin/bash
# Round-end refresh: GPU tests, smoke, every bench config (one JSON line each) into gpurun_out/.
mkdir -p gpurun_out/bench
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/bench/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/bench/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bench/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/bench/smoke.log
for cfg in ${CONFIGS:-c2 c1 c3 c4 c4poly c4jac c4gs2 c4prod c4ortho c5}; do
  timeout 900 python bench.py --config $cfg --steps 20 --warmup 5 > gpurun_out/bench/bench_$cfg.log 2>&1
done
timeout 900 python bench.py --config c3 --mode fast --steps 20 --warmup 5 > gpurun_out/bench/bench_c3fast.log 2>&1
