#!/bin/bash
# The reference arm (the reference's own CPU implementation on this box's host cores) for every config.
mkdir -p gpurun_out/ref
for cfg in ${CONFIGS:-c1 c2 c3 c4 c4poly c5 c4jac c4gs2 c4prod c4ortho}; do
  steps=5; [ "$cfg" = c5 ] && steps=3
  timeout 900 python bench.py --impl reference --config $cfg --steps $steps --warmup 1 > gpurun_out/ref/ref_$cfg.log 2>&1
done
