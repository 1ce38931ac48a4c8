#!/bin/bash
OUT=gpurun_out/r1f; mkdir -p $OUT
timeout 500 python -m pytest tests/test_reduce_kernel_gpu.py -x -q --timeout 200 > $OUT/kerneltest.log 2>&1; echo "kerneltest rc=$?" >> $OUT/log.txt
for cfg in "fine 2 4194304" "coarse 2 4194304" "coarse 1 4194304" "fine 1 4194304" "coarse 1 8388608" "coarse 2 8388608" "fine 2 8388608"; do
  set -- $cfg
  tag=$1-$2-$3
  FMX_GRAIN=$1 FMX_LANES=$2 timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-train --slice-bytes $3 --timeline $OUT/tl_$tag.json --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt
done
