#!/bin/bash
# Pipeline depth (FMX_SLOTS) x slice size, MPS instances, 7 ranks.
OUT=gpurun_out/r1n; mkdir -p $OUT
timeout 600 python -m pytest tests/test_allreduce_gpu.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
run() { tag=$1; shift; env $ENVS timeout 240 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-e2e --mode mps "$@" --out $OUT/bench_$tag.json > $OUT/bench_$tag.log 2>&1; echo "bench $tag rc=$?" >> $OUT/log.txt; }
for slots in 2 3 4; do
  for sb in 2097152 4194304 8388608; do
    ENVS=FMX_SLOTS=$slots run s$slots-$sb --slice-bytes $sb
  done
done
ENVS=FMX_SLOTS=3 run s3-4M-tl --slice-bytes 4194304 --timeline $OUT/tl_s3.json
ENVS="FMX_SLOTS=3 FMX_RAMP=0" run s3-4M-noramp --slice-bytes 4194304
ENVS="FMX_SLOTS=3 FMX_LANES=2" run s3-4M-l2 --slice-bytes 4194304
