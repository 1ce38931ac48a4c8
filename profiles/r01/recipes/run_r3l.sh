#!/bin/bash
OUT=gpurun_out/r3l; mkdir -p $OUT
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train --ranks-per-gpu 2 --out $OUT/bench_n2.json > $OUT/bench_n2.log 2>&1; echo "n2 rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --ranks-per-gpu 2 --out $OUT/sweep_n2.jsonl > $OUT/sweep_n2.log 2>&1; echo "sweep n2 rc=$?" >> $OUT/log.txt
timeout 900 python -m pytest tests/test_allreduce_gpu.py -x -q -k "two_ranks or host_buffer or join" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
