#!/bin/bash
# Round-1 final record: GPU suite, smoke, default bench + stamps, reference arm, sweeps, DP legs, ncu.
OUT=gpurun_out/r3f; mkdir -p $OUT
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench.json --stamps $OUT/stamps.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --sweep --out $OUT/sweep_n7.jsonl > $OUT/sweep_n7.log 2>&1; echo "sweep7 rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --sweep --ranks-per-gpu 2 --out $OUT/sweep_n2.jsonl > $OUT/sweep_n2.log 2>&1; echo "sweep2 rc=$?" >> $OUT/log.txt
for op in reduce_scatter allgather broadcast; do
  timeout 400 python bench.py --sweep --sweep-op $op --out $OUT/sweep_${op}_n7.jsonl > $OUT/sweep_$op.log 2>&1; echo "sweep $op rc=$?" >> $OUT/log.txt
done
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --train-no-sync --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-train --mode green > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/log.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $OUT/reduce_full python tools/reduce_once.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/log.txt
