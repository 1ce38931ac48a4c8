#!/bin/bash
# Round-2 closing record on the final code: GPU suite, smoke, bench (+stamps), reference arm,
# sweeps, DP legs (graph engine; eager DDP for comparison), PerfModel, ncu launch list + full.
OUT=gpurun_out/final; mkdir -p $OUT
timeout 1800 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 900 python bench.py --out $OUT/bench.json --stamps $OUT/stamps.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
python tools/analyze_stamps.py $OUT/stamps.json > $OUT/stamps_summary.txt 2>&1
timeout 300 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --sweep --out $OUT/sweep_n7.jsonl > $OUT/sweep_n7.log 2>&1; echo "sweep7 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --sweep --ranks-per-gpu 2 --out $OUT/sweep_n2.jsonl > $OUT/sweep_n2.log 2>&1; echo "sweep2 rc=$?" >> $OUT/log.txt
for op in reduce_scatter allgather broadcast; do
  timeout 500 python bench.py --sweep --sweep-op $op --out $OUT/sweep_${op}_n7.jsonl > $OUT/sweep_$op.log 2>&1; echo "sweep $op rc=$?" >> $OUT/log.txt
done
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --train-no-sync --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
timeout 400 python bench.py --train-only --train-model resnet50 --compress bf16 --out $OUT/train_resnet50_bf16.json > $OUT/train_r50b.log 2>&1; echo "train r50 bf16 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --train-engine ddp --bucket-mb 8 --out $OUT/train_resnet50_ddp.json > $OUT/train_r50ddp.log 2>&1; echo "train r50 ddp rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --ranks-per-gpu 1 --train-mode full --batch 224 --out $OUT/train_resnet50_full.json > $OUT/train_r50full.log 2>&1; echo "train r50 full rc=$?" >> $OUT/log.txt
python tools/calibrate_perfmodel.py $OUT/perfmodel_b200.json $OUT/train_resnet50.json $OUT/train_resnet50_full.json >> $OUT/log.txt 2>&1
timeout 400 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-train --mode green > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/log.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $OUT/reduce_full python tools/reduce_once.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/log.txt
python tools/ncu_summary.py $OUT/launches.csv $OUT/reduce_full.ncu-rep > $OUT/ncu_summary.json 2>> $OUT/log.txt
tail -n 2 $OUT/pytest_gpu.log > $OUT/pytest_gpu_tail.txt
cat $OUT/log.txt
