#!/bin/bash
# Round-2 closing record, second pass after the two-ranks-per-GPU schedule change: GPU suite,
# smoke (plain and under ncu), the default bench line, a timeline run, reference arm, sweeps,
# DP legs, PerfModel.  ncu captures of the (unchanged) kernels: profiles/r02/final, r2y.
OUT=gpurun_out/final2; mkdir -p $OUT
timeout 1800 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $OUT/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $OUT/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $OUT/log.txt
timeout 900 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --no-train --no-cpu-baseline --steps 5 --warmup 2 --stamps $OUT/stamps.json --out $OUT/bench_stamps.json > $OUT/bench_stamps.log 2>&1; echo "bench stamps rc=$?" >> $OUT/log.txt
python tools/analyze_stamps.py $OUT/stamps.json > $OUT/stamps_summary.txt 2>&1
timeout 300 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --sweep --out $OUT/sweep_n7.jsonl > $OUT/sweep_n7.log 2>&1; echo "sweep7 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --sweep --ranks-per-gpu 2 --out $OUT/sweep_n2.jsonl > $OUT/sweep_n2.log 2>&1; echo "sweep2 rc=$?" >> $OUT/log.txt
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --train-no-sync --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
timeout 400 python bench.py --train-only --train-model resnet50 --compress bf16 --out $OUT/train_resnet50_bf16.json > $OUT/train_r50b.log 2>&1; echo "train r50 bf16 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --train-engine ddp --bucket-mb 8 --out $OUT/train_resnet50_ddp.json > $OUT/train_r50ddp.log 2>&1; echo "train r50 ddp rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --ranks-per-gpu 1 --train-mode full --batch 224 --out $OUT/train_resnet50_full.json > $OUT/train_r50full.log 2>&1; echo "train r50 full rc=$?" >> $OUT/log.txt
python tools/calibrate_perfmodel.py $OUT/perfmodel_b200.json $OUT/train_resnet50.json $OUT/train_resnet50_full.json >> $OUT/log.txt 2>&1
tail -n 2 $OUT/pytest_gpu.log > $OUT/pytest_gpu_tail.txt
cat $OUT/log.txt
