#!/bin/bash
# Code check after the reduce-kernel load restructure: GPU suite, smoke (plain and under ncu),
# the default bench line, the reference arm; the reduce kernel timed alone (whole GPU / 1g green
# partition, zero-copy result / HBM only) and its ncu launch list + full captures.
OUT=gpurun_out/final4; mkdir -p $OUT
timeout 1800 python -m pytest tests -x -q -m gpu --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $OUT/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $OUT/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $OUT/log.txt
timeout 900 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
for g in 0 1; do for h in 0 1; do
  FMX_TIME=1 FMX_GREEN=$g FMX_NO_HOST=$h timeout 120 python tools/reduce_once.py >> $OUT/reduce_time.txt 2>&1
done; done
timeout 400 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-train --mode green > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/log.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $OUT/reduce_full python tools/reduce_once.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/log.txt
FMX_GREEN=1 FMX_NO_HOST=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $OUT/reduce_full_green_hbm python tools/reduce_once.py > $OUT/ncu_full_green.log 2>&1; echo "ncu full green rc=$?" >> $OUT/log.txt
python tools/ncu_summary.py $OUT/launches.csv $OUT/reduce_full.ncu-rep $OUT/reduce_full_green_hbm.ncu-rep > $OUT/ncu_summary.json 2> $OUT/ncu_summary.err
tail -n 2 $OUT/pytest_gpu.log > $OUT/pytest_gpu_tail.txt
python -c "
import json; d=json.loads(open('$OUT/bench.json').read().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), round(d['resnet50']['img_s']), d['resnet50']['replicas_agree'], d['clocks'])" >> $OUT/log.txt
cat $OUT/log.txt $OUT/pytest_gpu_tail.txt $OUT/reduce_time.txt
