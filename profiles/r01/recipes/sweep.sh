#!/bin/bash
# Config sweep of the 7-rank ResNet-50 gradient allreduce + ncu launch list / full capture.
OUT=gpurun_out/sweep; mkdir -p $OUT
for mode in green mps full; do
  for tr in ce zc; do
    for sb in 1048576 4194304; do
      echo "== $mode $tr $sb" >> $OUT/log.txt
      timeout 180 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --mode $mode \
        --transport $tr --slice-bytes $sb --out $OUT/tmp.json >> $OUT/log.txt 2>&1
      echo "rc=$?" >> $OUT/log.txt
      [ -f $OUT/tmp.json ] && python -c "
import json,sys; d=json.load(open('$OUT/tmp.json')); d['sweep']={'mode':'$mode','transport':'$tr','slice':$sb}
print(json.dumps(d))" >> $OUT/sweep.jsonl; rm -f $OUT/tmp.json
    done
  done
done
# ncu launch list over all rank processes (device time per launch, serialized)
timeout 300 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
echo "ncu1 rc=$?" >> $OUT/log.txt
timeout 400 ncu --target-processes all --set full --clock-control none --import-source on -k regex:fmx_reduce -s 4 -c 1 \
  -o $OUT/reduce_prof python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $OUT/ncu_full.log 2>&1
echo "ncu2 rc=$?" >> $OUT/log.txt
