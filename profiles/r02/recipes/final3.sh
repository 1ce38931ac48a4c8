#!/bin/bash
# Final code check (after the fused SGD step and the one-shot / pending-gather fix): GPU suite,
# smoke (plain and under ncu), the default bench line, the reference arm, the two-rank sweep.
OUT=gpurun_out/final3; mkdir -p $OUT
timeout 1800 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $OUT/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $OUT/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $OUT/log.txt
timeout 900 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
tail -n 2 $OUT/pytest_gpu.log > $OUT/pytest_gpu_tail.txt
python -c "
import json; d=json.loads(open('$OUT/bench.json').read().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), round(d['resnet50']['img_s']), d['resnet50']['replicas_agree'], d['clocks'])" >> $OUT/log.txt
cat $OUT/log.txt $OUT/pytest_gpu_tail.txt
