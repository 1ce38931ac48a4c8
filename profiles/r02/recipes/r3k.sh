# FMX_STAGE_AFTER_REDUCE: stage(R+1) after this rank's reduce(R) - device path A/B
set -x
O=gpurun_out/r3k; mkdir -p $O
for v in 0 1 0 1 0 1; do
FMX_STAGE_AFTER_REDUCE=$v timeout 600 python bench.py --no-train --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --out $O/bench_sar$v.json > /dev/null 2>&1
python -c "
import json; d=json.loads(open('$O/bench_sar$v.json').read().splitlines()[-1])
print('sar=$v', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), round(d['roofline']['launch_us'],1))"
done
FMX_STAGE_AFTER_REDUCE=1 timeout 600 python bench.py --no-train --no-cpu-baseline --no-e2e --steps 10 --warmup 3 --stamps $O/stamps_sar1.json --out $O/bench_stamps.json > /dev/null 2>&1
python tools/analyze_stamps.py $O/stamps_sar1.json > $O/stamps_sar1.txt 2>&1; head -8 $O/stamps_sar1.txt
