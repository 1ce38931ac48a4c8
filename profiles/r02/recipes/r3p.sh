# FMX_STAGE_ZC: stage D2H by the SM copy kernel, fetch/gather by copy engines - device path A/B
set -x
O=gpurun_out/r3p; mkdir -p $O
for v in 0 1 0 1 0 1; do
FMX_STAGE_ZC=$v timeout 600 python bench.py --no-train --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --out $O/bench_szc$v.json > $O/bench_szc$v.log 2>&1
python -c "
import json; d=json.loads(open('$O/bench_szc$v.json').read().splitlines()[-1])
print('szc=$v', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), round(d['roofline']['launch_us'],1))"
done
tail -n 2 $O/bench_szc1.log | cut -c1-300
