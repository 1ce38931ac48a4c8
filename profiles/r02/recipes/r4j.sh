# reduce-kernel grid cap vs its live (contended) store share and the allreduce
set -x
O=gpurun_out/r4j; mkdir -p $O
for rep in 1 2; do for c in 1184 64 32 16 8; do
FMX_REDUCE_CTAS=$c timeout 300 python bench.py --no-train --no-cpu-baseline --no-e2e --steps 20 --warmup 5 --out $O/bench_c$c.json > /dev/null 2>&1
python -c "
import json; d=json.loads(open('$O/bench_c$c.json').read().splitlines()[-1])
print('ctas=$c', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), round(d['roofline']['launch_us'],1), round(d['roofline']['isolated']['launch_us'],1))"
done; done
