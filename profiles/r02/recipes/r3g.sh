# experiment: the bench's allreduce (device path and host path) captured as a CUDA graph
set -x
O=gpurun_out/r3g; mkdir -p $O
for g in 0 1 0 1; do
FMX_BENCH_GRAPH=$g timeout 600 python bench.py --no-train --no-cpu-baseline --steps 20 --warmup 5 --out $O/bench_g$g.json > $O/bench_g$g.log 2>&1
python -c "
import json; d=json.loads(open('$O/bench_g$g.json').read().splitlines()[-1])
print('graph=$g', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['e2e']['ms_per_step'],3))"
done
tail -n 3 $O/bench_g1.log | cut -c1-300
