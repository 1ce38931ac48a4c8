# slice size vs the device path and the host path (e2e)
set -x
O=gpurun_out/r3i; mkdir -p $O
for sb in 2097152 3145728 4194304 8388608 16777216; do   # (run as two batches, summary.txt)
timeout 600 python bench.py --no-train --no-cpu-baseline --steps 20 --warmup 5 --slice-bytes $sb --out $O/bench_$sb.json > /dev/null 2>&1
python -c "
import json; d=json.loads(open('$O/bench_$sb.json').read().splitlines()[-1])
print('slice=$sb', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), d['e2e'].get('roofline', {}).get('frac') if isinstance(d['e2e'].get('roofline'), dict) else '')"
done
