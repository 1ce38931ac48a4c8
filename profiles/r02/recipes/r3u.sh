# two ranks per GPU: fetch lane + result slot by copy engine from 8 rounds (default) vs off;
# parity with the copy-engine result path forced on every round
set -x
O=gpurun_out/r3u; mkdir -p $O
FMX_RCE_ROUNDS=1 timeout 900 python -m pytest tests/test_allreduce_gpu.py tests/test_configs_gpu.py -m gpu -x -q > $O/pytest_rce1.log 2>&1; echo rc=$? >> $O/pytest_rce1.log
for v in 8 1000 8 1000; do
  FMX_RCE_ROUNDS=$v timeout 400 python bench.py --sweep --ranks-per-gpu 2 --sweep-max 1073741824 --out $O/sweep_n2_rce$v.jsonl > /dev/null 2>&1
  python -c "
import json
print('rce_rounds=$v', [(x['bytes']>>20, round(x['ms'],3), round(x.get('step_roofline_frac') or 0,3)) for x in map(json.loads, open('$O/sweep_n2_rce$v.jsonl')) if x['bytes'] >= 1<<24])"
done
tail -n 2 $O/pytest_rce1.log
