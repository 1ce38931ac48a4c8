# FMX_FETCH_LANE: the next round's fetch on the gather lane (double-buffered scratch) - A/B
set -x
O=gpurun_out/r3r; mkdir -p $O
FMX_FETCH_LANE=1 timeout 900 python -m pytest tests/test_allreduce_gpu.py tests/test_configs_gpu.py -m gpu -x -q > $O/pytest_fl.log 2>&1; echo rc=$? >> $O/pytest_fl.log
run() {  # tag ranks count fl
  FMX_FETCH_LANE=$4 timeout 300 python bench.py --ranks-per-gpu $2 --count $3 --no-train --no-cpu-baseline --no-e2e --steps 8 --warmup 3 --out $O/$1.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1])
print('$1', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['launch_us'],1))"
}
for rep in 1 2; do
for fl in 0 1; do
  run n2_64m_fl$fl 2 16777216 $fl
  run n2_1g_fl$fl 2 268435456 $fl
  run n7_r50_fl$fl 7 25557032 $fl
  run n7_64m_fl$fl 7 16777216 $fl
  run n7_1g_fl$fl 7 268435456 $fl
done; done
FMX_FETCH_LANE=1 timeout 300 python bench.py --ranks-per-gpu 2 --count 268435456 --no-train --no-cpu-baseline --no-e2e --steps 6 --warmup 2 --stamps $O/stamps_n2_fl1.json --out $O/stamps_bench.json > /dev/null 2>&1
python tools/analyze_stamps.py $O/stamps_n2_fl1.json > $O/stamps_n2_fl1.txt 2>&1; head -6 $O/stamps_n2_fl1.txt
tail -n 2 $O/pytest_fl.log
