# after the fused-SGD kernel change: full GPU suite, smoke, default bench line
set -x
O=gpurun_out/r4c; mkdir -p $O
timeout 1800 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/log.txt
timeout 900 python bench.py --out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/log.txt
python -c "
import json; d=json.loads(open('$O/bench.json').read().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), round(d['resnet50']['img_s']), d['resnet50']['replicas_agree'])" >> $O/log.txt
tail -n 2 $O/pytest_gpu.log >> $O/log.txt
cat $O/log.txt
