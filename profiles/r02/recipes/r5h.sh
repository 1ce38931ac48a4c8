# the shipped reduce kernel: joint loads for HBM sources, the round-1 per-vector form for host sources:
# full GPU suite, small-message A/B vs the pre-round kernel on one lease, default bench line
set -x
O=gpurun_out/r5h; mkdir -p $O
L=paper_2511_09143_b200/libflexshm.so
cp gpurun_ab/libflexshm_new3.so $L
timeout 1500 python -m pytest tests -x -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/log.txt
tail -n 2 $O/pytest_gpu.log >> $O/log.txt
for rep in 1 2; do for v in old new3; do
  cp gpurun_ab/libflexshm_$v.so $L
  timeout 300 python bench.py --sweep --sweep-max 4194304 --out $O/${v}_n7_$rep.jsonl > /dev/null 2>&1
  timeout 300 python bench.py --sweep --sweep-max 4194304 --ranks-per-gpu 2 --out $O/${v}_n2_$rep.jsonl > /dev/null 2>&1
done; done
cp gpurun_ab/libflexshm_new3.so $L
timeout 900 python bench.py --out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/log.txt
for f in $O/*.jsonl; do python -c "
import json,sys
print('$f'.split('/')[-1], ' '.join('%g'%round(json.loads(l)['ms'],4) for l in open('$f') if json.loads(l).get('op')=='allreduce'))"; done | sort > $O/summary.txt
python -c "
import json; d=json.loads(open('$O/bench.json').read().splitlines()[-1])
print('bench', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), round(d['e2e']['ms_per_step'],3), round(d['resnet50']['img_s']), d['resnet50']['replicas_agree'], d['clocks'])" >> $O/log.txt
cat $O/log.txt $O/summary.txt
