# small-message latency, old vs new reduce kernel (load restructure), same lease, alternating
set -x
O=gpurun_out/r5e; mkdir -p $O
L=paper_2511_09143_b200/libflexshm.so
for rep in 1 2; do for v in old new; do
  cp gpurun_ab/libflexshm_$v.so $L
  timeout 300 python bench.py --sweep --sweep-max 4194304 --out $O/${v}_n7_$rep.jsonl > /dev/null 2>&1
  timeout 300 python bench.py --sweep --sweep-max 4194304 --ranks-per-gpu 2 --out $O/${v}_n2_$rep.jsonl > /dev/null 2>&1
done; done
cp gpurun_ab/libflexshm_new.so $L
for f in $O/*.jsonl; do python -c "
import json,sys
print('$f'.split('/')[-1], ' '.join('%g'%round(json.loads(l)['ms'],4) for l in open('$f') if json.loads(l).get('op')=='allreduce'))"; done | tee $O/summary.txt
