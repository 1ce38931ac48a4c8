# reduce kernel: all U x B source loads in flight before accumulation (new) vs one vector's
# sources at a time (old), same lease; default schedule and fetch lane + CE result slot (fl)
set -x
O=gpurun_out/r5b; mkdir -p $O
L=paper_2511_09143_b200/libflexshm.so
use() { cp gpurun_ab/libflexshm_$1.so $L; }
use new
timeout 900 python -m pytest tests/test_reduce_kernel_gpu.py tests/test_allreduce_gpu.py tests/test_oneshot_gpu.py tests/test_ddp_arith_gpu.py tests/test_graph_dp_gpu.py -x -q > $O/pytest_new.log 2>&1; echo "pytest rc=$?" >> $O/summary.txt
tail -n 2 $O/pytest_new.log >> $O/summary.txt
B="python bench.py --no-train --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
FL="FMX_FETCH_LANE=1 FMX_RCE_ROUNDS=1"
run() {  # tag count env
  env $3 timeout 400 $B --count $2 --out $O/$1.json > $O/$1.log 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); r=d['roofline']
print('$1', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(r['launch_us'],1), round((r.get('isolated') or {}).get('launch_us',0),1))" >> $O/summary.txt
}
tr() {  # tag env
  env $2 timeout 600 python bench.py --train-only --train-model resnet50 --out $O/$1.json > $O/$1.log 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); r=d['resnet50']
print('$1', round(r['img_s']), round(r['ms_per_step'],2), r['replicas_agree'])" >> $O/summary.txt
}
for rep in 1 2; do
  for v in old new; do
    use $v
    run ${v}_def_c2_$rep 25557032 FMX_X=0
    run ${v}_fl_c2_$rep 25557032 "$FL"
    run ${v}_def_64m_$rep 16777216 FMX_X=0
    run ${v}_fl_64m_$rep 16777216 "$FL"
  done
done
for v in old new; do
  use $v
  run ${v}_def_1g 268435456 FMX_X=0
  run ${v}_fl_1g 268435456 "$FL"
  tr ${v}_trdef FMX_X=0
  tr ${v}_trfl "$FL"
done
use new
cat $O/summary.txt
