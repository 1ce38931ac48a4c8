# seven ranks: fetch lane + copy-engine result slot from round 1 (flrce) vs the defaults,
# allreduce 16 MiB, 64 MiB, 256 MiB (x2), 1 GiB (x1), C2 with the host path, ResNet-50 DP graph leg; two reps each
set -x
O=gpurun_out/r5a; mkdir -p $O
B="python bench.py --no-train --no-cpu-baseline --steps 5 --warmup 3"
FL="FMX_FETCH_LANE=1 FMX_RCE_ROUNDS=1"
run() {  # tag count env extra
  env $3 timeout 400 $B --count $2 $4 --out $O/$1.json > $O/$1.log 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); e=d.get('e2e') or {}
print('$1', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(d['roofline']['frac'],3), e.get('ms_per_step'))" >> $O/summary.txt
}
tr() {  # tag env
  env $2 timeout 600 python bench.py --train-only --train-model resnet50 --out $O/$1.json > $O/$1.log 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); r=d['resnet50']
print('$1', round(r['img_s']), round(r['ms_per_step'],2), r['replicas_agree'])" >> $O/summary.txt
}
for rep in 1 2; do
  for cnt in 4194304 16777216 67108864; do
    run def_${cnt}_$rep $cnt FMX_X=0 --no-e2e
    run fl_${cnt}_$rep $cnt "$FL" --no-e2e
  done
  run def_c2_$rep 25557032 FMX_X=0
  run fl_c2_$rep 25557032 "$FL"
  tr trdef_$rep FMX_X=0
  tr trfl_$rep "$FL"
done
run def_1g 268435456 FMX_X=0 --no-e2e
run fl_1g 268435456 "$FL" --no-e2e
cat $O/summary.txt
