# pacing the D2H stage: stage by the SM copy kernel (FMX_STAGE_ZC=1) with a CTA cap per
# launch (FMX_COPY_CTAS) so seven ranks' stage stores leave H2D more of the link
set -x
O=gpurun_out/r5c; mkdir -p $O
B="python bench.py --no-train --no-cpu-baseline --no-e2e --steps 5 --warmup 3"
run() {  # tag count env
  env $3 timeout 400 $B --count $2 --out $O/$1.json > $O/$1.log 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); r=d['roofline']
print('$1', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3), round(r['launch_us'],1))" >> $O/summary.txt
}
for rep in 1 2; do
  run def_c2_$rep 25557032 FMX_X=0
  run szc_c2_$rep 25557032 FMX_STAGE_ZC=1
  for k in 6 12 24 48 96; do
    run szc${k}_c2_$rep 25557032 "FMX_STAGE_ZC=1 FMX_COPY_CTAS=$k"
  done
done
run def_64m 16777216 FMX_X=0
for k in 12 24 48; do run szc${k}_64m 16777216 "FMX_STAGE_ZC=1 FMX_COPY_CTAS=$k"; done
cat $O/summary.txt
