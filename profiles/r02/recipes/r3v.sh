# seven ranks: result slot by copy engine, with and without the fetch lane
set -x
O=gpurun_out/r3v; mkdir -p $O
B="python bench.py --no-train --no-cpu-baseline --no-e2e --steps 5 --warmup 2"
run() {  # tag count "ENV=.."
  tag=$1; cnt=$2; envs=$3
  env $envs timeout 300 $B --count $cnt --out $O/$tag.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$tag.json').read().splitlines()[-1])
print('$tag', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3))"
}
for rep in 1 2; do for cnt in 16777216 25557032 268435456; do
  run def_$cnt $cnt FMX_X=0
  run rce_$cnt $cnt FMX_RESULT_VIA_CE=1
  run flrce_$cnt $cnt "FMX_FETCH_LANE=1 FMX_RCE_ROUNDS=1"
done; done
