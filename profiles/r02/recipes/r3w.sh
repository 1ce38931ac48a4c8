# seven ranks, mid sizes: at least N rounds per chunk (FMX_MIN_ROUNDS), slots
set -x
O=gpurun_out/r3w; mkdir -p $O
B="python bench.py --no-train --no-cpu-baseline --no-e2e --steps 6 --warmup 2"
run() {  # tag count "ENV=.."
  tag=$1; cnt=$2; envs=$3
  env $envs timeout 300 $B --count $cnt --out $O/$tag.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$tag.json').read().splitlines()[-1])
print('$tag', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3))"
}
for rep in 1 2; do for cnt in 16777216 25557032 67108864; do
  run def_$cnt $cnt FMX_X=0
  run mr4_$cnt $cnt FMX_MIN_ROUNDS=4
  run mr6_$cnt $cnt FMX_MIN_ROUNDS=6
  run k3_$cnt $cnt FMX_SLOTS=3
  run k3mr6_$cnt $cnt "FMX_SLOTS=3 FMX_MIN_ROUNDS=6"
done; done
