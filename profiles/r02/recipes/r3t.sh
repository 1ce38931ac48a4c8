# two ranks per GPU with the fetch lane: result slot by copy engine, slice, slots
set -x
O=gpurun_out/r3t; mkdir -p $O
B="python bench.py --ranks-per-gpu 2 --no-train --no-cpu-baseline --no-e2e --steps 8 --warmup 3"
run() {  # tag count "ENV=.." "extra args"
  tag=$1; cnt=$2; envs=$3; args=$4
  env $envs timeout 300 $B --count $cnt $args --out $O/$tag.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$tag.json').read().splitlines()[-1])
print('$tag', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3))"
}
for rep in 1 2; do for cnt in 16777216 268435456; do
  run fl_$cnt $cnt FMX_X=0 ""
  run flrce_$cnt $cnt FMX_RESULT_VIA_CE=1 ""
  run fls32_$cnt $cnt FMX_X=0 "--slice-bytes 33554432"
  run flk3_$cnt $cnt FMX_SLOTS=3 ""
  run flk2_$cnt $cnt FMX_SLOTS=2 ""
done; done
