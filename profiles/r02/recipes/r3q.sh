# two ranks per GPU (n=2): schedule variants at 64 MiB and 1 GiB, and a GPU-clock timeline
set -x
O=gpurun_out/r3q; mkdir -p $O
B="python bench.py --ranks-per-gpu 2 --no-train --no-cpu-baseline --no-e2e --steps 6 --warmup 2"
run() {  # tag count "ENV=.." "extra args"
  tag=$1; cnt=$2; envs=$3; args=$4
  env $envs timeout 300 $B --count $cnt $args --out $O/$tag.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$tag.json').read().splitlines()[-1])
print('$tag', round(d['ms_per_step'],3), round(d['step_roofline']['frac'],3))"
}
for cnt in 16777216 268435456; do
  run def_$cnt $cnt FMX_X=0 ""
  run rce_$cnt $cnt FMX_RESULT_VIA_CE=1 ""
  run k2_$cnt $cnt FMX_SLOTS=2 ""
  run k3_$cnt $cnt FMX_SLOTS=3 ""
  run s8_$cnt $cnt FMX_X=0 "--slice-bytes 8388608"
  run s32_$cnt $cnt FMX_X=0 "--slice-bytes 33554432"
  run ramp0_$cnt $cnt FMX_RAMP=0 ""
  run lanes2_$cnt $cnt FMX_LANES=2 ""
  run def2_$cnt $cnt FMX_X=0 ""
done
timeout 300 $B --count 268435456 --stamps $O/stamps_n2.json --out $O/stamps_bench.json > /dev/null 2>&1
python tools/analyze_stamps.py $O/stamps_n2.json > $O/stamps_n2.txt 2>&1; head -8 $O/stamps_n2.txt
