# BERT-base DP (link-bound): extra lanes in the graph (FMX_JOIN_LANES), bucket size
set -x
O=gpurun_out/r3x; mkdir -p $O
T="python bench.py --train-only --train-model bert"
run() {  # tag "ENV" "args"
  env $2 timeout 600 $T $3 --out $O/$1.json > /dev/null 2>&1
  python -c "
import json; d=json.loads(open('$O/$1.json').read().splitlines()[-1]); r=d['bert']
print('$1', round(r['seq_s']), round(r['ms_per_step'],2), r['replicas_agree'])"
}
run def FMX_X=0 ""
run jl3 FMX_JOIN_LANES=3 ""
run jl2 FMX_JOIN_LANES=2 ""
run jl3_b50 FMX_JOIN_LANES=3 "--bucket-mb 50"
run jl3_nodefer "FMX_JOIN_LANES=3 FMX_DEFER=0" ""
run def2 FMX_X=0 ""
