# DP: FMX_JOIN_LANES=2 with the stage lane at the side stream's priority; bucket sizes; stamps
set -x
O=gpurun_out/r2f; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
for i in 1 2; do
  FMX_JOIN_LANES=1 timeout 600 $T --out $O/train_jl1_$i.json > /dev/null 2>&1
  FMX_JOIN_LANES=2 timeout 600 $T --out $O/train_jl2_$i.json > $O/train_jl2_$i.log 2>&1
done
FMX_JOIN_LANES=2 timeout 600 $T --bucket-mb 4 --out $O/train_jl2_b4.json > /dev/null 2>&1
FMX_JOIN_LANES=2 timeout 600 $T --bucket-mb 16 --out $O/train_jl2_b16.json > /dev/null 2>&1
FMX_JOIN_LANES=1 timeout 600 $T --bucket-mb 16 --out $O/train_jl1_b16.json > /dev/null 2>&1
FMX_JOIN_LANES=2 timeout 600 $T --stamps $O/stamps_jl2.json --out $O/train_jl2_st.json > /dev/null 2>&1
FMX_JOIN_LANES=1 timeout 600 $T --stamps $O/stamps_jl1.json --out $O/train_jl1_st.json > /dev/null 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'])"; done
