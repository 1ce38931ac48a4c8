# DP: stage lane in join-stream mode (FMX_JOIN_LANES=2) A/B; one-to-one ResNet-50 (full GPU);
# n=2 large-message variants (result slot via copy engine, 32 MiB slices); default bench line
set -x
O=gpurun_out/r2e; mkdir -p $O
T="python bench.py --train-only --train-model resnet50"
for i in 1 2; do
  FMX_JOIN_LANES=1 timeout 600 $T --out $O/train_jl1_$i.json > /dev/null 2>&1
  FMX_JOIN_LANES=2 timeout 600 $T --out $O/train_jl2_$i.json > $O/train_jl2_$i.log 2>&1
done
timeout 900 python bench.py --train-only --train-model resnet50 --ranks-per-gpu 1 --train-mode full --batch 224 --out $O/train_resnet50_full.json > $O/train_full.log 2>&1
S="python bench.py --sweep --ranks-per-gpu 2 --sweep-max 1073741824"
timeout 600 $S > $O/sweep_n2.jsonl 2>/dev/null
FMX_RESULT_VIA_CE=1 timeout 600 $S > $O/sweep_n2_rce.jsonl 2>/dev/null
timeout 600 $S --slice-bytes 33554432 > $O/sweep_n2_s32.jsonl 2>/dev/null
timeout 600 python bench.py --steps 20 --warmup 5 --out $O/bench.json > $O/bench.log 2>&1
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'])"; done
tail -n 3 $O/train_jl2_1.log $O/train_full.log
