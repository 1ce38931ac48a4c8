# DP legs with the shipped kernel: ResNet-50 / BERT-base (graph engine, with the no-sync bound),
# MobileNetV2 at 4 ranks, ResNet-50 one-to-one (whole GPU) and the PerfModel recalibration
OUT=gpurun_out/r5i; mkdir -p $OUT
for m in resnet50 bert; do
  timeout 600 python bench.py --train-only --train-model $m --train-no-sync --out $OUT/train_$m.json > $OUT/train_$m.log 2>&1; echo "train $m rc=$?" >> $OUT/log.txt
done
timeout 400 python bench.py --train-only --train-model mobilenet_v2 --ranks-per-gpu 4 --train-no-sync --out $OUT/train_mobilenet_v2.json > $OUT/train_mbv2.log 2>&1; echo "train mbv2 rc=$?" >> $OUT/log.txt
timeout 400 python bench.py --train-only --train-model resnet50 --ranks-per-gpu 1 --train-mode full --batch 224 --out $OUT/train_resnet50_full.json > $OUT/train_r50full.log 2>&1; echo "train r50 full rc=$?" >> $OUT/log.txt
python tools/calibrate_perfmodel.py $OUT/perfmodel_b200.json $OUT/train_resnet50.json $OUT/train_resnet50_full.json >> $OUT/log.txt 2>&1
for f in $OUT/train_*.json; do python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); k=list(d)[0]; r=d[k]
ns=r.get('no_sync') or {}
print(k, r.get('img_s') or r.get('seq_s') or r.get('samples_s'), round(r['ms_per_step'],2), r.get('replicas_agree'), ns.get('img_s') or ns.get('seq_s'))" >> $OUT/log.txt; done
cat $OUT/log.txt
