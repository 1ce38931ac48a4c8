# PerfModel recalibration on the graph engine: one-to-many (7 x 1g, batch 32) vs one-to-one
# (the whole B200, batch 224), same model and engine
set -x
O=gpurun_out/r3h; mkdir -p $O
timeout 600 python bench.py --train-only --train-model resnet50 --train-no-sync --out $O/train_many.json > $O/train_many.log 2>&1
timeout 600 python bench.py --train-only --train-model resnet50 --ranks-per-gpu 1 --train-mode full --batch 224 --out $O/train_one.json > $O/train_one.log 2>&1
python tools/calibrate_perfmodel.py $O/perfmodel_b200.json $O/train_many.json $O/train_one.json
tail -n 2 $O/train_one.log | cut -c1-400
