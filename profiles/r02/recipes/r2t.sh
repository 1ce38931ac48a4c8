# graph engine + deferred gather (stage of bucket b+1 before the gather of b on one stream)
set -x
O=gpurun_out/r2t; mkdir -p $O
timeout 500 python -m pytest tests/test_graph_dp_gpu.py tests/test_ddp_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
T="python bench.py --train-only --train-model resnet50"
for d in 1 0 1 0; do
FMX_DEFER=$d timeout 600 $T --out $O/train_defer$d.json >> $O/train.log 2>&1
python -c "
import json; d=json.loads(open('$O/train_defer$d.json').read().splitlines()[-1]); r=d['resnet50']
print('defer=$d', r['img_s'], r['ms_per_step'], r['replicas_agree'])"
done
for b in 4 16; do
timeout 600 $T --bucket-mb $b --out $O/train_b$b.json >> $O/train.log 2>&1
python -c "
import json; d=json.loads(open('$O/train_b$b.json').read().splitlines()[-1]); r=d['resnet50']
print('bucket=$b', r['img_s'], r['ms_per_step'], r['replicas_agree'])"
done
FMX_HOOK_STAMP=1 timeout 600 $T --stamps $O/stamps_graph.json --out $O/train_stamps.json > /dev/null 2>&1
tail -3 $O/pytest.log
