# after the capture-state fixes: graph / DDP / stress GPU tests, ResNet-50 DP
set -x
O=gpurun_out/r3m; mkdir -p $O
timeout 1200 python -m pytest tests/test_graph_dp_gpu.py tests/test_ddp_gpu.py tests/test_stress_gpu.py tests/test_oneshot_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 600 python bench.py --train-only --train-model resnet50 --out $O/train_resnet50.json > /dev/null 2>&1
python -c "
import json; d=json.loads(open('$O/train_resnet50.json').read().splitlines()[-1]); r=d['resnet50']
print('resnet50', r['img_s'], r['ms_per_step'], r['replicas_agree'])"
tail -n 2 $O/pytest.log
