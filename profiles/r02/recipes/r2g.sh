# FMX_SYNC=kernel (flag signals / waits as one-warp kernels) vs stream memops:
# parity, DP training, headline, small-message sweep
set -x
O=gpurun_out/r2g; mkdir -p $O
FMX_SYNC=kernel timeout 900 python -m pytest tests/test_oneshot_gpu.py tests/test_allreduce_gpu.py -m gpu -x -q -k "mps or oneshot or seven or two" > $O/pytest_ksync.log 2>&1; echo "rc=$?" >> $O/pytest_ksync.log
T="python bench.py --train-only --train-model resnet50"
for i in 1 2; do
  timeout 600 $T --out $O/train_memop_$i.json > /dev/null 2>&1
  FMX_SYNC=kernel timeout 600 $T --out $O/train_ksync_$i.json > $O/train_ksync_$i.log 2>&1
done
B="python bench.py --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-e2e"
for i in 1 2; do
  timeout 300 $B > $O/ab_memop_$i.json 2>/dev/null
  FMX_SYNC=kernel timeout 300 $B > $O/ab_ksync_$i.json 2>/dev/null
done
timeout 300 python bench.py --sweep --sweep-max 16777216 > $O/sweep_memop.jsonl 2>/dev/null
FMX_SYNC=kernel timeout 300 python bench.py --sweep --sweep-max 16777216 > $O/sweep_ksync.jsonl 2>/dev/null
FMX_SYNC=kernel timeout 600 $T --stamps $O/stamps_ksync.json --out $O/train_ksync_st.json > /dev/null 2>&1
tail -n 2 $O/pytest_ksync.log
for f in $O/train_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); r=d['resnet50']; print(r['img_s'], r['ms_per_step'], r['replicas_agree'])"; done
for f in $O/ab_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); print(d['ms_per_step'], d['step_roofline']['frac'])"; done
