# graph engine: bf16-compressed exchange; the DP train leg across torchrun processes
# (2 logical GPUs on the one B200: 14 instance ranks, functional check, not a scaling number)
set -x
O=gpurun_out/r2x; mkdir -p $O
timeout 600 python -m pytest tests/test_graph_dp_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 600 python bench.py --train-only --train-model resnet50 --compress bf16 --out $O/train_bf16.json > $O/train_bf16.log 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633"
FMX_DEVICE_MAP=0,0 FMX_FAKE_BUS=1 timeout 900 $TR bench.py --gpus 2 --train-only --train-model resnet50 --train-steps 5 --train-warmup 3 --out $O/train_2lgpu.json > $O/train_2lgpu.log 2>&1; echo "rc=$?" >> $O/train_2lgpu.log
FMX_DEVICE_MAP=0,0 FMX_FAKE_BUS=1 timeout 900 $TR bench.py --gpus 2 --steps 5 --warmup 3 --train-steps 5 --train-warmup 3 --no-cpu-baseline --out $O/bench_2lgpu.json > $O/bench_2lgpu.log 2>&1; echo "rc=$?" >> $O/bench_2lgpu.log
tail -n 2 $O/pytest.log; tail -n 3 $O/train_bf16.log $O/train_2lgpu.log $O/bench_2lgpu.log | cut -c1-600
