#!/bin/bash
# bench.py under torchrun with 2 and 4 logical GPUs on one B200 (7 ranks each, fake bus ids).
OUT=gpurun_out/r3o; mkdir -p $OUT
FMX_FAKE_BUS=1 FMX_DEVICE_MAP=0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_n2gpu.log 2>&1; echo "torchrun 2 rc=$?" >> $OUT/log.txt
FMX_FAKE_BUS=1 FMX_DEVICE_MAP=0,0,0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_n4gpu.log 2>&1; echo "torchrun 4 rc=$?" >> $OUT/log.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29563 bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > $OUT/ref_n4gpu.log 2>&1; echo "ref 4 rc=$?" >> $OUT/log.txt
