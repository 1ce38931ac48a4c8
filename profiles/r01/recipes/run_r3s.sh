#!/bin/bash
# Final-state check: full GPU suite, smoke, default bench, torchrun with 4 logical GPUs.
OUT=gpurun_out/r3s; mkdir -p $OUT
timeout 1800 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference > $OUT/ref.out 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
FMX_FAKE_BUS=1 FMX_DEVICE_MAP=0,0,0,0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_n4gpu.log 2>&1; echo "torchrun 4 rc=$?" >> $OUT/log.txt
