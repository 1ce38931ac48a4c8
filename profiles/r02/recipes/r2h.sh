# one-shot with the OS_READY wait fused into the reduction (MPS ranks); small-message sweeps;
# BASELINE C4 / C3 bench lines on logical GPUs; device-path GPU-clock timeline
set -x
O=gpurun_out/r2h; mkdir -p $O
timeout 900 python -m pytest tests/test_oneshot_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 300 python bench.py --sweep --sweep-max 4194304 > $O/sweep_n7.jsonl 2>/dev/null
timeout 300 python bench.py --sweep --sweep-max 4194304 --ranks-per-gpu 2 > $O/sweep_n2.jsonl 2>/dev/null
FMX_SPIN_WAIT=0 timeout 300 python bench.py --sweep --sweep-max 262144 > $O/sweep_n7_nospin.jsonl 2>/dev/null
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
FMX_DEVICE_MAP=0,0 FMX_FAKE_BUS=1 timeout 900 $TR bench.py --gpus 2 --ranks-per-gpu 7 --dtype bf16 --count 109483778 --steps 10 --warmup 3 --no-train --no-cpu-baseline --out $O/bench_c4_logical.json > $O/bench_c4.log 2>&1; echo "c4 rc=$?" >> $O/bench_c4.log
FMX_DEVICE_MAP=0,0 FMX_FAKE_BUS=1 timeout 900 $TR bench.py --gpus 2 --ranks-per-gpu 2 --count 3504872 --steps 20 --warmup 5 --no-train --no-cpu-baseline --out $O/bench_c3_logical.json > $O/bench_c3.log 2>&1; echo "c3 rc=$?" >> $O/bench_c3.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-train --no-cpu-baseline --no-e2e --stamps $O/stamps.json --out $O/bench_stamps.json > $O/bench_stamps.log 2>&1
python tools/analyze_stamps.py $O/stamps.json > $O/stamps_summary.txt 2>&1
tail -n 2 $O/pytest.log $O/smoke.log $O/bench_c4.log $O/bench_c3.log; head -30 $O/stamps_summary.txt
