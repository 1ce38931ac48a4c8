# one-shot small-message allreduce: parity + latency sweep; batched-copy probe
set -x
O=gpurun_out/r2c; mkdir -p $O
timeout 900 python -m pytest tests/test_oneshot_gpu.py tests/test_allreduce_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python bench.py --sweep --sweep-max 4194304 > $O/sweep_n7.jsonl 2> $O/sweep_n7.err; echo "rc=$?" >> $O/sweep_n7.err
timeout 300 python bench.py --sweep --sweep-max 4194304 --ranks-per-gpu 2 > $O/sweep_n2.jsonl 2> $O/sweep_n2.err
FMX_ONESHOT_MAX=0 timeout 300 python bench.py --sweep --sweep-max 262144 > $O/sweep_n7_nooneshot.jsonl 2>&1
# (probe source removed: the batched-copy API it used is closed on this pool)
# (probe source removed: the batched-copy API it used is closed on this pool)
tail -n 3 $O/pytest.log; cat $O/sweep_n7.jsonl | cut -c1-200; cat $O/probe_batch.jsonl
