# Does host-link traffic slow the GPU's own compute (eager launches vs CUDA graph)?
set -x
O=gpurun_out/r2o; mkdir -p $O
timeout 300 python tools/probe_launch_contention.py > $O/probe_full.jsonl 2> $O/probe_full.err
PROBE_COPIES=80 CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=14 timeout 400 python tools/with_mps.py python tools/probe_launch_contention.py > $O/probe_mps14.jsonl 2> $O/probe_mps14.err
cat $O/probe_*.jsonl; tail -3 $O/*.err
