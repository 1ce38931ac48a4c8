# why BERT's graph replay is slower than eager inside a 14 % MPS client
set -x
O=gpurun_out/r2u; mkdir -p $O
timeout 300 python tools/probe_mps_graph.py > $O/probe_full.jsonl 2> $O/probe_full.err
CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=14 timeout 400 python tools/with_mps.py python tools/probe_mps_graph.py > $O/probe_mps14.jsonl 2> $O/probe_mps14.err
cat $O/probe_*.jsonl; tail -n 3 $O/probe_mps14.err
