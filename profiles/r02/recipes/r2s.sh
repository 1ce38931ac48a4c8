# graph engine knobs: FMX_JOIN_LANES (stage / gather lanes as graph branches), FMX_MIN_ROUNDS;
# BERT eager-vs-graph step probe
set -x
O=gpurun_out/r2s; mkdir -p $O
FMX_JOIN_LANES=3 timeout 500 python -m pytest tests/test_graph_dp_gpu.py -m gpu -x -q > $O/pytest_jl3.log 2>&1; echo rc=$? >> $O/pytest_jl3.log
T="python bench.py --train-only --train-model resnet50"
for jl in 1 2 3; do for mr in 1 2; do
FMX_JOIN_LANES=$jl FMX_MIN_ROUNDS=$mr timeout 600 $T --out $O/train_jl${jl}_mr${mr}.json > /dev/null 2>&1
done; done
timeout 300 python tools/probe_graph_step.py bert > $O/probe_bert_full.jsonl 2>&1
CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=14 timeout 300 python tools/with_mps.py python tools/probe_graph_step.py bert > $O/probe_bert_mps14.jsonl 2>&1
for f in $O/train_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().splitlines()[-1]); k=list(d)[0]; r=d[k]; u=[x for x in r if x.endswith('_s')][0]
print(k, r[u], r['ms_per_step'], r['replicas_agree'])"; done
tail -2 $O/pytest_jl3.log; cat $O/probe_bert_*.jsonl | grep probe
