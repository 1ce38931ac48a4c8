# fetch lane on by default at <= 2 ranks per GPU: GPU tests + the two-rank sweep
set -x
O=gpurun_out/r3s; mkdir -p $O
timeout 1500 python -m pytest tests/test_allreduce_gpu.py tests/test_stress_gpu.py tests/test_graph_dp_gpu.py tests/test_ddp_gpu.py tests/test_configs_gpu.py -m gpu -x -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 400 python bench.py --sweep --ranks-per-gpu 2 --out $O/sweep_n2.jsonl > $O/sweep_n2.log 2>&1
python -c "
import json
for l in open('$O/sweep_n2.jsonl'):
    x=json.loads(l); print(x['bytes'], round(x['ms'],3), round(x.get('step_roofline_frac') or 0,3))"
tail -n 2 $O/pytest.log
