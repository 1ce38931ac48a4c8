# reduce kernel's zero-copy result store under concurrent copy-engine traffic (probe);
# result slot by copy engine A/B on the headline
set -x
O=gpurun_out/r2k; mkdir -p $O
timeout 120 python tools/probe_zc_contention.py > $O/probe_zc_full.jsonl 2>&1
CUDA_MPS_ACTIVE_THREAD_PERCENTAGE=14 timeout 120 python tools/with_mps.py python tools/probe_zc_contention.py > $O/probe_zc_mps14.jsonl 2>&1
B="python bench.py --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-e2e"
for i in 1 2 3; do
  timeout 300 $B > $O/ab_base_$i.json 2>/dev/null
  FMX_RESULT_VIA_CE=1 timeout 300 $B > $O/ab_rce_$i.json 2>/dev/null
done
cat $O/probe_zc_*.jsonl
for f in $O/ab_*.json; do echo $f; python -c "import json; d=json.loads(open('$f').read().splitlines()[-1]); print(d['ms_per_step'], d['step_roofline']['frac'], d['roofline']['launch_us'])"; done
