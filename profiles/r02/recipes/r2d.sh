# FMX_RAMP=4 (remainder-sized first round) A/B on the headline + large-size sweeps;
# compute-sanitizer; one-to-one ResNet-50 (PerfModel calibration); smoke
set -x
O=gpurun_out/r2d; mkdir -p $O
B="python bench.py --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-e2e"
for i in 1 2 3; do
  FMX_RAMP=0 timeout 300 $B > $O/ab_ramp0_$i.json 2>/dev/null
  FMX_RAMP=4 timeout 300 $B > $O/ab_ramp4_$i.json 2>/dev/null
done
for r in 0 4; do
  FMX_RAMP=$r timeout 600 python bench.py --sweep > $O/sweep_n7_ramp$r.jsonl 2>/dev/null
  FMX_RAMP=$r timeout 600 python bench.py --sweep --ranks-per-gpu 2 > $O/sweep_n2_ramp$r.jsonl 2>/dev/null
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
# sanitizers: the reduce kernel alone, then the 2-rank smoke (all processes)
export FMX_ITERS=2
for t in memcheck racecheck synccheck initcheck; do
  timeout 300 compute-sanitizer --tool $t --error-exitcode 9 python tools/reduce_once.py > $O/sanitize_reduce_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_reduce_$t.log
done
for t in memcheck synccheck; do
  FMX_SERIALIZE=1 timeout 600 compute-sanitizer --tool $t --target-processes all --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > $O/sanitize_smoke_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_smoke_$t.log
done
# PerfModel: one-to-many (7 x 1g MPS, batch 32) vs one-to-one (whole GPU, batch 224)
timeout 900 python bench.py --train-only --train-model resnet50 --train-no-sync --out $O/train_resnet50.json > $O/train_resnet50.log 2>&1
timeout 900 python bench.py --train-only --train-model resnet50 --ranks-per-gpu 1 --train-mode full --batch 224 --out $O/train_resnet50_full.json > $O/train_resnet50_full.log 2>&1
tail -n 2 $O/*.log
for f in $O/ab_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().splitlines()[-1]); print(d['ms_per_step'], d['step_roofline']['frac'])"; done
