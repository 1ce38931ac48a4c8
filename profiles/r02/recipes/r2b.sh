# HEAD verification after the container restore: full GPU suite, smoke, driver-style ncu smoke, bench
set -x
O=gpurun_out/r2b; mkdir -p $O
nvidia-smi -L > $O/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $O/ncu_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $O/ref.log 2>&1; echo "ref rc=$?" >> $O/ref.log
tail -n 3 $O/pytest.log $O/smoke.log $O/ncu_smoke.log $O/bench.log $O/ref.log
