# HEAD check: full GPU suite, smoke, default bench line (graph-engine ResNet-50 leg), reference arm
set -x
O=gpurun_out/r2w; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py --out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
timeout 600 python bench.py --impl reference --out $O/ref.json > $O/ref.log 2>&1; echo "ref rc=$?" >> $O/ref.log
tail -n 3 $O/pytest.log $O/smoke.log $O/bench.log $O/ref.log
