set -x
O=gpurun_out/r2a; mkdir -p $O
nvidia-smi -L > $O/smi.txt
timeout 120 ncu --target-processes all bash -c 'env | grep -i -E "inject|nsight|^nv_|nsys"' > $O/ncu_env.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "ddp_arith or reduce_kernel or test_ddp_gpu" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $O/ncu_smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/bench.log
tail -n 3 $O/pytest.log $O/ncu_smoke.log $O/bench.log
