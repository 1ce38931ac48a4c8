# size sweeps with the final kernels (n = 7 and n = 2), and a second default bench line
set -x
O=gpurun_out/r5d; mkdir -p $O
timeout 600 python bench.py --sweep --out $O/sweep_n7.jsonl > $O/sweep_n7.log 2>&1; echo "sweep7 rc=$?" >> $O/log.txt
timeout 400 python bench.py --sweep --ranks-per-gpu 2 --out $O/sweep_n2.jsonl > $O/sweep_n2.log 2>&1; echo "sweep2 rc=$?" >> $O/log.txt
timeout 900 python bench.py --out $O/bench.json > $O/bench.log 2>&1; echo "bench rc=$?" >> $O/log.txt
cat $O/log.txt
