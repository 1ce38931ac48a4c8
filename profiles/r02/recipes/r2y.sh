# round-2 ncu evidence on the final kernels: launch list of the default bench allreduce
# (device path, serialise mode under the profiler), full capture of one reduce piece, and
# the driver's ncu-instrumented 2-rank smoke
set -x
O=gpurun_out/r2y; mkdir -p $O
timeout 400 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-train --mode green > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $O/ncu_launch.log
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $O/reduce_full python tools/reduce_once.py > $O/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $O/ncu_full.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $O/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $O/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $O/ncu_smoke.log
python tools/ncu_summary.py $O/launches.csv $O/reduce_full.ncu-rep > $O/ncu_summary.json 2> $O/ncu_summary.err
tail -n 2 $O/ncu_launch.log $O/ncu_full.log $O/ncu_smoke.log; head -c 3000 $O/ncu_summary.json
