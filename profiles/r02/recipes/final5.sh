#!/bin/bash
# Closing check of the shipped kernel: smoke plain and under ncu (the driver's instrumented smoke),
# reference arm, ncu launch list of the default allreduce and a full capture of one reduce piece
OUT=gpurun_out/final5; mkdir -p $OUT
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --target-processes all -c 400 --csv --log-file $OUT/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" > $OUT/ncu_smoke.log 2>&1; echo "ncu smoke rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
timeout 400 ncu --target-processes all --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --no-train --mode green > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> $OUT/log.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:fmx_reduce -s 2 -c 1 -o $OUT/reduce_full python tools/reduce_once.py > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/log.txt
python tools/ncu_summary.py $OUT/launches.csv $OUT/reduce_full.ncu-rep > $OUT/ncu_summary.json 2> $OUT/ncu_summary.err
cat $OUT/log.txt $OUT/smoke.log; tail -n 3 $OUT/ncu_smoke.log
