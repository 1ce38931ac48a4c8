#!/bin/bash
OUT=gpurun_out/r2o; mkdir -p $OUT
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench.json --stamps $OUT/stamps.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/ref.json 2> $OUT/ref.err; echo "ref rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench2.json > $OUT/bench2.log 2>&1; echo "bench2 rc=$?" >> $OUT/log.txt
