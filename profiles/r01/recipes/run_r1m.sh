#!/bin/bash
# Host-link capacity with 1 and 7 processes, with and without MPS.
OUT=gpurun_out/r1m; mkdir -p $OUT
timeout 400 python tools/probe_ce_multi.py $OUT/ce_nomps.jsonl > $OUT/ce_nomps.log 2>&1; echo "nomps rc=$?" >> $OUT/log.txt
timeout 400 python tools/with_mps.py python tools/probe_ce_multi.py $OUT/ce_mps.jsonl > $OUT/ce_mps.log 2>&1; echo "mps rc=$?" >> $OUT/log.txt
