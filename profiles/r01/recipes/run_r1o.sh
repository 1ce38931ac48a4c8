#!/bin/bash
# SM zero-copy vs copy-engine host-link capacity, 1 and 7 MPS clients.
OUT=gpurun_out/r1o; mkdir -p $OUT
timeout 500 python tools/with_mps.py python tools/probe_ce_multi.py $OUT/zc_mps.jsonl zc_d2h,zc_h2d,zc_bidir,ce+zc_d2h,bidir > $OUT/zc_mps.log 2>&1; echo "mps rc=$?" >> $OUT/log.txt
