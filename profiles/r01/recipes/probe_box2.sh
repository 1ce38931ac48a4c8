#!/bin/bash
# Probe 2: cross-process direction concurrency, with and without MPS.
OUT=gpurun_out/probe2; mkdir -p $OUT
cat /usr/bin/nvidia-cuda-mps-control > $OUT/mps_wrapper.txt 2>&1
run_set() {  # $1 = tag
  for kinds in rw HD rD Hw rr HH ww DD; do
    for bl in 16 148; do
      pids=()
      for r in 0 1; do timeout 60 ./tools/probe_hostlink dir $r 2 $kinds $bl >> $OUT/dir_$1.jsonl 2>&1 & pids+=($!); done
      for p in "${pids[@]}"; do wait $p; done
      case $kinds in H*|D*) if [ $bl = 16 ]; then continue; fi;; esac
    done
  done
  # 7 processes: 3 zc readers + 4 zc writers ; and CE
  for kinds in rrrwwww HHHDDDD rrrDDDD; do
    pids=()
    for r in 0 1 2 3 4 5 6; do timeout 60 ./tools/probe_hostlink dir $r 7 $kinds 16 >> $OUT/dir7_$1.jsonl 2>&1 & pids+=($!); done
    for p in "${pids[@]}"; do wait $p; done
  done
}
run_set nomps
export CUDA_MPS_PIPE_DIRECTORY=/tmp/mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
timeout 20 nvidia-cuda-mps-control -d > $OUT/mps_start.txt 2>&1; echo "rc=$?" >> $OUT/mps_start.txt
sleep 1
timeout 30 ./tools/probe_hostlink info >> $OUT/mps_start.txt 2>&1
run_set mps
for r in 0 1; do timeout 60 ./tools/probe_hostlink pair $r 2 16 > $OUT/pair_mps_$r.jsonl 2>&1 & done; wait
echo quit | timeout 20 nvidia-cuda-mps-control >> $OUT/mps_start.txt 2>&1
cp -r /tmp/mps_log $OUT/ 2>/dev/null
