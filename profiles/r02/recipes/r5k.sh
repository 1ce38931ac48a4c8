# 28 ranks over 4 logical GPUs, a shorter soak than r5j's (60 ops did not finish in 1200 s)
O=gpurun_out/r5k; mkdir -p $O
start=$(date +%s)
timeout 840 python tools/soak.py 28 4 mps 405 25 > $O/soak_n28_4gpu.log 2>&1; echo "rc=$? wall_s=$(( $(date +%s) - start ))" >> $O/soak_n28_4gpu.log
tail -n 3 $O/soak_n28_4gpu.log
