# soaks with the shipped reduce kernel: random collective programs, sha256-exact vs the oracle
set -x
O=gpurun_out/r5g; mkdir -p $O
timeout 1200 python tools/soak.py 7 1 mps 301 300 > $O/soak_n7.log 2>&1; echo "rc=$?" >> $O/soak_n7.log
timeout 900 python tools/soak.py 2 1 mps 302 150 > $O/soak_n2.log 2>&1; echo "rc=$?" >> $O/soak_n2.log
timeout 900 python tools/soak.py 5 1 green 303 100 > $O/soak_n5_green.log 2>&1; echo "rc=$?" >> $O/soak_n5_green.log
timeout 1200 python tools/soak.py 14 2 mps 304 100 > $O/soak_n14_2gpu.log 2>&1; echo "rc=$?" >> $O/soak_n14_2gpu.log
timeout 900 python tools/graph_soak.py 7 305 12 300 50 > $O/graph_soak_n7.log 2>&1; echo "rc=$?" >> $O/graph_soak_n7.log
tail -n 2 $O/*.log
