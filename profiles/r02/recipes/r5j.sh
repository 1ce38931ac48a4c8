# soaks with the shipped kernel (host sources in round 1's form): random collective programs,
# sha256-exact vs the oracle
O=gpurun_out/r5j; mkdir -p $O
timeout 1200 python tools/soak.py 7 1 mps 401 300 > $O/soak_n7.log 2>&1; echo "rc=$?" >> $O/soak_n7.log
timeout 900 python tools/soak.py 3 1 green 402 120 > $O/soak_n3_green.log 2>&1; echo "rc=$?" >> $O/soak_n3_green.log
timeout 1200 python tools/soak.py 28 4 mps 403 60 > $O/soak_n28_4gpu.log 2>&1; echo "rc=$?" >> $O/soak_n28_4gpu.log
timeout 900 python tools/graph_soak.py 3 404 16 300 50 1 > $O/graph_soak_n3_sticky.log 2>&1; echo "rc=$?" >> $O/graph_soak_n3_sticky.log
tail -n 2 $O/*.log
