#!/bin/bash
# Re-entry check: GPU parity suite + smoke on the restored tree, then the r1i schedule sweep.
OUT=gpurun_out/r1j; mkdir -p $OUT
nvidia-smi -q | head -40 > $OUT/smi.txt
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/log.txt
bash tools/run_r1i.sh
cp -r gpurun_out/r1i $OUT/ 2>/dev/null
