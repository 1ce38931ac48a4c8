#!/bin/bash
# First-touch placement + CPU pinning: GPU suite, default bench, affinity probe.
OUT=gpurun_out/r2a; mkdir -p $OUT
python -c "
import os, torch
from paper_2511_09143_b200.instance import gpu_cpus
p = torch.cuda.get_device_properties(0)
print('nvml cpus', gpu_cpus(f'{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0'), 'allowed', len(os.sched_getaffinity(0)))
" > $OUT/affinity.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/log.txt
timeout 600 python bench.py --out $OUT/bench.json > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/log.txt
