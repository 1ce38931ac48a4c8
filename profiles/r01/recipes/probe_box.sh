#!/bin/bash
# Box probe. Output: gpurun_out/probe/*.
set -x
OUT=gpurun_out/probe; mkdir -p $OUT
{
nvidia-smi
nvidia-smi -q | grep -i -E "MIG|Product|Bus Id|Link|PCIe|Gen|Width|Max|Current" | head -80
nvidia-smi topo -m
nvidia-smi mig -lgip 2>&1 | head -40
which nvidia-cuda-mps-control nvidia-cuda-mps-server; ls -la /usr/bin/nvidia* 2>&1 | head -30
lscpu; numactl -H 2>&1 | head; nproc; free -g; df -h /dev/shm; ulimit -l
cat /proc/meminfo | head -5
} > $OUT/system.txt 2>&1
timeout 60 ./tools/probe_hostlink info > $OUT/info.jsonl 2>&1
timeout 300 ./tools/probe_hostlink bw > $OUT/bw.jsonl 2>&1
for np in 2 7; do
  for bl in 16 148; do
    pids=()
    for r in $(seq 0 $((np-1))); do timeout 120 ./tools/probe_hostlink pair $r $np $bl > $OUT/pair_${np}_${bl}_$r.jsonl 2>&1 & pids+=($!); done
    for p in "${pids[@]}"; do wait $p; done
  done
done
timeout 120 python - > $OUT/green.txt 2>&1 <<'PY'
import torch, time
print(torch.cuda.get_device_name(0), torch.cuda.get_device_properties(0))
for n in (8, 16, 18, 20, 24, 32):
    try:
        g = torch.cuda.GreenContext.create(n, 0)
        g.set_context()
        s = g.Stream()
        with torch.cuda.stream(s):
            x = torch.randn(1 << 24, device="cuda"); y = x * 2
            torch.cuda.synchronize()
            t = time.time()
            for _ in range(20): y = x * 2
            torch.cuda.synchronize()
        print("green", n, "ok", (time.time() - t) / 20 * 1e3, "ms")
        g.pop_context()
    except Exception as e:
        print("green", n, "ERR", repr(e))
PY
