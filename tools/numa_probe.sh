#!/bin/bash
# Where do pinned buffers land relative to the GPU, and does a 44 GB host allocation
# (the C1 full-size reference test) change the PCIe rates of the next process?
out=gpurun_out/numa_probe.log; : > $out
{
lscpu | grep -E "NUMA|Socket|Model name|^CPU\(s\)"
for d in /sys/bus/pci/devices/*; do if [ "$(cat $d/class 2>/dev/null)" = "0x030200" ]; then echo "gpu $d numa_node $(cat $d/numa_node) local_cpus $(cat $d/local_cpulist)"; fi; done
grep -E "MemTotal|MemFree|^Cached" /proc/meminfo
cat /sys/devices/system/node/node*/meminfo 2>/dev/null | grep -E "MemFree|FilePages"
taskset -p $$
echo "--- probe (fresh)"; python tools/pcie_probe.py
echo "--- after touching 44 GB of host memory in another process"
python -c "
import numpy as np
a = np.ones(44 * (1 << 27), dtype=np.float64); print(a[::1<<20].sum())
"
cat /sys/devices/system/node/node*/meminfo 2>/dev/null | grep -E "MemFree|FilePages"
python tools/pcie_probe.py
} >> $out 2>&1
