#!/bin/bash
# Session 4: host-side diagnosis of a box whose e2e leg ran at 406/s instead of 517/s (NUMA / PCIe / CPU)
OUT=gpurun_out/s4k
mkdir -p $OUT
{
nvidia-smi topo -m
echo; nvidia-smi --query-gpu=pci.bus_id,pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max,pcie.link.width.max --format=csv
BUS=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//')
echo "bus $BUS"; cat /sys/bus/pci/devices/0000$BUS/numa_node 2>/dev/null; cat /sys/bus/pci/devices/0000$BUS/local_cpulist 2>/dev/null
echo; lscpu | head -30
echo; cat /sys/devices/system/node/online 2>/dev/null; for n in /sys/devices/system/node/node*; do echo $n $(cat $n/cpulist); done
echo; python -c "import os; print('affinity', sorted(os.sched_getaffinity(0)))"
echo; cat /proc/loadavg; nproc
echo; uptime
} > $OUT/host.txt 2>&1
timeout 300 python tools/pcie_probe.py > $OUT/pcie_probe.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_cfg2.jsonl 2> $OUT/bench.err
ls -la $OUT
