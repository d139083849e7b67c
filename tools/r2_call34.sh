#!/bin/bash
# e2e timeline at the bench workload + PCIe probe
mkdir -p gpurun_out
timeout 600 python tools/e2e_timeline.py 27 16 > gpurun_out/c34_tl16.txt 2>&1
timeout 600 python tools/e2e_timeline.py 27 64 > gpurun_out/c34_tl64.txt 2>&1
timeout 300 python tools/pcie_probe.py > gpurun_out/c34_pcie.txt 2>&1
echo done
