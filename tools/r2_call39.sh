#!/bin/bash
mkdir -p gpurun_out
for v in "" "PRE_PROBE=1" "PRE_STEPS=23" "PRE_SMI=1 PRE_STEPS=23"; do
  echo "== $v" >> gpurun_out/c39.txt
  env $v timeout 300 python tools/e2e_repro.py >> gpurun_out/c39.txt 2>&1
done
echo done
