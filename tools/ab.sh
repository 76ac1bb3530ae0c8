#!/bin/bash
# A/B timing of apply variants selected by environment knobs
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/ab.log
for cfg in 2 3; do for s in tensor4 tensor2; do
  for env in "HF_PDL=0" "HF_PDL=1"; do
    env $env timeout 120 python tools/time_apply.py $s $cfg >> gpurun_out/ab.log 2>&1
  done
done; done
cat gpurun_out/ab.log
