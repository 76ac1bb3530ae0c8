#!/bin/bash
# A/B timing: the in-tree libhf.so vs abtmp/libhf_prev.so (previous build), same box, interleaved
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/ab.log
for rep in 1 2; do for cfg in ${CFGS:-2 3}; do for s in ${STRATS:-tensor4 tensor2 scalar}; do
  timeout 120 env HF_LIB=$PWD/abtmp/libhf_prev.so python tools/time_apply.py $s $cfg | sed 's/^/prev /' >> gpurun_out/ab.log 2>&1
  timeout 120 python tools/time_apply.py $s $cfg | sed 's/^/new  /' >> gpurun_out/ab.log 2>&1
done; done; done
cat gpurun_out/ab.log
