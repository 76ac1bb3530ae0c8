#!/bin/bash
# A/B of small-level latency and the CG iteration: in-tree libhf.so vs abtmp/libhf_prev.so
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/ab_small.log
for rep in 1 2; do
  HF_LIB=$PWD/abtmp/libhf_prev.so timeout 200 python tools/small_latency.py 4 8 16 | sed 's/^/prev /' >> gpurun_out/ab_small.log 2>&1
  timeout 200 python tools/small_latency.py 4 8 16 | sed 's/^/new  /' >> gpurun_out/ab_small.log 2>&1
done
HF_LIB=$PWD/abtmp/libhf_prev.so timeout 300 python tools/prof_cg.py 4 5 2>/dev/null | head -1 | sed 's/^/prev /' >> gpurun_out/ab_small.log
timeout 300 python tools/prof_cg.py 4 5 2>/dev/null | head -1 | sed 's/^/new  /' >> gpurun_out/ab_small.log
cat gpurun_out/ab_small.log
