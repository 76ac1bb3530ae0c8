#!/bin/bash
# A/B of the graph-replayed Lanczos step (HF_LANCZOS_GRAPH=0/1): GMG setup at configs 4 and 1, same box, interleaved
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/ab_lanczos.log
for rep in 1 2; do for g in 0 1; do
  HF_LANCZOS_GRAPH=$g timeout 300 python tools/prof_setup.py 4 2>&1 | tail -n 7 | sed "s/^/g=$g cfg4 /" >> gpurun_out/ab_lanczos.log
  HF_LANCZOS_GRAPH=$g timeout 300 python tools/prof_setup.py 1 2>&1 | tail -n 5 | sed "s/^/g=$g cfg1 /" >> gpurun_out/ab_lanczos.log
done; done
cat gpurun_out/ab_lanczos.log
