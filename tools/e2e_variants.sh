#!/bin/bash
# e2e step time per forced host-pipeline variant (HF_E2E_ORDER=0..3) and the host-side split
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/e2e_variants.log
for v in 0 1 2 3; do
  HF_E2E_ORDER=$v timeout 120 python tools/e2e_steps.py 2>&1 | tail -n 4 | sed "s/^/order=$v /" >> gpurun_out/e2e_variants.log
done
timeout 120 python tools/e2e_host_overhead.py >> gpurun_out/e2e_variants.log 2>&1
cat gpurun_out/e2e_variants.log
