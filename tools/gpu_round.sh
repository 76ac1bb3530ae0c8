#!/bin/bash
# One GPU round: parity tests, smoke, bench, launch list, ncu of the top kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/prof_apply.py tensor4 2 5 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_apply.py tensor4 2 5 > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_apply.py tensor4 2 5 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_t4 -f python tools/prof_apply.py tensor4 2 5 > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/t_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/ncu_full.log
