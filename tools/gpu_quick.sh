#!/bin/bash
# Quick GPU iteration: parity tests + bench (with and without L2 prefetch) + ncu of the apply.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu.log
timeout 240 python bench.py --steps 20 --warmup 5 --no-newton --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
HF_L2_PREFETCH=0 timeout 240 python bench.py --steps 20 --warmup 5 --no-newton --no-cpu > gpurun_out/bench_nopf.log 2>&1
if [ -n "$PROF" ]; then
timeout 300 python tools/prof_apply.py $PROF > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_apply -f python tools/prof_apply.py $PROF > gpurun_out/ncu_full.log 2>&1
fi
tail -n 3 gpurun_out/t_gpu.log; tail -n 2 gpurun_out/bench.log | cut -c1-1500
