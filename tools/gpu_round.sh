#!/bin/bash
# One GPU round: parity tests, smoke, bench (both arms), launch list, ncu of the apply kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > gpurun_out/ncu_launch.log 2>&1
timeout 300 python tools/prof_apply.py tensor4 2 5 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_apply -s 2 -c 1 -o gpurun_out/prof_t4 -f python tools/prof_apply.py tensor4 2 5 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/t_gpu.log gpurun_out/smoke.log gpurun_out/bench.log gpurun_out/bench_ref.log gpurun_out/ncu_full.log | cut -c1-400
HF_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench_n2_gloo.log 2>&1; echo "n2 rc=$?" >> gpurun_out/bench_n2_gloo.log
