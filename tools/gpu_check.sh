cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.log 2>&1
timeout 900 python -m pytest tests/test_gpu_ops.py -q --maxfail=30 > gpurun_out/t_ops.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_mg.py -q --maxfail=10 > gpurun_out/t_mg.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
tail -3 gpurun_out/t_ops.log gpurun_out/t_mg.log gpurun_out/smoke.log gpurun_out/bench.log
