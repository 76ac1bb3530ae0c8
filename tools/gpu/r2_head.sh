# HEAD check: GPU suite, smoke, default bench.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/head
nvidia-smi -L > gpurun_out/head/smi.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/head/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/head/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/head/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/head/smoke.log
timeout 900 python bench.py > gpurun_out/head/bench.json 2> gpurun_out/head/bench.err; echo "bench rc=$?"
tail -n 3 gpurun_out/head/pytest_gpu.log gpurun_out/head/smoke.log
