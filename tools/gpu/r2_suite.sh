set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,memory.total --format=csv
free -g | head -2; nproc
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest exit $?"
tail -5 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench exit $?"
tail -c 3000 gpurun_out/r2_bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1; echo "ref exit $?"
HF_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-extra > gpurun_out/r2_bench_n2_gloo.json 2> gpurun_out/r2_bench_n2_gloo.err; echo "n2 exit $?"
tail -c 2000 gpurun_out/r2_bench_n2_gloo.err
