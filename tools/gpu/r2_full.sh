set -x
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu_full.log 2>&1; echo "pytest exit $?"
tail -n 5 gpurun_out/r2_pytest_gpu_full.log
timeout 900 python bench.py > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench exit $?"
HF_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 4 --steps 5 --warmup 3 --no-extra > gpurun_out/r2_bench_n4_gloo.json 2> gpurun_out/r2_bench_n4_gloo.err; echo "n4 exit $?"
tail -c 1500 gpurun_out/r2_bench_n4_gloo.err
