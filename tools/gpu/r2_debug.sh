cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/debug
HF_LIB=$PWD/paper_1904_13131_b200/libhf_debug.so timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/debug/pytest_gpu_debug_bounds.log 2>&1; echo "rc=$?" >> gpurun_out/debug/pytest_gpu_debug_bounds.log
tail -3 gpurun_out/debug/pytest_gpu_debug_bounds.log
