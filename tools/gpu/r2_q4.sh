cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -n 2
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "full_size_vs_oracle and 3 or numpy_apply" 2>&1 | tail -n 2
CFGS="3 2" bash tools/gpu/ab2.sh > /dev/null
python tools/ab_summary.py gpurun_out/ab2.log
