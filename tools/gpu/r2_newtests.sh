cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_verify.py tests/test_gpu_refside.py -q -p no:cacheprovider 2>&1 | tail -n 40
