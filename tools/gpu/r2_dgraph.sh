cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_distributed.py -x -q -p no:cacheprovider -k graph 2>&1 | tail -n 30
