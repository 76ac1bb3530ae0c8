cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "every_instantiated" 2>&1 | tail -n 40
