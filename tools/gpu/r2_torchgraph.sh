cd $GRAFT_REPO_ROOT
HF_GRAPH=torch timeout 1500 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_refside.py -q -p no:cacheprovider -k "not updated_in_place" 2>&1 | tail -n 3
