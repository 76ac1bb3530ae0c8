cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_mg.py -q -p no:cacheprovider -k "updated_in_place or vcycle" 2>&1 | tail -n 15
