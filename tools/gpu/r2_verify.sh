set -x
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu_full.log 2>&1; echo "pytest exit $?"
tail -n 5 gpurun_out/r2_pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()"
for rep in 1 2 3; do
  HF_APPLY=line timeout 300 python tools/time_variants.py 2 --strategies=tensor4 | sed "s/^/line /"
  HF_APPLY=chain timeout 300 python tools/time_variants.py 2 --strategies=tensor4 | sed "s/^/chain /"
done 2>&1 | grep -v Warn | cut -c1-160
timeout 300 python tools/time_variants.py 3 | cut -c1-200
