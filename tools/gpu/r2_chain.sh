set -x
cd $GRAFT_REPO_ROOT
HF_APPLY=chain timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_refside.py tests/test_gpu_mg.py -x -q -p no:cacheprovider > gpurun_out/r2_pytest_chain.log 2>&1; echo "pytest chain exit $?"
tail -3 gpurun_out/r2_pytest_chain.log
HF_APPLY=chain timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "full_size_vs_oracle" > gpurun_out/r2_pytest_chain_fs.log 2>&1; echo "pytest chain fs exit $?"
tail -3 gpurun_out/r2_pytest_chain_fs.log
for i in 1 2; do
HF_APPLY=line timeout 600 python tools/time_variants.py 2 > gpurun_out/r2_tv_line_$i.jsonl 2>&1
HF_APPLY=chain timeout 600 python tools/time_variants.py 2 > gpurun_out/r2_tv_chain_$i.jsonl 2>&1
done
cat gpurun_out/r2_tv_*.jsonl
