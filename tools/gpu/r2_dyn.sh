set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_distributed.py -x -q -p no:cacheprovider > gpurun_out/r2_pytest_dyn.log 2>&1; echo "pytest dyn exit $?"
tail -n 3 gpurun_out/r2_pytest_dyn.log
HF_APPLY=chain timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_mg.py -x -q -p no:cacheprovider > gpurun_out/r2_pytest_dyn_chain.log 2>&1; echo "pytest dyn chain exit $?"
tail -n 3 gpurun_out/r2_pytest_dyn_chain.log
for i in 1 2; do
HF_STATIC_TILES=1 HF_APPLY=line timeout 600 python tools/time_variants.py 2 3 > gpurun_out/r2_tv_static_line_$i.jsonl 2>&1
HF_APPLY=line timeout 600 python tools/time_variants.py 2 3 > gpurun_out/r2_tv_dyn_line_$i.jsonl 2>&1
HF_APPLY=chain timeout 600 python tools/time_variants.py 2 > gpurun_out/r2_tv_dyn_chain_$i.jsonl 2>&1
done
for f in gpurun_out/r2_tv_*_line_1.jsonl gpurun_out/r2_tv_dyn_chain_1.jsonl; do echo $f; cut -c1-200 $f; done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/r2_ncu_dyn_tensor4_2 python tools/prof_variant.py tensor4 2 4 > /dev/null 2>&1; echo "ncu exit $?"
