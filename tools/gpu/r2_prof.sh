set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_refside.py -x -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu_b.log 2>&1; echo "pytest exit $?"
tail -3 gpurun_out/r2_pytest_gpu_b.log
timeout 600 python tools/time_variants.py 2 3 > gpurun_out/r2_time_variants.jsonl 2>&1; echo "tv exit $?"
cat gpurun_out/r2_time_variants.jsonl
for v in "tensor4 2" "tensor2 2" "scalar 2" "tensor4 3" "tensor2 3"; do
  set -- $v
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/r2_ncu_$1_$2 python tools/prof_variant.py $1 $2 4 > gpurun_out/r2_ncu_$1_$2.log 2>&1; echo "ncu $v exit $?"
done
ls -la gpurun_out
