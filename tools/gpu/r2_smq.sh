set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_mg.py -x -q -p no:cacheprovider 2>&1 | tail -n 2
HF_APPLY=chain timeout 600 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -n 2
CFGS="2 3" bash tools/gpu/ab2.sh > /dev/null
python tools/ab_summary.py gpurun_out/ab2.log
for v in "tensor4 2" "tensor2 2" "scalar 2"; do
  HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py $v
done
