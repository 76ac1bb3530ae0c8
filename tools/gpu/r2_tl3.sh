cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/tl3
for v in "tensor4 3" "tensor2 3" "scalar 3" "scalar 2"; do
  HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py $v
done 2>&1 | grep -v Warn | tee gpurun_out/tl3/timeline.log
mv gpurun_out/timeline_*.npy gpurun_out/tl3/
