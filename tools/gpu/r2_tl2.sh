cd $GRAFT_REPO_ROOT
for v in "tensor4 2" "tensor2 2"; do
  HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py $v
done
