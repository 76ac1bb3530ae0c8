cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for fb in 8 3 2; do
  HF_FILL_BLOCKS=$fb timeout 300 python tools/time_variants.py 2 --strategies=tensor4,tensor2 | sed "s/^/fb$fb /"
done
done 2>&1 | grep -v Warn | tee gpurun_out/ab_fill.log
for fb in 8 3; do
  HF_FILL_BLOCKS=$fb HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py tensor4 2
done
