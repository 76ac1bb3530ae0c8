# A/B of the in-tree libhf.so against abtmp/libhf_base.so on one box, interleaved:
#   CFGS="2 3" STRATS="tensor4,tensor2,scalar" bash tools/gpu/ab2.sh
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2 3; do
  for cfg in ${CFGS:-2}; do
    HF_LIB=$PWD/abtmp/libhf_base.so timeout 300 python tools/time_variants.py $cfg --strategies=${STRATS:-tensor4,tensor2,scalar} | sed 's/^/base /'
    timeout 300 python tools/time_variants.py $cfg --strategies=${STRATS:-tensor4,tensor2,scalar} | sed 's/^/new  /'
  done
done 2>&1 | grep -v Warn | tee gpurun_out/ab2.log
