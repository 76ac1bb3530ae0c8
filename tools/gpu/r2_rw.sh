cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for n in base rw4 rw5; do
  if [ $n = base ]; then L=""; else L="HF_LIB=$PWD/paper_1904_13131_b200/libhf_$n.so"; fi
  env $L timeout 300 python tools/time_variants.py 3 --strategies=tensor4 | sed "s/^/$n /"
done
for n in base ss12 ss10 ss8; do
  if [ $n = base ]; then L=""; else L="HF_LIB=$PWD/paper_1904_13131_b200/libhf_$n.so"; fi
  env $L timeout 300 python tools/time_variants.py 2 --strategies=scalar | sed "s/^/$n /"
done
done 2>&1 | grep -v Warn | cut -c1-170 | tee gpurun_out/ab_rw_scalar.log
