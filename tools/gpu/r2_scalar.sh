cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for n in base s12u s10u s8u s10f; do
  if [ $n = base ]; then L=""; else L="HF_LIB=$PWD/paper_1904_13131_b200/libhf_$n.so"; fi
  env $L timeout 300 python tools/time_variants.py 2 3 --strategies=scalar | sed "s/^/$n /"
done
done 2>&1 | grep -v Warn | tee gpurun_out/ab_scalar.log
