# A/B: k_cheb's single-use operands (b, inv_d, d, mask) as streaming accesses, on top of evict-first + reverse + evict-last y.
cd $GRAFT_REPO_ROOT; O=gpurun_out/l2hint4; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2 3; do
  for v in base veccs; do
    L=$P/libhf.so
    [ $v = veccs ] && L=$P/libhf_veccs.so
    timeout 300 env HF_LIB=$L python tools/smoother_time.py 32 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
    timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4 /" >> $O/ab.log
    timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4t2 /" >> $O/ab.log
  done
done
cat $O/ab.log
