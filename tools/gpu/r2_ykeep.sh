# A/B: k_cheb stores y_next (the next apply's initialisation) with the evict-last L2 policy.
cd $GRAFT_REPO_ROOT; O=gpurun_out/ykeep; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2 3; do for v in base ykeep; do
  L=$P/libhf_$v.so; [ $v = base ] && L=$P/libhf.so
  timeout 300 env HF_LIB=$L python tools/smoother_time.py 32 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
  timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4 /" >> $O/ab.log
  timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4t2 /" >> $O/ab.log
done; done
cat $O/ab.log
