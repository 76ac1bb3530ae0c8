# A/B of the L2 residency hints (HF_L2HINT 0 / 1 / 2), one call, interleaved.
cd $GRAFT_REPO_ROOT; O=gpurun_out/l2hint; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2; do
  for v in base l2h1 l2h2; do
    L=$P/libhf_$v.so; [ $v = base ] && L=$P/libhf.so
    for s in tensor4 tensor2 scalar; do for cfg in 2 3; do
      timeout 120 env HF_LIB=$L python tools/time_apply.py $s $cfg | sed "s/^/$v /" >> $O/ab.log 2>&1
    done; done
    timeout 300 env HF_LIB=$L python tools/smoother_time.py 32 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
    timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 2>/dev/null | head -4 | cut -c1-220 | sed "s/^/$v cg4 /" >> $O/ab.log
    timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -4 | cut -c1-220 | sed "s/^/$v cg4t2 /" >> $O/ab.log
  done
done
cat $O/ab.log
