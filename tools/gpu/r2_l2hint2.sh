# A/B: evict-last x/y (libhf_l2xy.so) and reverse sweeps on large levels (HF_REVERSE=1) against the evict-first build.
cd $GRAFT_REPO_ROOT; O=gpurun_out/l2hint2; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2 3; do
  for v in base l2xy rev; do
    L=$P/libhf.so; R=0
    [ $v = l2xy ] && L=$P/libhf_l2xy.so
    [ $v = rev ] && R=1
    if [ $v != rev ]; then
      for s in tensor4 tensor2; do for cfg in 2 3; do
        timeout 120 env HF_LIB=$L python tools/time_apply.py $s $cfg | sed "s/^/$v /" >> $O/ab.log 2>&1
      done; done
    fi
    timeout 300 env HF_LIB=$L HF_REVERSE=$R python tools/smoother_time.py 32 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
    timeout 300 env HF_LIB=$L HF_REVERSE=$R python tools/prof_cg.py 4 5 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4 /" >> $O/ab.log
    timeout 300 env HF_LIB=$L HF_REVERSE=$R python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4t2 /" >> $O/ab.log
  done
done
cat $O/ab.log
