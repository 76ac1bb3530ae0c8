# A/B: evict-last x only / y only / both, each with reverse sweeps on the large level, against evict-first + forward.
cd $GRAFT_REPO_ROOT; O=gpurun_out/l2hint3; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2; do
  for v in base rev l2x_rev l2y_rev l2xy_rev; do
    L=$P/libhf.so; R=1
    [ $v = base ] && R=0
    [ $v = l2x_rev ] && L=$P/libhf_l2x.so
    [ $v = l2y_rev ] && L=$P/libhf_l2y.so
    [ $v = l2xy_rev ] && L=$P/libhf_l2xy.so
    if [ $v != rev ]; then
      for s in tensor4 tensor2 scalar; do
        timeout 120 env HF_LIB=$L python tools/time_apply.py $s 2 | sed "s/^/$v /" >> $O/ab.log 2>&1
      done
    fi
    timeout 300 env HF_LIB=$L HF_REVERSE=$R python tools/smoother_time.py 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
    timeout 300 env HF_LIB=$L HF_REVERSE=$R python tools/prof_cg.py 4 5 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4 /" >> $O/ab.log
    timeout 300 env HF_LIB=$L HF_REVERSE=$R python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4t2 /" >> $O/ab.log
  done
done
cat $O/ab.log
