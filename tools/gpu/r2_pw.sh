# A/B: per-point mbarrier waits in every tile (pw1) / in the first tile only (pw2) vs one wait per tile.
cd $GRAFT_REPO_ROOT; O=gpurun_out/pw; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2 3; do for v in base pw1 pw2; do
  L=$P/libhf_$v.so; [ $v = base ] && L=$P/libhf.so
  for s in tensor4 tensor2 scalar; do
    timeout 120 env HF_LIB=$L python tools/time_apply.py $s 2 | sed "s/^/$v /" >> $O/ab.log 2>&1
  done
  timeout 300 env HF_LIB=$L python tools/smoother_time.py 8 16 32 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
done; done
cat $O/ab.log
