# A/B: tensor2 at 3D Q2 with 13 / 14 warps per block (128 registers, small spills) vs 12 (153 registers).
cd $GRAFT_REPO_ROOT; O=gpurun_out/t2w; mkdir -p $O; : > $O/ab.log
P=$PWD/paper_1904_13131_b200
for rep in 1 2 3; do for v in base t2w13 t2w14; do
  L=$P/libhf_$v.so; [ $v = base ] && L=$P/libhf.so
  timeout 120 env HF_LIB=$L python tools/time_apply.py tensor2 2 | sed "s/^/$v /" >> $O/ab.log 2>&1
  timeout 300 env HF_LIB=$L python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/$v cg4t2 /" >> $O/ab.log
done; done
cat $O/ab.log
