cd $GRAFT_REPO_ROOT; O=gpurun_out/cgfused; mkdir -p $O; : > $O/ab.log
for v in 0 1 0 1 0 1; do
  timeout 900 env HF_CG_FUSED=$v python bench.py --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python tools/bench_brief.py $O/bench_$v.json | grep -E "newton |newton_solve|cfg1" | sed "s/^/fused$v /" >> $O/ab.log
done
cat $O/ab.log
