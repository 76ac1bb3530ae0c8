cd $GRAFT_REPO_ROOT; O=gpurun_out/pw; mkdir -p $O; : > $O/ab2.log
P=$PWD/paper_1904_13131_b200
for v in base pw2 base pw2 base pw2; do
  L=$P/libhf_$v.so; [ $v = base ] && L=$P/libhf.so
  timeout 900 env HF_LIB=$L python bench.py --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python tools/bench_brief.py $O/bench_$v.json | grep -E "headline|^variants |cfg3|newton |cfg1|cfg5" | sed "s/^/$v /" >> $O/ab2.log
done
cat $O/ab2.log
