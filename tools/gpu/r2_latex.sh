# A/B: chained apply (fill = 2) issues its first TMA chunks before waiting for the primary (default) vs waits first (libhf_earlyx.so).
cd $GRAFT_REPO_ROOT; O=gpurun_out/latex; mkdir -p $O; : > $O/ab.log; : > $O/ab2.log
P=$PWD/paper_1904_13131_b200
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_verify.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for rep in 1 2 3; do for v in early late; do
  L=$P/libhf.so; [ $v = early ] && L=$P/libhf_earlyx.so
  timeout 300 env HF_LIB=$L python tools/smoother_time.py 8 16 32 64 2>&1 | sed "s/^/$v /" >> $O/ab.log
done; done
for v in early late early late; do
  L=$P/libhf.so; [ $v = early ] && L=$P/libhf_earlyx.so
  timeout 900 env HF_LIB=$L python bench.py --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python tools/bench_brief.py $O/bench_$v.json | grep -E "headline|newton |cfg1|newton_solve" | sed "s/^/$v /" >> $O/ab2.log
done
cat $O/ab.log $O/ab2.log
