# A/B: three-term Chebyshev updates (HF_CHEB3=1, default) vs stored direction (0).
cd $GRAFT_REPO_ROOT; O=gpurun_out/cheb3; mkdir -p $O; : > $O/ab.log; : > $O/ab2.log
timeout 1500 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_refside.py tests/test_gpu_verify.py tests/test_gpu_distributed.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for rep in 1 2 3; do for v in 0 1; do
  timeout 300 env HF_CHEB3=$v python tools/smoother_time.py 8 16 32 64 2>&1 | sed "s/^/cheb3_$v /" >> $O/ab.log
  timeout 300 env HF_CHEB3=$v python tools/prof_cg.py 4 5 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/cheb3_$v cg4 /" >> $O/ab.log
  timeout 300 env HF_CHEB3=$v python tools/prof_cg.py 4 5 tensor2 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/cheb3_$v cg4t2 /" >> $O/ab.log
done; done
for v in 0 1 0 1; do
  timeout 900 env HF_CHEB3=$v python bench.py --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python tools/bench_brief.py $O/bench_$v.json | grep -E "newton|cfg1|cfg5" | sed "s/^/cheb3_$v /" >> $O/ab2.log
done
cat $O/ab.log $O/ab2.log
