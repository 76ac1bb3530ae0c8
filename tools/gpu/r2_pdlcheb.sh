# A/B: the Chebyshev update as the cell kernel's programmatic dependent (HF_PDL_CHEB=1, default) vs a plain launch (0).
cd $GRAFT_REPO_ROOT; O=gpurun_out/pdlcheb; mkdir -p $O; : > $O/ab.log
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_verify.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for rep in 1 2 3; do for v in 0 1; do
  timeout 300 env HF_PDL_CHEB=$v python tools/smoother_time.py 8 16 32 64 2>&1 | sed "s/^/pdl$v /" >> $O/ab.log
  timeout 300 env HF_PDL_CHEB=$v python tools/prof_cg.py 4 5 2>/dev/null | head -3 | cut -c1-220 | sed "s/^/pdl$v cg4 /" >> $O/ab.log
done; done
for v in 0 1; do
  timeout 900 env HF_PDL_CHEB=$v python bench.py --no-cpu > $O/bench_pdl$v.json 2> $O/bench_pdl$v.err
done
cat $O/ab.log
