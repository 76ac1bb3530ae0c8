# A/B: late release of the cell kernel's dependents; every level chained (HF_PDL_CHEB_MAX_DOFS huge) vs no chaining.
cd $GRAFT_REPO_ROOT; O=gpurun_out/pdlcheb2; mkdir -p $O; : > $O/ab.log
export HF_PDL_CHEB_MAX_DOFS=100000000000
timeout 900 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_verify.py tests/test_gpu_ops.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; tail -2 $O/pytest.log
for rep in 1 2 3; do for v in 0 1; do
  timeout 300 env HF_PDL_CHEB=$v python tools/smoother_time.py 8 16 32 64 2>&1 | sed "s/^/pdl$v /" >> $O/ab.log
done; done
for v in 0 1 0 1; do
  timeout 900 env HF_PDL_CHEB=$v python bench.py --no-cpu > $O/bench_pdl$v.json 2> $O/bench_pdl$v.err
  python tools/bench_brief.py $O/bench_pdl$v.json | grep -E "headline|newton |cfg1" | sed "s/^/pdl$v /" >> $O/ab2.log
done
cat $O/ab.log $O/ab2.log
