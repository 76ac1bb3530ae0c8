# A/B: fused Lanczos step (HF_LANCZOS_FUSED=1, default) vs the five separate vector kernels + fill (0).
cd $GRAFT_REPO_ROOT; O=gpurun_out/lanczos; mkdir -p $O; : > $O/ab.log
timeout 1500 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_refside.py tests/test_gpu_verify.py -m gpu -q -p no:cacheprovider -x > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for rep in 1 2 3; do for v in 0 1; do
  timeout 300 env HF_LANCZOS_FUSED=$v python tools/prof_gmg_build.py 2>/dev/null | grep -E "build_gmg_wall|k_lanczos|k_jacobi|k_fill|k_dot" | cut -c1-160 | sed "s/^/fused$v /" >> $O/ab.log
done; done
for v in 0 1 0 1; do
  timeout 900 env HF_LANCZOS_FUSED=$v python bench.py --no-cpu > $O/bench_$v.json 2> $O/bench_$v.err
  python tools/bench_brief.py $O/bench_$v.json | grep -E "newton |newton_solve|cfg1" | sed "s/^/fused$v /" >> $O/ab.log
done
cat $O/ab.log
