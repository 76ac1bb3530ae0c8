cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/bench2
for i in 1 2; do timeout 1200 python bench.py --no-cpu > gpurun_out/bench2/bench_$i.json 2> gpurun_out/bench2/bench_$i.err; echo "rc=$?"; done
