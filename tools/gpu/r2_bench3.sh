cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/bench3
for i in 1 2 3; do HF_GRAPH_TIMING=1 timeout 1200 python bench.py --no-cpu > gpurun_out/bench3/bench_$i.out 2> gpurun_out/bench3/bench_$i.err; echo "rc=$?"; done
