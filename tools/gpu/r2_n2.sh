cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/n2
for n in 2 4; do
  s=$(date +%s)
  HF_BENCH_BACKEND=gloo timeout 1500 python bench.py --gpus $n > gpurun_out/n2/bench_n$n.json 2> gpurun_out/n2/bench_n$n.err; echo "n=$n rc=$? secs=$(( $(date +%s) - s ))"
done
