# Final round-2 evidence at HEAD: GPU suite, smoke, bench (both arms), launch list, ncu of the headline kernel.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
nvidia-smi -L > gpurun_out/final2/smi.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final2/smoke.log
timeout 1200 python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final2/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > gpurun_out/final2/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final2/launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > gpurun_out/final2/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/final2/ncu_tensor4_2 python tools/prof_variant.py tensor4 2 4 > gpurun_out/final2/ncu_tensor4_2.log 2>&1; echo "ncu rc=$?"
tail -n 3 gpurun_out/final2/pytest_gpu.log gpurun_out/final2/smoke.log
for v in "tensor2 2" "scalar 2" "tensor4 3" "tensor2 3" "scalar 3"; do
  set -- $v
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/final2/ncu_$1_$2 python tools/prof_variant.py $1 $2 4 > gpurun_out/final2/ncu_$1_$2.log 2>&1; echo "ncu $v rc=$?"
done
HF_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-newton > gpurun_out/final2/bench_n2_gloo.json 2> gpurun_out/final2/bench_n2_gloo.err; echo "n2 rc=$?"
