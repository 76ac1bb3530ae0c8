# Final evidence of the round at HEAD: GPU suite (normal and bounds-checking build), smoke, bench (both arms),
# launch list, ncu of every variant, the N = 2 functional run over gloo on one GPU.
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5f; mkdir -p $O
nvidia-smi -L > $O/smi.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 600 python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > $O/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
for v in "tensor4 2" "tensor2 2" "scalar 2" "tensor4 3" "tensor2 3" "scalar 3"; do
  set -- $v
  timeout 300 python tools/prof_variant.py $1 $2 4 > $O/plain_$1_$2.log 2>&1 && \
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o $O/ncu_$1_$2 python tools/prof_variant.py $1 $2 4 > $O/ncu_$1_$2.log 2>&1; echo "ncu $v rc=$?"
done
HF_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-newton > $O/bench_n2_gloo.json 2> $O/bench_n2_gloo.err; echo "n2 rc=$?"
if [ -f paper_1904_13131_b200/libhf_debug.so ]; then
  HF_LIB=$PWD/paper_1904_13131_b200/libhf_debug.so timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu_debug_bounds.log 2>&1; echo "debug pytest rc=$?" >> $O/pytest_gpu_debug_bounds.log
fi
tail -n 3 $O/pytest_gpu.log $O/smoke.log $O/pytest_gpu_debug_bounds.log
