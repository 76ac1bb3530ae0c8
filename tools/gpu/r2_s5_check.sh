# Session-5 check at HEAD after the container was re-created: GPU suite, smoke, bench (both arms).
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5; mkdir -p $O
nvidia-smi -L > $O/smi.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2>&1; echo "ref rc=$?"
tail -n 3 $O/pytest_gpu.log $O/smoke.log
