# GPU suite + smoke + bench at the working tree.
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5b; mkdir -p $O
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"
tail -n 3 $O/pytest_gpu.log $O/smoke.log
