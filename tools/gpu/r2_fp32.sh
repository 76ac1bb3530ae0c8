cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/fp32
echo "== standalone prof_cg fp32 / fp64 (new lib)"
HF_COARSE_PRECISION=fp32 timeout 600 python tools/prof_cg.py 4 5 2>&1 | grep -v Warn | head -3 | cut -c1-600
HF_COARSE_PRECISION=fp64 timeout 600 python tools/prof_cg.py 4 5 2>&1 | grep -v Warn | head -1 | cut -c1-300
echo "== standalone prof_cg fp32 (old lib c74bd84)"
HF_LIB=$PWD/paper_1904_13131_b200/libhf_old.so HF_COARSE_PRECISION=fp32 timeout 600 python tools/prof_cg.py 4 5 2>&1 | grep -v Warn | head -1 | cut -c1-300
echo "== bench order"
timeout 900 python - <<'PY'
import sys, json
sys.argv=['bench.py']
import bench
print('fp64', json.dumps(bench._newton_iteration()))
print('fp32', json.dumps(bench._newton_iteration('fp32')))
print('fp32 again', json.dumps(bench._newton_iteration('fp32')))
PY
