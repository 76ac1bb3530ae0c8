cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/graph
timeout 1500 python -m pytest tests/test_gpu_mg.py tests/test_gpu_mixed.py tests/test_gpu_refside.py tests/test_gpu_distributed.py -x -q -p no:cacheprovider 2>&1 | tail -n 5
timeout 900 python - <<'PY' 2>&1 | grep -v Warn
import sys, json, os
sys.argv=['bench.py']
import bench
for mode in ('native','torch','native'):
    os.environ['HF_GRAPH']=mode
    r=bench._newton_solve_cfg4()
    print(mode,'total_s',round(r['total_s'],3),'per-iteration wall',[x['wall_s'] for x in r['iterations']])
    n=bench._newton_iteration(); print(mode,'newton iteration runs', [round(x,4) for x in n['runs_s']], 'setup', round(n['setup_s'],4), 'cg/it', round(n['s_per_cg_iteration']*1e3,3))
PY
