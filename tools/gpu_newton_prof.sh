cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python tools/prof_newton.py 4 2 tensor4 > gpurun_out/pn_t4.log 2>&1
timeout 300 python tools/prof_newton.py 4 1 tensor2 > gpurun_out/pn_t2.log 2>&1
timeout 300 python tools/prof_cg.py 4 5 tensor4 > gpurun_out/pcg_t4.log 2>&1
timeout 300 python tools/prof_cg.py 4 5 tensor2 > gpurun_out/pcg_t2.log 2>&1
timeout 300 python tools/prof_cg.py 4 5 scalar > gpurun_out/pcg_sc.log 2>&1
tail -n 30 gpurun_out/pn_*.log
