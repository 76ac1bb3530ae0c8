cd $GRAFT_REPO_ROOT; O=gpurun_out/s5q; mkdir -p $O
timeout 600 python tools/prof_setup.py 4 > $O/prof_setup_cfg4.log 2>&1
timeout 900 python tools/prof_cg.py 5 3 > $O/prof_cg_cfg5.log 2>&1
timeout 600 python tools/prof_cg.py 4 5 > $O/prof_cg_cfg4.log 2>&1
tail -n 30 $O/prof_setup_cfg4.log; cut -c1-200 $O/prof_cg_cfg5.log | head -30
