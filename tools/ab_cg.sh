cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out; : > gpurun_out/abcg.log
for rep in 1 2; do for cfg in 1 4; do
  timeout 200 env HF_LIB=$PWD/abtmp/libhf_prev.so python tools/prof_cg.py $cfg 5 2>/dev/null | head -1 | sed "s/^/prev $cfg /" >> gpurun_out/abcg.log
  timeout 200 python tools/prof_cg.py $cfg 5 2>/dev/null | head -1 | sed "s/^/new  $cfg /" >> gpurun_out/abcg.log
done; done
cat gpurun_out/abcg.log
