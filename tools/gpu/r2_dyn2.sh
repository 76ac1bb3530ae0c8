set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
./tools/probes/lat_probe
timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider > gpurun_out/r2_pytest_dyn2.log 2>&1; echo "pytest dyn exit $?"
tail -n 2 gpurun_out/r2_pytest_dyn2.log
for i in 1 2; do
HF_STATIC_TILES=1 timeout 600 python tools/time_variants.py 2 > gpurun_out/r2_tv2_static_$i.jsonl 2>&1
timeout 600 python tools/time_variants.py 2 > gpurun_out/r2_tv2_dyn_$i.jsonl 2>&1
HF_STATIC_TILES=1 HF_APPLY=chain timeout 600 python tools/time_variants.py 2 --strategies=tensor4 > gpurun_out/r2_tv2_static_chain_$i.jsonl 2>&1
HF_APPLY=chain timeout 600 python tools/time_variants.py 2 --strategies=tensor4 > gpurun_out/r2_tv2_dyn_chain_$i.jsonl 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
done
