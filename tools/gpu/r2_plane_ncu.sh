set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/plane
timeout 300 python tools/prof_variant.py tensor2 2 4 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_ --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/plane/ncu_plane_t2 python tools/prof_variant.py tensor2 2 4 > gpurun_out/plane/ncu.log 2>&1; echo "ncu rc=$?"
