cd $GRAFT_REPO_ROOT
for arm in line chain; do
  HF_APPLY=$arm timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/r2_ncu_${arm}_tensor2_2 python tools/prof_variant.py tensor2 2 4 > /dev/null 2>&1; echo "ncu $arm exit $?"
done
