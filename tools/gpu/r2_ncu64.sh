# ncu --set full of the tensor4 / tensor2 apply at 64^3 Q2 (config 4's fine level)
cd $GRAFT_REPO_ROOT; O=gpurun_out/ncu64; mkdir -p $O
for s in tensor4 tensor2; do
  timeout 600 python tools/prof_variant.py $s 4 4 > $O/plain_$s.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o $O/ncu_${s}_64 python tools/prof_variant.py $s 4 4 > $O/ncu_$s.log 2>&1; echo "ncu $s rc=$?"
done
cat $O/plain_tensor4.log
