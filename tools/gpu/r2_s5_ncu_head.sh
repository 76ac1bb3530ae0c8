set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/s5n; mkdir -p $O
timeout 600 python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > $O/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-extra --no-cpu > $O/ncu_launch.log 2>&1; echo "launch list rc=$?"
for v in "tensor4 2" "tensor4 3"; do
  set -- $v
  timeout 300 python tools/prof_variant.py $1 $2 4 > $O/plain_$1_$2.log 2>&1 && \
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_apply_line --launch-skip 2 --launch-count 1 \
    -f -o $O/ncu_$1_$2 python tools/prof_variant.py $1 $2 4 > $O/ncu_$1_$2.log 2>&1; echo "ncu $v rc=$?"
done
