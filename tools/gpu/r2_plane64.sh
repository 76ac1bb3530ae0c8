set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/plane
for rep in 1 2; do
  for arm in base new; do
    case $arm in
      base) E="HF_LIB=$PWD/abtmp/libhf_base.so";;
      new) E="HF_DYN_ROUNDS=0";;
    esac
    env $E timeout 300 python tools/time_apply.py tensor2 4 | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn | tee gpurun_out/plane/ab64.log
