# Plane-parallel tensor2 kernel (3D Q2): parity, then A/B against the base build.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/plane
timeout 1200 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_mixed.py -x -q -p no:cacheprovider -k "not config5" 2>&1 | tail -n 15
HF_LIB=$PWD/paper_1904_13131_b200/libhf_g3.so timeout 1200 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -n 3
for rep in 1 2 3; do
  for arm in base new g3; do
    case $arm in
      base) E="HF_LIB=$PWD/abtmp/libhf_base.so";;
      new) E="HF_DYN_ROUNDS=0";;
      g3) E="HF_DYN_ROUNDS=0 HF_LIB=$PWD/paper_1904_13131_b200/libhf_g3.so";;
    esac
    env $E timeout 300 python tools/time_variants.py 2 --strategies=${STRATS:-tensor2} | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn | tee gpurun_out/plane/ab.log
timeout 300 python tools/prof_variant.py tensor2 2 4 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_apply_ --launch-skip 2 --launch-count 1 \
    -f -o gpurun_out/plane/ncu_plane_t2 python tools/prof_variant.py tensor2 2 4 > gpurun_out/plane/ncu.log 2>&1; echo "ncu rc=$?"
