# Hybrid (static + tail queue) tile schedule: parity, then A/B against the base build and
# the static schedule inside one call; per-warp timelines.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/hyb
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "not config5" 2>&1 | tail -n 3
for rep in 1 2 3; do
  for arm in base d0 d1 d2 d3; do
    case $arm in
      base) E="HF_LIB=$PWD/abtmp/libhf_base.so";;
      d0) E="HF_DYN_ROUNDS=0";;
      d1) E="HF_DYN_ROUNDS=1";;
      d2) E="HF_DYN_ROUNDS=2";;
      d3) E="HF_DYN_ROUNDS=3";;
    esac
    env $E timeout 300 python tools/time_variants.py ${CFGS:-2 3} | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn > gpurun_out/hyb/ab.log
python - <<'PY'
import json, numpy as np
from collections import defaultdict
d=defaultdict(list)
for line in open('gpurun_out/hyb/ab.log'):
    arm,_,js=line.strip().partition(' ')
    if not js.startswith('{'): continue
    r=json.loads(js); d[(r['cfg'],r['strategy'],arm)].append((r['b2b_us'],r['clean_flushed_us']))
arms=('base','d0','d1','d2','d3')
for c,s in sorted({(c,s) for c,s,_ in d}):
    print(f"cfg{c} {s:8s}", " | ".join(f"{a} {np.median(np.array(d[(c,s,a)])[:,0]):6.2f}/{np.median(np.array(d[(c,s,a)])[:,1]):6.2f}" for a in arms if (c,s,a) in d))
PY
for D in 0 2; do for v in "tensor4 2" "tensor2 2"; do
  HF_DYN_ROUNDS=$D HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py $v | sed "s/^/D$D /"
  set -- $v; mv gpurun_out/timeline_$1_$2.npy gpurun_out/hyb/timeline_$1_$2_D$D.npy
done; done 2>&1 | grep -v Warn | tee gpurun_out/hyb/timeline.log
