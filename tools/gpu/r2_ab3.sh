# A/B of the in-tree libhf.so against abtmp/libhf_base.so (same box, interleaved) after a quick parity run.
set -x
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab3
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_fullsize.py tests/test_gpu_mixed.py -x -q -p no:cacheprovider -k "not config5" 2>&1 | tail -n 3
for rep in 1 2 3; do
  for arm in base new; do
    case $arm in
      base) E="HF_LIB=$PWD/abtmp/libhf_base.so";;
      new) E="HF_X=1";;
    esac
    env $E timeout 300 python tools/time_variants.py ${CFGS:-2 3} | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn > gpurun_out/ab3/ab.log
python - <<'PY'
import json, numpy as np
from collections import defaultdict
d=defaultdict(list)
for line in open('gpurun_out/ab3/ab.log'):
    arm,_,js=line.strip().partition(' ')
    if not js.startswith('{'): continue
    r=json.loads(js); d[(r['cfg'],r['strategy'],arm)].append((r['b2b_us'],r['clean_flushed_us']))
arms=('base','new')
for c,s in sorted({(c,s) for c,s,_ in d}):
    print(f"cfg{c} {s:8s}", " | ".join(f"{a} {np.median(np.array(d[(c,s,a)])[:,0]):6.2f}/{np.median(np.array(d[(c,s,a)])[:,1]):6.2f}" for a in arms if (c,s,a) in d))
PY
