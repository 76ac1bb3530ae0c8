cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/hoist
HF_LIB=$PWD/paper_1904_13131_b200/libhf_hoist.so timeout 900 python -m pytest tests/test_gpu_ops.py -x -q -p no:cacheprovider 2>&1 | tail -n 2
for rep in 1 2 3; do
  for arm in base hoist; do
    case $arm in
      base) E="HF_LIB=$PWD/abtmp/libhf_base.so";;
      hoist) E="HF_LIB=$PWD/paper_1904_13131_b200/libhf_hoist.so";;
    esac
    env $E timeout 300 python tools/time_variants.py 2 | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn > gpurun_out/hoist/ab.log
python - <<'PY'
import json, numpy as np
from collections import defaultdict
d=defaultdict(list); arms=[]
for line in open('gpurun_out/hoist/ab.log'):
    arm,_,js=line.strip().partition(' ')
    if not js.startswith('{'): continue
    if arm not in arms: arms.append(arm)
    r=json.loads(js); d[(r['cfg'],r['strategy'],arm)].append((r['b2b_us'],r['clean_flushed_us']))
for c,s in sorted({(c,s) for c,s,_ in d}):
    print(f"cfg{c} {s:8s}", " | ".join(f"{a} {np.median(np.array(d[(c,s,a)])[:,0]):6.2f}/{np.median(np.array(d[(c,s,a)])[:,1]):6.2f}" for a in arms if (c,s,a) in d))
PY
