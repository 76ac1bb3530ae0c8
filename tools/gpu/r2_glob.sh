set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py tests/test_gpu_mg.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider -k "not config5 and not config4" 2>&1 | tail -n 2
for rep in 1 2 3; do
  for arm in base static glob; do
    case $arm in
      base) E="HF_LIB=$PWD/abtmp/libhf_base.so";;
      static) E="HF_SCHED=static";;
      glob) E="";;
    esac
    env $E timeout 300 python tools/time_variants.py 2 3 | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn > gpurun_out/ab3.log
python - <<'PY'
import json, numpy as np
from collections import defaultdict
d=defaultdict(list)
for line in open('gpurun_out/ab3.log'):
    arm,_,js=line.strip().partition(' ')
    if not js.startswith('{'): continue
    r=json.loads(js); d[(r['cfg'],r['strategy'],arm)].append((r['b2b_us'],r['clean_flushed_us']))
for c,s in sorted({(c,s) for c,s,_ in d}):
    print(f"cfg{c} {s:8s}", " | ".join(f"{a} {np.median(np.array(d[(c,s,a)])[:,0]):6.2f}/{np.median(np.array(d[(c,s,a)])[:,1]):6.2f}" for a in ('base','static','glob')))
PY
for v in "tensor4 2" "tensor2 2"; do
  HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py $v
done
