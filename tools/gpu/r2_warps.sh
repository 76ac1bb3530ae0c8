cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/warps
for rep in 1 2; do
  for w in 0 7 8 9 10 11; do
    HF_APPLY_WARPS=$w timeout 300 python tools/time_variants.py 3 --strategies=tensor2 | sed "s/^/w$w /"
    HF_APPLY_WARPS=$w timeout 300 python tools/time_variants.py 2 --strategies=tensor2 | sed "s/^/w$w /"
  done
  for w in 0 5 6 7; do
    HF_APPLY_WARPS=$w timeout 300 python tools/time_variants.py 3 --strategies=scalar,tensor4 | sed "s/^/w$w /"
    HF_APPLY_WARPS=$w timeout 300 python tools/time_variants.py 2 --strategies=scalar | sed "s/^/w$w /"
  done
done 2>&1 | grep -v Warn > gpurun_out/warps/ab.log
python - <<'PY'
import json, numpy as np
from collections import defaultdict
d=defaultdict(list); arms=[]
for line in open('gpurun_out/warps/ab.log'):
    arm,_,js=line.strip().partition(' ')
    if not js.startswith('{'): continue
    if arm not in arms: arms.append(arm)
    r=json.loads(js); d[(r['cfg'],r['strategy'],arm)].append((r['b2b_us'],r['clean_flushed_us']))
for c,s in sorted({(c,s) for c,s,_ in d}):
    print(f"cfg{c} {s:8s}", " | ".join(f"{a} {np.median(np.array(d[(c,s,a)])[:,0]):6.2f}/{np.median(np.array(d[(c,s,a)])[:,1]):6.2f}" for a in arms if (c,s,a) in d))
PY
