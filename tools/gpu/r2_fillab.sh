cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/fillab
for rep in 1 2 3; do
  for arm in "u4" "u8_b8" "u8_b3" "u8_b2" "u16_b2" "u16_b1" "u16_b3"; do
    case $arm in
      u4) E="HF_X=1";;
      u8_b8) E="HF_FILL_UNROLL=8 HF_FILL_BLOCKS=8";;
      u8_b3) E="HF_FILL_UNROLL=8 HF_FILL_BLOCKS=3";;
      u8_b2) E="HF_FILL_UNROLL=8 HF_FILL_BLOCKS=2";;
      u16_b2) E="HF_FILL_UNROLL=16 HF_FILL_BLOCKS=2";;
      u16_b1) E="HF_FILL_UNROLL=16 HF_FILL_BLOCKS=1";;
      u16_b3) E="HF_FILL_UNROLL=16 HF_FILL_BLOCKS=3";;
    esac
    env $E timeout 300 python tools/time_variants.py 2 --strategies=tensor4,tensor2 | sed "s/^/$arm /"
  done
done 2>&1 | grep -v Warn > gpurun_out/fillab/ab.log
python - <<'PY'
import json, numpy as np
from collections import defaultdict
d=defaultdict(list); arms=[]
for line in open('gpurun_out/fillab/ab.log'):
    arm,_,js=line.strip().partition(' ')
    if not js.startswith('{'): continue
    if arm not in arms: arms.append(arm)
    r=json.loads(js); d[(r['cfg'],r['strategy'],arm)].append((r['b2b_us'],r['clean_flushed_us']))
for c,s in sorted({(c,s) for c,s,_ in d}):
    print(f"cfg{c} {s:8s}", " | ".join(f"{a} {np.median(np.array(d[(c,s,a)])[:,0]):6.2f}/{np.median(np.array(d[(c,s,a)])[:,1]):6.2f}" for a in arms if (c,s,a) in d))
PY
