cd $GRAFT_REPO_ROOT
timeout 600 python - <<'PY' 2>&1 | grep -v Warn
import sys, os, gc, numpy as np, torch
sys.path.insert(0,'tests')
from _cases import golden, product_levels, rel
from paper_1904_13131_b200 import build_gmg, build_transfers
g = golden("mg_3d_8.npz"); probs = product_levels(g); transfers = build_transfers(probs); b = g["b"]
def fresh(u, use_graph=True):
    return build_gmg(probs, u, "tensor4", seed=0, transfers=transfers, use_graph=use_graph)
u1=g["ubar"]; u2=0.5*g["ubar"]
e_a=fresh(u2,False).apply(b); e_b=fresh(u2,False).apply(b)
print('eager vs eager (two hierarchies)', rel(e_a,e_b))
h=fresh(u2,False); print('eager twice same hierarchy', rel(h.apply(b), h.apply(b)))
for mode in ('torch','native'):
    os.environ['HF_GRAPH']=mode
    first=fresh(u1); z1=first.apply(b); print(mode,'first updated?', getattr(first._graph,'updated',None))
    del first; gc.collect()
    second=fresh(u2); z2=second.apply(b); print(mode,'second updated?', getattr(second._graph,'updated',None), 'vs eager', rel(z2,e_a), 'replay again', rel(second.apply(b), z2))
    lam=[(lv.lam_max, lv.lam_min) for lv in second.levels]
    print(mode, 'lam', lam[:2])
h=fresh(u2,False); print('eager lam', [(lv.lam_max, lv.lam_min) for lv in h.levels][:2])
PY
