cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/fp32
timeout 1500 python - <<'PY' 2>&1 | grep -v Warn
import sys, json, ctypes as ct, time
sys.argv=['bench.py']
import bench, torch
from paper_1904_13131_b200._lib import lib
def pool(tag):
    a,b=ct.c_longlong(),ct.c_longlong(); lib().hf_pool_info(ct.byref(a),ct.byref(b))
    free,total=torch.cuda.mem_get_info()
    print(tag,'pooled GB',a.value/2**30,'live GB',b.value/2**30,'torch reserved GB',torch.cuda.memory_reserved()/2**30,'device free GB',free/2**30, flush=True)
from paper_1904_13131_b200 import MatrixFreeTangent
from paper_1904_13131_b200.workloads import make_workload
pool('start')
r=bench._newton_iteration('fp32'); print('fp32 first', r['s_per_cg_iteration']); pool('after fp32')
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for cid,mm in ((2,64),(3,32)):
    wlb=make_workload(cid,seed=0,m=mm); pb=wlb.fine
    xb=torch.from_numpy(wlb.x).cuda(); yb=torch.empty_like(xb)
    for s in ("tensor4","tensor2","scalar"):
        op=MatrixFreeTangent(pb,wlb.ubar,s); bench._time_steps(op,xb,yb,10,3,flush); del op
    del xb,yb,wlb,pb
    pool(f'after big {cid}')
r=bench._newton_iteration(); print('fp64', r['s_per_cg_iteration']); pool('after fp64')
r=bench._newton_iteration('fp32'); print('fp32 after big', r['s_per_cg_iteration'], r['cg_iterations']); pool('after fp32 #2')
lib().hf_pool_release(); pool('released')
r=bench._newton_iteration('fp32'); print('fp32 after release', r['s_per_cg_iteration']); pool('end')
PY
