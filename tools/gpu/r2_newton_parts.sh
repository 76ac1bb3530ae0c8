# u_rel of the 4-Morton-box Newton against one GPU, several runs, three-term (1) and stored-direction (0) smoothers
cd $GRAFT_REPO_ROOT; O=gpurun_out/nparts; mkdir -p $O; : > $O/log.txt
for v in 1 0 1 0 1 0; do
  for part in "4 morton" "2 slab"; do set -- $part
  HF_CHEB3=$v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$1 --master-addr 127.0.0.1 --master-port 29517 tests/dist_worker.py --backend gloo --cells 8 --config 2 --newton --partition $2 2>/dev/null | grep DISTRESULT | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l[len('DISTRESULT '):]); print('cheb3=$v', '$1 $2', 'u_rel', d['u_rel'], 'cg', [int(x[3]) for x in d['single']], [int(x[3]) for x in d['dist']])" >> $O/log.txt
  done
done
cat $O/log.txt
