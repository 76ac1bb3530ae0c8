cd $GRAFT_REPO_ROOT
for rep in 1 2; do for pdl in 0 1; do
  HF_PDL=$pdl HF_LIB=$PWD/abtmp/libhf_prev.so timeout 120 python tools/time_apply.py tensor4 2 | sed "s/^/prev pdl=$pdl /"
  HF_PDL=$pdl timeout 120 python tools/time_apply.py tensor4 2 | sed "s/^/new  pdl=$pdl /"
done; done
