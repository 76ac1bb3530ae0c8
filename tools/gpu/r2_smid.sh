cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out/smid
for rep in 1 2 3; do
  HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py tensor4 2 > /dev/null 2>&1
  mv gpurun_out/timeline_tensor4_2.npy gpurun_out/smid/t4_$rep.npy; mv gpurun_out/timeline_tensor4_2_smid.npy gpurun_out/smid/t4_${rep}_smid.npy
done
HF_LIB=paper_1904_13131_b200/libhf_tl.so timeout 300 python tools/timeline.py tensor2 2 > /dev/null 2>&1
mv gpurun_out/timeline_tensor2_2.npy gpurun_out/smid/t2_1.npy; mv gpurun_out/timeline_tensor2_2_smid.npy gpurun_out/smid/t2_1_smid.npy
nvidia-smi -L
