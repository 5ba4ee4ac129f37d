# Gram split policy sweep (per-launch klog timelines) + one ncu --set full capture of a mid-size NN launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for w in 3 6 12 24; do
  STG_GRAM_WAVES=$w STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/klog_w$w.txt 2>&1
  echo "waves $w rc=$?"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_nn_tma_kernel --launch-skip 40 --launch-count 3 \
  -o gpurun_out/nn_mid python tools/profile_step.py --warmup 2 --steps 1 > gpurun_out/ncu_nn.log 2>&1
echo "ncu rc=$?"
