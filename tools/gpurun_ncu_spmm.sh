cd $GRAFT_REPO_ROOT
CMD="python tools/profile_step.py --steps 1 --warmup 1"
timeout 300 $CMD > gpurun_out/ps_plain.txt 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -c 8 -o gpurun_out/spmm_full $CMD > gpurun_out/ncu_spmm.log 2>&1
echo "rc=$?"
