# ncu --set full captures of the step's SpMM and DMMA Gram launches at config 3
# (one step after two warm-up steps), plus the launch list of the same command.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits"
timeout 300 $CMD > gpurun_out/ps_plain.txt 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/ps_plain.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm --launch-skip-before-match 0 -c 40 -o gpurun_out/spmm_cfg3 $CMD > gpurun_out/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_tma|gram_reduce|gram_stream" -c 60 -o gpurun_out/gram_cfg3 $CMD > gpurun_out/ncu_gram.log 2>&1; echo "ncu gram rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ls -la gpurun_out
