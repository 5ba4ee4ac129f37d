# ncu --set full captures of the step's SpMM and DMMA Gram launches at config 3
# (one step after two warm-up steps), exported to CSV on the box.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits"
timeout 300 $CMD > gpurun_out/ncu/ps_plain.txt 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -c 14 -o /tmp/spmm_cfg3 $CMD > gpurun_out/ncu/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"
ncu -i /tmp/spmm_cfg3.ncu-rep --page raw --csv > gpurun_out/ncu/spmm_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/spmm_cfg3.ncu-rep --page details --csv > gpurun_out/ncu/spmm_cfg3_details.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gram_tma|gram_reduce|gram_stream" -c 30 -o /tmp/gram_cfg3 $CMD > gpurun_out/ncu/ncu_gram.log 2>&1; echo "ncu gram rc=$?"
ncu -i /tmp/gram_cfg3.ncu-rep --page raw --csv > gpurun_out/ncu/gram_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/gram_cfg3.ncu-rep --page details --csv > gpurun_out/ncu/gram_cfg3_details.csv 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_cfg3.csv $CMD > gpurun_out/ncu/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ls -la gpurun_out/ncu; du -sh gpurun_out
