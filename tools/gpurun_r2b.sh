# bench at the driver's command (device tracker_init X0), a per-launch timeline
# of one config-3 step, and ncu --set full of the step's SpMM launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo "bench rc=$?"
head -c 600 gpurun_out/r2b/bench.json; echo
STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/r2b/klog.txt 2>&1; echo "klog rc=$?"
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits --real-x0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -c 14 -o /tmp/spmm_cfg3 $CMD > gpurun_out/r2b/ncu_spmm.log 2>&1; echo "ncu spmm rc=$?"
ncu -i /tmp/spmm_cfg3.ncu-rep --page raw --csv > gpurun_out/r2b/spmm_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/spmm_cfg3.ncu-rep --page details --csv > gpurun_out/r2b/spmm_cfg3_details.csv 2>/dev/null
cp /tmp/spmm_cfg3.ncu-rep gpurun_out/r2b/
ls -la gpurun_out/r2b
