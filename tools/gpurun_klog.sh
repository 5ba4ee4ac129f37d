cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/klog.txt 2>&1; echo "klog rc=$?"
timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 3 > gpurun_out/phases.txt 2>&1; echo "phases rc=$?"
tail -3 gpurun_out/phases.txt
