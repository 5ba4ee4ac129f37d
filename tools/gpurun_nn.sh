cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
AB_ENV=STG_NN_TILE=1 bash tools/gpurun_abn.sh
STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/klog.txt 2>&1; echo "klog rc=$?"
