cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s4a
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4a/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s4a/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4a/pytest_gpu.log
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s4a/bench.json 2> gpurun_out/s4a/bench.err; echo "bench rc=$?"
head -c 900 gpurun_out/s4a/bench.json
STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/s4a/klog.txt 2>&1; echo "klog rc=$?"
