# the whole GPU suite (what the driver runs at round end) plus the cfg4 basis check
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
STG_SKETCH_LOG=1 timeout 600 python tools/dbg_cfg4.py > gpurun_out/dbg_cfg4.log 2>&1; grep -E "sketch|step1|D gpu" gpurun_out/dbg_cfg4.log | tail -12
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|Error|error" gpurun_out/pytest_gpu.log | tail -12
grep -E "^FAILED" gpurun_out/pytest_gpu.log | head -20
