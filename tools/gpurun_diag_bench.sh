# init + full-size parity tests, bench at the driver's command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_init.py -x -q -s > gpurun_out/pytest_init.log 2>&1; echo "pytest init rc=$?"; grep -E "restarts|passed|failed|Error" gpurun_out/pytest_init.log | tail -12
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/d1.json 2> gpurun_out/d1.err; echo "d1 rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/d1.json",):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["value"], d["e2e"]["value"], d["step_ms"], d["step_ms_e2e"])
    except Exception as e: print(f, e)
PY
timeout 1800 python -m pytest tests/test_gpu_fullsize_parity.py -x -q -s > gpurun_out/pytest_full.log 2>&1; echo "pytest full rc=$?"; grep -E "step|worst|init|passed|failed|Error" gpurun_out/pytest_full.log | tail -40
