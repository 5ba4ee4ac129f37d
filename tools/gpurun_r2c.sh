# full GPU suite + smoke + the driver's bench command, after the SpMM / Gram-reduce / wire changes
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2c/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/r2c/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r2c/pytest_gpu.log | tail -2; grep -E "^FAILED|Error" gpurun_out/r2c/pytest_gpu.log | head -10
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2c/bench.json 2> gpurun_out/r2c/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2c/bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "tracker-only", round(d["tracker_step_only"]["value"], 1),
      "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), "cpu", d.get("cpu_baseline", {}).get("value"), d["clocks"])
PY
