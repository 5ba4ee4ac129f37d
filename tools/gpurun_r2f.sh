cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2f
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2f/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r2f/pytest_gpu.log | tail -2; grep -E "^FAILED|Error" gpurun_out/r2f/pytest_gpu.log | head -10
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2f/bench.json 2> gpurun_out/r2f/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2f/bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "tracker-only", round(d["tracker_step_only"]["value"], 1), "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), d["roofline"]["traffic"])
PY
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 9000 --csv --log-file gpurun_out/r2f/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r2f/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/r2f/launches_cfg3.csv 2 | head -50
