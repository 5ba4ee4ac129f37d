cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2o
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2o/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2o/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/r2o/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r2o/pytest_gpu.log | tail -2; grep -E "^FAILED|Error" gpurun_out/r2o/pytest_gpu.log | head -10
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2o/bench.json 2> gpurun_out/r2o/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2o/bench.json").read().strip().splitlines()[-1])
print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "tracker-only", round(d["tracker_step_only"]["value"], 1),
      "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), "cpu", d.get("cpu_baseline", {}).get("value"), d["clocks"])
print({k: (round(v["ms_per_step"], 3), round(v.get("frac_of_roofline_bound", 0), 3)) for k, v in d["kernel_classes"].items()})
PY
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2o/reference.json 2> gpurun_out/r2o/reference.err; echo "ref rc=$?"; head -c 400 gpurun_out/r2o/reference.json
