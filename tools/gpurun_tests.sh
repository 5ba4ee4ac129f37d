# the whole GPU suite (what the driver runs at round end) plus the bench at the driver's command
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_spec.json 2> gpurun_out/b_spec.err; echo "bench rc=$?"
STG_NO_SPEC=1 timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_nospec.json 2> gpurun_out/b_nospec.err; echo "bench nospec rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/b_spec.json", "gpurun_out/b_nospec.json"):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "tracker-only", d.get("tracker_step_only", {}).get("value"),
              "roof", d["roofline"]["kernel"], round(d["roofline"]["frac"], 3), d["roofline"].get("frac_of_roofline_bound"))
        for k, v in d["kernel_classes"].items():
            print("   ", k, {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in v.items()})
    except Exception as e:
        print(f, "ERR", e)
PY
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -3
grep -E "^FAILED" gpurun_out/pytest_gpu.log | head -20
