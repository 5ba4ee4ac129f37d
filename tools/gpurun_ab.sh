# parity of the current build, then an A/B of an env switch on the cfg3 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench a rc=$?"
env ${AB_ENV:-STG_GRAM_UNFUSED=1} timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err; echo "bench b rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/bench_a.json", "gpurun_out/bench_b.json"):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "failed", e); continue
    print(f, round(d["value"], 2), round(d["e2e"]["value"], 2), {k: round(v["ms_per_step"], 3) for k, v in d["kernel_classes"].items()})
PY
