# parity of the current build, the cfg3 bench and a per-launch timeline (STG_KLOG)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_a.json"))
print(round(d["value"], 2), round(d["e2e"]["value"], 2), {k: round(v["ms_per_step"], 3) for k, v in d["kernel_classes"].items()})
PY
STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/klog.txt 2>&1; echo "klog rc=$?"
