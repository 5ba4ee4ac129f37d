cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2m
python tools/kbench.py small 2>&1 | tail -4
STG_TRI_TWOPASS=1 python tools/kbench.py small 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_trackers.py tests/test_gpu_init.py -x -q > gpurun_out/r2m/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2m/pytest.log; grep -E "^FAILED|Error|assert" gpurun_out/r2m/pytest.log | head
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2m/b_$name.json 2> gpurun_out/r2m/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/r2m/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: round(kc[k]["ms_per_step"], 3) for k in ("eigensolver", "dmma_gram")})
PY
}
run fused X=1
run twopass STG_TRI_TWOPASS=1
run fused2 X=1
