cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2n
python tools/kbench.py small 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q > gpurun_out/r2n/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2n/pytest.log; grep -E "^FAILED|Error|assert" gpurun_out/r2n/pytest.log | head
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2n/b.json 2> gpurun_out/r2n/b.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2n/b.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print("value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: round(kc[k]["ms_per_step"], 3) for k in ("eigensolver", "dmma_gram")})
PY
