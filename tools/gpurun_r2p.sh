cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2p
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_kernels.py tests/test_gpu_trackers.py tests/test_gpu_blocks.py -x -q > gpurun_out/r2p/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2p/pytest.log; grep -E "^FAILED|Error|assert" gpurun_out/r2p/pytest.log | head
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2p/b_$name.json 2> gpurun_out/r2p/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/r2p/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: round(kc[k]["ms_per_step"], 3) for k in ("eigensolver", "dmma_gram_narrow", "cholesky")})
PY
}
run kearly X=1
run knormal STG_NO_K_EARLY=1
run kearly2 X=1
run knormal2 STG_NO_K_EARLY=1
STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > gpurun_out/r2p/klog.txt 2>&1; echo "klog rc=$?"
