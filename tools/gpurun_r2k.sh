cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2k
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_kernels.py -x -q > gpurun_out/r2k/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2k/pytest.log; grep -E "^FAILED|Error" gpurun_out/r2k/pytest.log | head
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2k/b_$name.json 2> gpurun_out/r2k/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/r2k/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: (round(kc[k]["ms_per_step"], 3), round(kc[k].get("frac_hbm", 0), 3)) for k in ("spmm", "spmm_sketch")})
PY
}
run t2 X=1
run t1 STG_SPMM_TMAX=1
run t4all STG_SPMM_TMAX=4 STG_SPMM_FUSED_MIN_M=1000
run t2all STG_SPMM_TMAX=2 STG_SPMM_FUSED_MIN_M=1000
