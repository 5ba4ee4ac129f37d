cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2i
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_kernels.py tests/test_gpu_shard.py -x -q > gpurun_out/r2i/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2i/pytest.log; grep -E "^FAILED|Error" gpurun_out/r2i/pytest.log | head
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2i/b_$name.json 2> gpurun_out/r2i/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/r2i/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: (round(kc[k]["ms_per_step"], 3), round(kc[k].get("frac_hbm", 0), 3)) for k in ("spmm", "spmm_sketch")})
PY
}
run chunk X=1
run nochunk STG_SPMM_NOCHUNK=1
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits"
timeout 900 ncu --set full --clock-control none -f -k regex:spmm -c 8 -o /tmp/spmmc $CMD > gpurun_out/r2i/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/spmmc.ncu-rep --page raw --csv > gpurun_out/r2i/spmmc_raw.csv 2>/dev/null
