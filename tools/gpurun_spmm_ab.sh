# SpMM fused-kernel check: parity tests, A/B bench against the 3-kernel path, ncu of the fused launches
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sab
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_edge_cases.py -x -q > gpurun_out/sab/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/sab/pytest.log
for v in fused unfused; do
  if [ $v = unfused ]; then export STG_SPMM_UNFUSED=1; fi
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sab/b_$v.json 2> gpurun_out/sab/b_$v.err
  python - $v <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/sab/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: (round(kc[k]["ms_per_step"], 3), round(kc[k].get("frac_hbm", 0), 3)) for k in ("spmm", "spmm_sketch")})
PY
done
unset STG_SPMM_UNFUSED
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits --real-x0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:spmm -c 6 -o /tmp/spmmf $CMD > gpurun_out/sab/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/spmmf.ncu-rep --page raw --csv > gpurun_out/sab/spmmf_raw.csv 2>/dev/null
cp /tmp/spmmf.ncu-rep gpurun_out/sab/
