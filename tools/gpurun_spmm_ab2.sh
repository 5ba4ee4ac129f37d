cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sab2
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/sab2/b_$name.json 2> gpurun_out/sab2/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/sab2/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: (round(kc[k]["ms_per_step"], 3), round(kc[k].get("frac_hbm", 0), 3)) for k in ("spmm", "spmm_sketch")})
PY
}
run allfused STG_SPMM_FUSED_MIN_M=1
run default X=1
run unfused STG_SPMM_UNFUSED=1
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits --real-x0"
STG_SPMM_FUSED_MIN_M=1 timeout 900 ncu --set full --clock-control none -k regex:spmm -c 6 -o /tmp/spmmf $CMD > gpurun_out/sab2/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/spmmf.ncu-rep --page raw --csv > gpurun_out/sab2/spmmf_raw.csv 2>/dev/null
