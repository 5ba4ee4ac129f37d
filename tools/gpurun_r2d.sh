# sketch-factor fold, 129-way bisection, rotation beside the next ingestion: GPU suite + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r2d/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r2d/pytest_gpu.log | tail -2; grep -E "^FAILED|Error" gpurun_out/r2d/pytest_gpu.log | head -10
python tools/kbench.py small > gpurun_out/r2d/kb_small.txt 2>&1; cat gpurun_out/r2d/kb_small.txt
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d/b_$name.json 2> gpurun_out/r2d/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/r2d/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), "trk", round(d["tracker_step_only"]["value"],1), {k: round(kc[k]["ms_per_step"], 3) for k in ("dmma_gram", "dmma_gemm", "eigensolver", "rotate_x")})
PY
}
run new X=1
run nofold STG_NO_SKETCH_FOLD=1
run rotinline STG_ROT_INLINE=1
run new2 X=1
