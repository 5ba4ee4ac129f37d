cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab3
python tools/kbench.py gram > gpurun_out/ab3/kb_new.txt 2>&1
STG_GRAM_REDUCE_OLD=1 python tools/kbench.py gram > gpurun_out/ab3/kb_old.txt 2>&1
paste gpurun_out/ab3/kb_old.txt gpurun_out/ab3/kb_new.txt | awk -F'\t' '{print $1 " || " $2}'
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab3/b_$name.json 2> gpurun_out/ab3/b_$name.err
  python - $name <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab3/b_{v}.json").read().strip().splitlines()[-1])
kc = d["kernel_classes"]
print(v, "value", round(d["value"], 1), "e2e", round(d["e2e"]["value"], 1), {k: (round(kc[k]["ms_per_step"], 3), round(kc[k].get("frac_of_roofline_bound", 0), 3)) for k in ("dmma_gram", "dmma_gram_narrow", "dmma_gemm")})
PY
}
run new X=1
run old STG_GRAM_REDUCE_OLD=1
run new2 X=1
