# bench lines for every BASELINE config (round 2), the cfg5 k sweep, and the
# reference arm on one host thread (the reference's serial build)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/cfgs
for c in cfg1 cfg2 cfg4; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfgs/bench_$c.json 2> gpurun_out/cfgs/bench_$c.err; echo "$c rc=$?"
done
for k in 32 16 64; do
  timeout 1500 python bench.py --config cfg5 --k $k --steps 5 --warmup 3 > gpurun_out/cfgs/bench_cfg5_k$k.json 2> gpurun_out/cfgs/bench_cfg5_k$k.err; echo "cfg5 k=$k rc=$?"
done
timeout 1500 python bench.py --impl reference --cpu-threads 1 --steps 1 --warmup 0 > gpurun_out/cfgs/reference_1thread.json 2> gpurun_out/cfgs/reference_1thread.err; echo "ref1 rc=$?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/cfgs/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f.split("/")[-1], "value", round(d["value"], 2), "e2e", round(d["e2e"]["value"], 2), "roof", r.get("kernel"), round(r.get("frac", 0), 3), "clk", d.get("clocks"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
