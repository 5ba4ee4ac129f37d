# round-2 final records: GPU suite, the driver's bench command (both arms), every BASELINE config
cd $GRAFT_REPO_ROOT
O=gpurun_out/final; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "bench rc=$?"
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference_cfg3.json 2> $O/bench_reference_cfg3.err; echo "ref rc=$?"
for c in cfg1 cfg2 cfg4; do
  timeout 1500 python bench.py --config $c --steps 10 --warmup 3 > $O/bench_$c.json 2> $O/bench_$c.err; echo "$c rc=$?"
done
for k in 32 16 64; do
  timeout 1500 python bench.py --config cfg5 --k $k --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg5_k$k.json 2> $O/bench_cfg5_k$k.err; echo "cfg5 k=$k rc=$?"
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/final/bench*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d.get("roofline") or {}
        print(f.split("/")[-1], "value", round(d["value"], 3), "e2e", round(d["e2e"]["value"], 3), "roof", r.get("kernel"), round(r.get("frac", 0) or 0, 3), "clk", d.get("clocks"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
    except Exception as e:
        print(f, "ERR", e)
PY
