# A/B of an env switch on the cfg3 bench, alternating runs: AB_ENV="VAR=1" bash tools/gpurun_abn.sh
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for r in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_a$r.json 2>/dev/null
  env $AB_ENV timeout 300 python bench.py --no-cpu-baseline > gpurun_out/ab_b$r.json 2>/dev/null
done
python - <<'PY'
import json
for arm in "ab":
    v = []
    for r in (1, 2, 3):
        try:
            d = json.load(open(f"gpurun_out/ab_{arm}{r}.json")); v.append(round(d["value"], 1))
        except Exception as e:
            v.append(None)
    print(arm, v, d["kernel_classes"]["eigensolver"]["ms_per_step"] if d else None)
PY
