cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
for r in 1 2; do
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pin$r.json 2> gpurun_out/bench_pin.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_pin$r.json')); print(d['value'], d['e2e'])"
done
