cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_res.json 2> gpurun_out/bench_res.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_res.json')); print(d['value'], d['e2e']['value'], d['spmm_full'])"
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/bench_res5.json 2> gpurun_out/bench_res5.err; echo "cfg5 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_res5.json')); print(d['value'], d['e2e']['value'], d['spmm_full'])"
