cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -x -q -s > gpurun_out/fullsize.log 2>&1; echo "fullsize rc=$?" >> gpurun_out/fullsize.log
tail -5 gpurun_out/fullsize.log
timeout 600 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg3.json')); print(d['value'], d['e2e'], d['roofline'])"
