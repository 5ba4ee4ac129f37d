cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
AB_ENV=STG_NN_STAGES3=1 bash tools/gpurun_abn.sh
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg4.json')); print('cfg4', d['value'], d['kernel_classes']['dmma_gram']['ms_per_step'])"
