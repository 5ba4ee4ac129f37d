# config 5: parity at s17 (device generator), then bench lines at s22 and s25
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -k config5 -x -q -s > gpurun_out/cfg5_test.log 2>&1; echo "test rc=$?" >> gpurun_out/cfg5_test.log
timeout 600 python bench.py --config cfg5 --scale 22 --steps 5 --warmup 3 > gpurun_out/bench_cfg5_s22.json 2> gpurun_out/bench_cfg5_s22.err; echo "s22 rc=$?"
timeout 1500 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "s25 rc=$?"
tail -3 gpurun_out/cfg5_test.log; tail -3 gpurun_out/bench_cfg5.err
