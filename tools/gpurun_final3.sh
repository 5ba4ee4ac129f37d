# Final bench lines of the round (all five BASELINE configs on one B200)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/f_cfg3.json 2> gpurun_out/f_cfg3.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/f_cfg5.json 2> gpurun_out/f_cfg5.err; echo "cfg5 rc=$?"
timeout 600 python bench.py --config cfg1 --no-cpu-baseline > gpurun_out/f_cfg1.json 2> gpurun_out/f_cfg1.err; echo "cfg1 rc=$?"
timeout 600 python bench.py --config cfg2 --no-cpu-baseline > gpurun_out/f_cfg2.json 2> gpurun_out/f_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/f_cfg4.json 2> gpurun_out/f_cfg4.err; echo "cfg4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_ref.json 2> gpurun_out/f_ref.err; echo "ref rc=$?"
