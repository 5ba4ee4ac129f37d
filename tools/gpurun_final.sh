# Round-end evidence: bench lines (cfg3 default with CPU baseline, cfg5 s25, cfg4), the ncu launch list of the
# cfg3 bench, and one ncu --set full capture of the step's Gram launches (dominant class)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python bench.py > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 900 python bench.py --config cfg4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu.log 2>&1
echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tma_kernel \
  -o gpurun_out/gram_full python tools/profile_step.py --real-x0 --warmup 0 --steps 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"
