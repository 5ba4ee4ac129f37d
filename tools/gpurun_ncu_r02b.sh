# round-2 (second half) profiles after the persistent DMMA kernels: the ncu launch list of the
# bench command and ncu --set full of the step's Gram / row-local GEMM launches (cfg3)
cd $GRAFT_REPO_ROOT
O=gpurun_out/ncu3; mkdir -p $O
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/b.json 2> $O/b.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file $O/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py $O/launches_cfg3.csv 2 > $O/launch_summary.txt 2>&1
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits"
timeout 300 $CMD > $O/ps_plain.txt 2>&1; echo "plain rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -f -k regex:"gram_persist|gram_reduce_chunked|gemm_nn_persist" -c 40 -o /tmp/dmma_cfg3_r02b $CMD > $O/ncu_dmma.log 2>&1; echo "ncu dmma rc=$?"
ncu -i /tmp/dmma_cfg3_r02b.ncu-rep --page raw --csv > $O/dmma_cfg3_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/dmma_cfg3_raw.csv $O/ncu_dmma_cfg3_r02b.txt > /dev/null
ncu -i /tmp/dmma_cfg3_r02b.ncu-rep --page details --csv > $O/dmma_cfg3_details.csv 2>/dev/null
ls -la $O
