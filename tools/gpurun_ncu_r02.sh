# round-2 profiles: the ncu launch list of the bench command, ncu --set full of the
# step's Gram launches (cfg3) and GEMM launches (cfg4), exported to CSV on the box
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ncu2
timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2/b.json 2> gpurun_out/ncu2/b.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/ncu2/launches_cfg3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu2/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
CMD="python tools/profile_step.py --steps 1 --warmup 2 --device-edits"
timeout 300 $CMD > gpurun_out/ncu2/ps_plain.txt 2>&1; echo "plain rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -f -k regex:"gram_tma|gram_reduce_chunked|gram_stream" -c 24 -o /tmp/gram_cfg3_r02 $CMD > gpurun_out/ncu2/ncu_gram.log 2>&1; echo "ncu gram rc=$?"
ncu -i /tmp/gram_cfg3_r02.ncu-rep --page raw --csv > gpurun_out/ncu2/gram_cfg3_raw.csv 2>/dev/null
ncu -i /tmp/gram_cfg3_r02.ncu-rep --page details --csv > gpurun_out/ncu2/gram_cfg3_details.csv 2>/dev/null
CMD4="python tools/profile_step.py --config cfg4 --steps 1 --warmup 0 --k 64 --device-edits"
timeout 900 $CMD4 > gpurun_out/ncu2/ps4_plain.txt 2>&1; echo "plain4 rc=$?"
timeout 1800 ncu --set full --clock-control none -f -k regex:"gemm_nn_tma" -c 12 -o /tmp/gemm_cfg4_r02 $CMD4 > gpurun_out/ncu2/ncu_gemm4.log 2>&1; echo "ncu gemm4 rc=$?"
ncu -i /tmp/gemm_cfg4_r02.ncu-rep --page raw --csv > gpurun_out/ncu2/gemm_cfg4_raw.csv 2>/dev/null
ls -la gpurun_out/ncu2
