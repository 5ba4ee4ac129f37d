cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
for sc in 14 20; do
timeout 600 python bench.py --sharded --scale $sc --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sharded_$sc.json 2> gpurun_out/bench_sharded_$sc.err; echo "sharded $sc rc=$?"
timeout 600 python bench.py --scale $sc --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain_$sc.json 2> gpurun_out/bench_plain_$sc.err; echo "plain $sc rc=$?"
done
