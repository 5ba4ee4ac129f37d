# What the driver runs at round end: build, smoke, GPU tests, default bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/re_smoke.log 2>&1; echo "build+smoke rc=$?"
tail -1 gpurun_out/re_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/re_pytest.log 2>&1; echo "pytest rc=$?"
tail -1 gpurun_out/re_pytest.log
timeout 600 python bench.py > gpurun_out/re_bench.json 2> gpurun_out/re_bench.err; echo "bench rc=$?"
head -c 300 gpurun_out/re_bench.json
