# GPU test suite (optionally a subset: $1 = pytest -k expression)
cd $GRAFT_REPO_ROOT
if [ -n "$1" ]; then K="-k $1"; X=""; else K=""; X="-x"; fi
timeout 1200 python -m pytest tests -m gpu $X -q $K -s > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
