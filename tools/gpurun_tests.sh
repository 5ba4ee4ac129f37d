# GPU test suite (optionally a subset: $1 = pytest -k expression)
cd $GRAFT_REPO_ROOT
if [ -n "$1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -s -k "$1" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
