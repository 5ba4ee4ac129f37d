cd $GRAFT_REPO_ROOT
echo "== tma, all-thread release"; python tools/dbg_det.py 2>&1 | tail -14
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x 2>&1 | tail -3
