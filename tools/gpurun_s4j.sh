cd $GRAFT_REPO_ROOT
O=gpurun_out/s4j; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent or config4_shape" -s > $O/pytest_new.log 2>&1; echo "pytest rc=$?"; grep -E "persistent .* step|passed|failed" $O/pytest_new.log | tail -8
bash tools/gpurun_ncu_r02b.sh
