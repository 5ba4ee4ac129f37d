cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python tools/dbg_init.py 262144 1 2 > gpurun_out/dbg_init.log 2>&1; cat gpurun_out/dbg_init.log | tail -3
timeout 600 python tools/dbg_init.py 262144 1 2 x > gpurun_out/dbg_init2.log 2>&1; cat gpurun_out/dbg_init2.log | tail -3
timeout 600 python tools/dbg_init.py 262144 1 0 x > gpurun_out/dbg_init3.log 2>&1; cat gpurun_out/dbg_init3.log | tail -3
