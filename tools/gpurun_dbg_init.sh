cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
STG_LZ_LOG2=1 STG_LZ_LOG=1 timeout 900 python tools/dbg_cfg4c.py 6 > gpurun_out/dbg_c6.log 2>&1; grep -E "lzdbg|ERR|ok|restart [0-6] " gpurun_out/dbg_c6.log | head -40
