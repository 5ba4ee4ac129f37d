cd $GRAFT_REPO_ROOT
export STG_SHARD_DEBUG=1
timeout 240 python tools/dbg_shard.py $1 > gpurun_out/dbg.log 2>&1
