cd $GRAFT_REPO_ROOT
O=gpurun_out/s4i; mkdir -p $O
t() { name=$1; shift; env "$@" timeout 600 python -m pytest "tests/test_gpu_fullsize_parity.py::test_fullsize_parity[cfg4]" -x -q -s > $O/t_$name.log 2>&1; echo "$name rc=$? $(grep -E 'cfg4 step' $O/t_$name.log | head -2 | tr '\n' ' ')"; }
t nnold STG_NN_NOPERSIST=1
t gramold STG_GRAM_NOPERSIST=1
t nors STG_GRAM_NORS=1
t noorder STG_GRAM_NOORDER=1
t rotinline STG_ROT_INLINE=1
