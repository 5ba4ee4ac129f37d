cd $GRAFT_REPO_ROOT
O=gpurun_out/s4q; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_trackers.py tests/test_gpu_edge_cases.py tests/test_gpu_blocks.py tests/test_gpu_wire.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
bench() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${ARGS} > $O/b_$name.json 2> $O/b_$name.err; python -c "
import json,sys
d=json.loads(open('$O/b_$name.json').read().strip().splitlines()[-1]); kc=d['kernel_classes']; print('$name', round(d['value'],1), round(d['e2e']['value'],1), {k: round(kc[k]['ms_per_step'],3) for k in ('masked_gram_x','csr_merge','spmm') if k in kc})"; }
bench nodefer STG_NO_MERGE_DEFER=1
bench new X=1
bench nodefer2 STG_NO_MERGE_DEFER=1
bench new2 X=1
ARGS="--config cfg4 --steps 6 --warmup 3" bench c4old STG_NO_MERGE_DEFER=1
ARGS="--config cfg4 --steps 6 --warmup 3" bench c4new X=1
