cd $GRAFT_REPO_ROOT
O=gpurun_out/s4n; mkdir -p $O
for bw in 0 1 2; do echo "BLOCK_WAVES=$bw"; BLOCK_WAVES=$bw ./tools/microbench/gram_pipe | grep -E "heavy-first +(200x200 sym waves (6|12)|164x100 waves (6|12)|64x200 waves  6)"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "persistent or config4_shape or rsvd" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
bench() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/b_$name.json 2> $O/b_$name.err; python -c "
import json,sys
d=json.loads(open('$O/b_$name.json').read().strip().splitlines()[-1]); kc=d['kernel_classes']; print('$name', round(d['value'],1), round(d['e2e']['value'],1), {k: round(kc[k]['ms_per_step'],3) for k in ('dmma_gram','dmma_gemm','eigensolver')})"; }
bench bw0 X=1
bench bw1 STG_GRAM_BLOCK_WAVES=1
bench bw2 STG_GRAM_BLOCK_WAVES=2
bench bw3 STG_GRAM_BLOCK_WAVES=3
