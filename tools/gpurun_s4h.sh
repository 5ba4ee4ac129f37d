cd $GRAFT_REPO_ROOT
O=gpurun_out/s4h; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.log
run() { name=$1; shift; env "$@" timeout 900 python bench.py --no-cpu-baseline ${ARGS} > $O/b_$name.json 2> $O/b_$name.err; python -c "
import json,sys
d=json.loads(open('$O/b_$name.json').read().strip().splitlines()[-1]); kc=d['kernel_classes']; print('$name', round(d['value'],2), round(d['e2e']['value'],2), {k: (round(v['ms_per_step'],3), round(v.get('frac_of_roofline_bound') or 0,2)) for k,v in kc.items() if k.startswith('dmma')})"; }
ARGS="--config cfg4 --steps 6 --warmup 3" run cfg4_old STG_NN_NOPERSIST=1 STG_GRAM_NOPERSIST=1
ARGS="--config cfg4 --steps 6 --warmup 3" run cfg4_new X=1
ARGS="--config cfg2" run cfg2_old STG_NN_NOPERSIST=1 STG_GRAM_NOPERSIST=1
ARGS="--config cfg2" run cfg2_new X=1
ARGS="--config cfg1" run cfg1_new X=1
ARGS="--config cfg5 --steps 5 --warmup 3 --k 32" run cfg5_old STG_NN_NOPERSIST=1 STG_GRAM_NOPERSIST=1
ARGS="--config cfg5 --steps 5 --warmup 3 --k 32" run cfg5_new X=1
