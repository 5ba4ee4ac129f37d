# A/B of library builds on the cfg3 bench: LIBS="name=path ..." bash tools/gpurun_ab_lib.sh
cd $GRAFT_REPO_ROOT
O=gpurun_out/ablib; mkdir -p $O
bench() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/b_$name.json 2> $O/b_$name.err; python -c "
import json,sys
d=json.loads(open('$O/b_$name.json').read().strip().splitlines()[-1]); kc=d['kernel_classes']; print('$name', round(d['value'],1), round(d['e2e']['value'],1), {k: round(kc[k]['ms_per_step'],3) for k in ('dmma_gram','dmma_gemm') if k in kc})"; }
for r in 1 2; do
  bench base$r X=1
  for kv in $LIBS; do bench ${kv%%=*}$r STG_LIB=$PWD/${kv#*=}; done
done
