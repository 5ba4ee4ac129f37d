# A/B of development switches on the config-3 bench (short runs)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ab
run() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab/$name.json 2> gpurun_out/ab/$name.err; python - "$name" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab/{n}.json").read().strip().splitlines()[-1])
    kc = d["kernel_classes"]
    print(f"{n:14s} value {d['value']:7.1f} e2e {d['e2e']['value']:7.1f} spmm {kc['spmm']['ms_per_step']:.3f} sk {kc['spmm_sketch']['ms_per_step']:.3f} "
          f"gram {kc['dmma_gram']['ms_per_step']:.3f} gemm {kc['dmma_gemm']['ms_per_step']:.3f} eig {kc['eigensolver']['ms_per_step']:.3f} "
          f"gn {kc['dmma_gram_narrow']['ms_per_step']:.3f} nn_n {kc['dmma_gemm_narrow']['ms_per_step']:.3f}")
except Exception as e:
    print(n, "ERR", e)
PY
}
run base X=1
run slabs STG_SPMM_SLABS=1
run base2 X=1
