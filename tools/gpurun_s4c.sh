cd $GRAFT_REPO_ROOT
O=gpurun_out/s4c; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_trackers.py tests/test_gpu_edge_cases.py -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
klog() { name=$1; shift; env "$@" STG_KLOG=1 timeout 300 python tools/profile_step.py --real-x0 --device-edits --warmup 3 --steps 1 > $O/klog_$name.txt 2>&1; echo "klog $name rc=$?"; }
klog base STG_NN_NOPERSIST=1 STG_GRAM_NOPERSIST=1
klog rs X=1
klog rsg STG_NN_NOPERSIST=1
klog rsn STG_GRAM_NOPERSIST=1
python tools/klog_summary.py $O/klog_base.txt $O/klog_rs.txt $O/klog_rsg.txt $O/klog_rsn.txt > $O/summary.txt 2>&1
cat $O/summary.txt
bench() { name=$1; shift; env "$@" timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $O/b_$name.json 2> $O/b_$name.err; python -c "
import json,sys
d=json.loads(open('$O/b_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['value'],1), round(d['e2e']['value'],1))"; }
bench base STG_NN_NOPERSIST=1 STG_GRAM_NOPERSIST=1
bench rs X=1
bench rsg STG_NN_NOPERSIST=1
bench rsn STG_GRAM_NOPERSIST=1
