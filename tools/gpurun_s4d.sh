cd $GRAFT_REPO_ROOT
O=gpurun_out/s4d; mkdir -p $O
klog() { name=$1; shift; env "$@" STG_KLOG=1 STG_NO_SPEC=1 timeout 300 python tools/profile_step.py --device-edits --warmup 2 --steps 1 > $O/klog_$name.txt 2>&1; echo "klog $name rc=$?"; }
klog rs X=1
klog skip STG_LIB=$PWD/tools/ab/lib_skipmma.so
python tools/klog_summary.py $O/klog_rs.txt $O/klog_skip.txt > $O/summary.txt 2>&1
cat $O/summary.txt
tail -5 $O/klog_skip.txt
