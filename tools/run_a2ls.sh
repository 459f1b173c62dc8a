# GPU-box helper: block-mode local sweeps A/B (tools/libttc_l2.so, libttc_l3.so against libttc_old.so) on A2ii / A2iii.
O=gpurun_out
for v in l2 l3; do TTC_LIB_PATH=tools/libttc_$v.so timeout 900 python -m pytest tests/test_gpu_ttsvd.py -q -x > $O/a2_t_$v.log 2>&1; echo "t $v rc=$?"; tail -1 $O/a2_t_$v.log; done
bash tools/run_ab.sh A2ii old l2
bash tools/run_ab.sh A2ii old l3
bash tools/run_ab.sh A2iii old l2
bash tools/run_ab.sh A2iii old l3
