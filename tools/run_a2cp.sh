# GPU-box helper: CTA-per-pair column-length threshold A/B (tools/libttc_p1024.so, libttc_p16384.so against libttc_old.so).
O=gpurun_out
for v in p1024 p16384; do TTC_LIB_PATH=tools/libttc_$v.so timeout 900 python -m pytest tests/test_gpu_ttsvd.py -q -x > $O/a2_t_$v.log 2>&1; echo "t $v rc=$?"; tail -1 $O/a2_t_$v.log; done
bash tools/run_ab.sh A2ii old p1024
bash tools/run_ab.sh A2iii old p1024
bash tools/run_ab.sh A2iii old p16384
