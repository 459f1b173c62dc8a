O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 300 python -m pytest tests/test_gpu_inner.py -q -k "r64_tcgen05 or c4_full" > $O/c4_t.log 2>&1; echo "t rc=$?"; tail -2 $O/c4_t.log
bash tools/run_ab.sh C4 new old
