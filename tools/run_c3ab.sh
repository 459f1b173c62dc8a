# GPU-box helper: contraction parity on tools/libttc_new.so, then alternating A/B of libttc_old vs libttc_new on C3.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 600 python -m pytest tests/test_gpu_contract.py tests/test_gpu_splice.py tests/test_gpu_guard.py -q -x > $O/c3_t.log 2>&1; echo "t rc=$?"; tail -2 $O/c3_t.log
bash tools/run_ab.sh C3 old new
