# GPU-box helper: rank-16 parity on tools/libttc_new.so, then alternating A/B of libttc_old vs libttc_new on C2.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 600 python -m pytest tests/test_gpu_inner.py tests/test_gpu_guard.py -q -x -k "c2 or C2 or rank16 or integer or tagged or determinism or virtual or stay" > $O/c2_t.log 2>&1; echo "t rc=$?"; tail -2 $O/c2_t.log
bash tools/run_ab.sh C2 old new
