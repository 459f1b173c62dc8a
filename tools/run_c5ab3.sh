# GPU-box helper: C5 tests on the new build, then alternating A/B of tools/libttc_old.so vs libttc_new.so on C5.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 600 python -m pytest tests/test_gpu_inner.py tests/test_gpu_guard.py -q -x -k "c5 or C5 or ffma or variants or cost_ordered or virtual or integer or edge or stay" > $O/c5_t.log 2>&1; echo "t rc=$?"; tail -1 $O/c5_t.log
bash tools/run_ab.sh C5 old new
