# GPU-box helper: C5 tests on the new build, then alternating A/B of tools/libttc_old.so vs libttc_new.so on C5
# and on the rank-profile sweep.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 600 python -m pytest tests/test_gpu_inner.py tests/test_gpu_guard.py -q -x -k "c5 or C5 or ffma or variants or cost_ordered or virtual or integer or edge or stay" > $O/c5_t.log 2>&1; echo "t rc=$?"; tail -2 $O/c5_t.log
bash tools/run_ab.sh C5 old new
for L in old new; do echo "== $L"; TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python tools/c5_shapes.py 2>&1 | tail -5; done
