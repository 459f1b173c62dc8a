# GPU-box helper: TT-SVD parity on tools/libttc_new.so, then alternating A/B of libttc_old vs libttc_new on A2.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 900 python -m pytest tests/test_gpu_ttsvd.py -q -x > $O/a2_t.log 2>&1; echo "t rc=$?"; tail -2 $O/a2_t.log
bash tools/run_ab.sh A2 old new
