# GPU-box helper: reconstruction parity on tools/libttc_new.so (tensor-core D and, TTC_RECON_FFMA=1, the FP32 D),
# then A/B of libttc_old vs libttc_new on R1 and A2.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 900 python -m pytest tests/test_gpu_reconstruct.py tests/test_gpu_guard.py tests/test_gpu_ttsvd.py tests/test_gpu_splice.py -q -x > $O/r1_t.log 2>&1; echo "t rc=$?"; tail -2 $O/r1_t.log
TTC_RECON_FFMA=1 TTC_LIB_PATH=tools/libttc_new.so timeout 900 python -m pytest tests/test_gpu_reconstruct.py -q -x > $O/r1_t2.log 2>&1; echo "t2 rc=$?"; tail -2 $O/r1_t2.log
bash tools/run_ab.sh R1 old new
bash tools/run_ab.sh A2 old new
