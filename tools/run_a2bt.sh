# GPU-box helper: ttsvd_big CTA size A/B (tools/libttc_t256.so against libttc_old.so).
O=gpurun_out
TTC_LIB_PATH=tools/libttc_t256.so timeout 900 python -m pytest tests/test_gpu_ttsvd.py -q -x > $O/a2_t_t256.log 2>&1; echo "t rc=$?"; tail -1 $O/a2_t_t256.log
bash tools/run_ab.sh A2ii old t256
bash tools/run_ab.sh A2iii old t256
