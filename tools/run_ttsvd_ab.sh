O=gpurun_out
timeout 400 python -m pytest tests/test_gpu_ttsvd.py -q -x 2>&1 | tail -1
for L in old new old new; do echo "== $L"; TTC_LIB_PATH=tools/libttc_$L.so python tools/ttsvd_big_probe.py 2>&1 | grep -E "\(400, 400\) B 8|20, 4\)|\(400, 100\)"; done
