# GPU-box helper for C4 kernel experiments: A/B of two builds of libttc.so copied into tools/ (see DESIGN §6 C4).
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c4 or C4 or r64 or reentr" 2>&1 | tail -3
python tools/c4_err.py 2>&1 | tail -4
bash tools/run_ab.sh C4 old new
