mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ttsvd.py -m gpu -q -p no:cacheprovider > gpurun_out/ts_pytest.log 2>&1
echo done
