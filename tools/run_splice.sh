mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_splice.py tests/test_gpu_contract.py -m gpu -q -p no:cacheprovider > gpurun_out/sp_pytest.log 2>&1
timeout 300 python bench.py --config S1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/sp_bench.json 2> gpurun_out/sp_bench.err
if [ "$1" = "ncu" ]; then
CMD="python bench.py --config S1 --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:splice -s 1 -c 1 -o gpurun_out/sp_full -f $CMD > gpurun_out/sp_ncu.log 2>&1
fi
echo done
