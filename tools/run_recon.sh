mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_reconstruct.py -m gpu -q -p no:cacheprovider > gpurun_out/rc_pytest.log 2>&1
timeout 300 python bench.py --config R1 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/rc_bench.json 2> gpurun_out/rc_bench.err
if [ "$1" = "ncu" ]; then
CMD="python bench.py --config R1 --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:reconstruct -s 1 -c 1 -o gpurun_out/rc_full -f $CMD > gpurun_out/rc_ncu.log 2>&1
fi
echo done
