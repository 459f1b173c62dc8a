mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu22.log 2>&1
CMD="python bench.py --config C5 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain22.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_tc -s 1 -c 1 -o gpurun_out/prof22_c5 $CMD > gpurun_out/ncu22.log 2>&1
echo done
