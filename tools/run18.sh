mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "inner" > gpurun_out/pytest_gpu19.log 2>&1
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench19_C4.json 2> gpurun_out/bench19_C4.err
CMD="python bench.py --config C4 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain19.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_r64 -s 1 -c 1 -o gpurun_out/prof19_c4 $CMD > gpurun_out/ncu19.log 2>&1
echo done
