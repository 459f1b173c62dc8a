mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "inner" > gpurun_out/pytest_gpu28.log 2>&1
for c in C5 C1; do timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench28_$c.json 2> gpurun_out/bench28_$c.err; done
CMD="python bench.py --config C5 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain28.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_wpp -s 1 -c 1 -o gpurun_out/prof28_c5 $CMD > gpurun_out/ncu28.log 2>&1
echo done
