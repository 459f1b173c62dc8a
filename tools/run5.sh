mkdir -p gpurun_out
timeout 120 ./tools/microbench > gpurun_out/micro5.json 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "inner" > gpurun_out/pytest_gpu5.log 2>&1
for c in C2 C5; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench5_${c}.json 2> gpurun_out/bench5_${c}.err; done
CMD="python bench.py --config C2 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_tc -s 1 -c 1 -o gpurun_out/prof5_c2 $CMD > gpurun_out/ncu5.log 2>&1
echo done
