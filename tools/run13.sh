mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "contract" > gpurun_out/pytest_gpu17.log 2>&1
timeout 300 python bench.py --config C3 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench17_C3.json 2> gpurun_out/bench13_C3.err
CMD="python bench.py --config C3 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/plain17.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract -s 1 -c 1 -o gpurun_out/prof17_c3 $CMD > gpurun_out/ncu17.log 2>&1
echo done
