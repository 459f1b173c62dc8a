mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 120 ./tools/microbench > gpurun_out/micro.json 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
for c in C2 C1 C3 C4 C5; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
echo done
