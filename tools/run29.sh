mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu29.log 2>&1
for c in C2 C5 C4 C3 C1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench29_$c.json 2> gpurun_out/bench29_$c.err; done
echo done
