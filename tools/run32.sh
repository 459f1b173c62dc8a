mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu32.log 2>&1
for r in 1 2; do
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench32_$r.json 2> gpurun_out/bench32_$r.err
done
echo done
