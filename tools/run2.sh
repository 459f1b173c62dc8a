mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "inner or smoke" > gpurun_out/pytest_gpu2.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "contract" > gpurun_out/pytest_gpu2c.log 2>&1
for c in C2 C5 C1; do timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench2_$c.json 2> gpurun_out/bench2_$c.err; done
echo done
