mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "inner" > gpurun_out/pytest_gpu4.log 2>&1
for m in cpasync bulk32 bulk1; do for c in C2 C5; do TTC_COPY=$m timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/bench4_${c}_$m.json 2> gpurun_out/bench4_${c}_$m.err; done; done
echo done
