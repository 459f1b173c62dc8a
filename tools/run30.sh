mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "c2 or tagged or determinism or integer" > gpurun_out/pytest_gpu30.log 2>&1
for r in 1 2; do
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench30_s3_$r.json 2> /dev/null
TTC_LIB_PATH=$PWD/build/alt2/libttc_s2.so timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench30_s2_$r.json 2> /dev/null
done
echo done
