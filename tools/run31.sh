mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu31.log 2>&1
for c in C1 C2 C3 C4 C5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench31_$c.json 2> gpurun_out/bench31_$c.err
done
bash tools/run_evidence.sh
