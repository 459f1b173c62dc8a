# Status sweep: GPU tests, one bench line per config, smoke.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > gpurun_out/st_smi.csv 2>&1
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/st_pytest.log 2>&1
for c in C2 C3 C4 C5; do
timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/st_bench_$c.json 2> gpurun_out/st_bench_$c.err
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/st_smoke.log 2>&1
echo done
