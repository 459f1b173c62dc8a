# round-2 first GPU call: smoke, GPU tests, default bench (with sub-results), C2 on the FFMA path, reference arm
O=gpurun_out
nvidia-smi -L
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -m gpu -q --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
TTC_KERNEL=ffma timeout 300 python bench.py --no-sub --no-cpu --no-e2e > $O/bench_c2_ffma.json 2> $O/bench_c2_ffma.err; echo "ffma rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref.json 2> $O/ref.err; echo "ref rc=$?"
