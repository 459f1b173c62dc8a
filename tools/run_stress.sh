# GPU-box helper: the hot-kernel parity / determinism / guard tests repeated (races in the mbarrier / TMA / tcgen05
# pipelines would show up as an occasional mismatch).
O=gpurun_out
for r in 1 2 3 4 5; do
timeout 600 python -m pytest tests/test_gpu_inner.py tests/test_gpu_guard.py -q -x -p no:cacheprovider > $O/stress_$r.log 2>&1; echo "round $r rc=$? $(tail -1 $O/stress_$r.log)"
done
