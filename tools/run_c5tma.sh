# GPU-box helper: C5 parity tests, then the FP32 warp-per-pair kernel with cp.async (TTC_FFMA_TMA=0) and TMA
# staging (default) in alternating bench runs.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c5 or C5 or ffma or variants or cost_ordered or virtual or integer or edge" > $O/c5_t.log 2>&1; echo "t rc=$?"; tail -3 $O/c5_t.log
for r in 1 2; do for t in 0 1; do
TTC_FFMA_TMA=$t timeout 300 python bench.py --config C5 --no-sub --no-cpu --no-e2e --steps 5 --warmup 3 > $O/c5_$t.json 2>$O/c5_$t.err
python -c "
import json; d=json.load(open('$O/c5_$t.json')); print('tma=$t', d['value'], d['roofline']['frac'])" || tail -5 $O/c5_$t.err
done; done
