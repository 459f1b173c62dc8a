# GPU-box helper: rank-16 kernel with TMA-box staging (default) vs bulk-copy staging (TTC_R16_BULK=1): parity of
# both, then alternating C2 bench runs.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_inner.py tests/test_gpu_guard.py -q -x -k "c2 or C2 or rank16 or integer or tagged or determinism or virtual or stay" > $O/c2_t.log 2>&1; echo "t rc=$?"; tail -2 $O/c2_t.log
TTC_R16_BULK=1 timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c2 or C2 or rank16" > $O/c2_t2.log 2>&1; echo "t2 rc=$?"; tail -1 $O/c2_t2.log
for r in 1 2; do for m in bulk tma; do
if [ "$m" = "bulk" ]; then export TTC_R16_BULK=1; else unset TTC_R16_BULK; fi
timeout 300 python bench.py --config C2 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c2m.json 2>$O/c2m.err
python -c "
import json; d=json.load(open('$O/c2m.json')); print('$m', round(d['value']/1e6,3), round(d['roofline']['frac'],3))" || tail -3 $O/c2m.err
done; done
