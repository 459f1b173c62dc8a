# GPU-box helper: the one-warp-per-pair rank-16 kernel (TTC_KERNEL=r16w): C2 parity tests through it, then C2 A/B.
O=gpurun_out
TTC_KERNEL=r16w timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c2 or C2 or rank16 or integer or tagged or determinism or virtual" > $O/r16w_t.log 2>&1; echo "t rc=$?"; tail -3 $O/r16w_t.log
for r in 1 2; do for k in default r16w; do
if [ "$k" = "default" ]; then unset TTC_KERNEL; else export TTC_KERNEL=$k; fi
timeout 300 python bench.py --config C2 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c2w.json 2>$O/c2w.err
python -c "
import json; d=json.load(open('$O/c2w.json')); print('$k', round(d['value']/1e6,3), round(d['roofline']['frac'],3))" || tail -3 $O/c2w.err
done; done
