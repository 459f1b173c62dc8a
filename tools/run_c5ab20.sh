O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_inner.py tests/test_gpu_guard.py -q -x -k "c5 or C5 or ffma or variants or cost_ordered or virtual or integer or edge or stay or reentr" > $O/c5s_t.log 2>&1; echo "tests rc=$?"; tail -2 $O/c5s_t.log
for r in 1 2; do for L in old new; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C5 --no-sub --no-cpu --no-e2e > $O/c5o.json 2>$O/c5o.err
python -c "
import json; d=json.load(open('$O/c5o.json')); print('$L', round(d['value']/1e6,3), round(d['roofline']['frac'],3))"
done; done
