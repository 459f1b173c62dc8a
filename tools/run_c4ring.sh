# GPU-box helper: C4 ring-depth variants (tools/libttc_<v>.so: raw / lo slots), parity of each, two bench rounds.
O=gpurun_out
for L in r5l2 r6l1; do TTC_LIB_PATH=tools/libttc_$L.so timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c4 or C4 or r64" 2>&1 | tail -1; done
for r in 1 2; do for L in old new r5l2 r6l1; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c4r.json 2>$O/c4r.err
python -c "
import json; d=json.load(open('$O/c4r.json')); print('$L', round(d['value']/1e6,4))" || tail -2 $O/c4r.err
done; done
