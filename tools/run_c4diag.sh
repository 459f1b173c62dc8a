# GPU-box helper: C4 with a diagnostic build (lo workers doing nothing; results wrong) against the current one.
O=gpurun_out
for r in 1 2; do for L in old nothing; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c4d.json 2>$O/c4d.err
python -c "
import json; d=json.load(open('$O/c4d.json')); print('$L', round(d['value']/1e6,3))" || tail -2 $O/c4d.err
done; done
