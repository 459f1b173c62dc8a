O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_ttsvd.py -q -x 2>&1 | tail -1
for r in 1 2; do for L in old new; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config A2 --no-sub --no-cpu --no-e2e > $O/a2.json 2>$O/a2.err; python -c "
import json; d=json.load(open('$O/a2.json')); print('$L', round(d['value']/1e3,1), round(d['roofline']['frac'],3))"
done; done
