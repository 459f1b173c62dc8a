# GPU-box helper for C4 kernel experiments: A/B of two builds of libttc.so copied into tools/ (see DESIGN §6 C4).
O=gpurun_out
for r in 1 2; do for L in old M128 NOLOMMA; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c4e.json 2>$O/c4e.err
python -c "
import json; d=json.load(open('$O/c4e.json')); print('$L', round(d['value']/1e6,3))"
done; done
