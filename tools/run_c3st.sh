# GPU-box helper: C3 with the output's store flavour varied (.cs streaming = old, write-back = wb, L1::no_allocate = na).
O=gpurun_out
for r in 1 2; do for L in old wb na; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C3 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c3s.json 2>$O/c3s.err
python -c "
import json; d=json.load(open('$O/c3s.json')); print('$L', round(d['value']/1e6,3), round(d['roofline']['frac'],3))" || tail -2 $O/c3s.err
done; done
