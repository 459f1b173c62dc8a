# GPU-box helper: r16w ring-depth / warps-per-CTA variants on C2 (TTC_KERNEL=r16w), two rounds, plus the default kernel.
O=gpurun_out
for r in 1 2; do for L in old s6w2 s8w1 s10w1 s12w1; do
if [ "$L" = "old" ]; then unset TTC_KERNEL; else export TTC_KERNEL=r16w; fi
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C2 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c2w.json 2>$O/c2w.err
python -c "
import json; d=json.load(open('$O/c2w.json')); print('$L', round(d['value']/1e6,3), round(d['roofline']['frac'],3))" || tail -3 $O/c2w.err
done; done
