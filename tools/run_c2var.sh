# GPU-box helper: C2 bench for several inner_r16 build variants (tools/libttc_<v>.so), two rounds.
O=gpurun_out
for r in 1 2; do for v in old a b c e f; do
TTC_LIB_PATH=tools/libttc_$v.so timeout 300 python bench.py --config C2 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/v_$v.json 2>$O/v_$v.err
python -c "
import json; d=json.load(open('$O/v_$v.json')); print('$v', round(d['value']/1e6,3), round(d['roofline']['frac'],3))" || tail -3 $O/v_$v.err
done; done
