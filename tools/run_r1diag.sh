# GPU-box helper: R1 phase diagnostics (builds only / builds + stores with K = 0; results wrong) and the write bandwidth.
O=gpurun_out
python tools/hbm_rw.py
for L in old nod sto; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config R1 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/r1d.json 2>$O/r1d.err
python -c "
import json; d=json.load(open('$O/r1d.json')); print('$L', round(d['value']/1e6,3), round(d['ms_per_step'],4))" || tail -2 $O/r1d.err
done
