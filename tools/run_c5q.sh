# GPU-box helper: C5 with the FP32 kernel's queue depth 4 (old) / 6 / 8 (TTC_FFMA_Q builds), two rounds.
O=gpurun_out
for r in 1 2; do for L in old q6 q8; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C5 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c5q.json 2>$O/c5q.err
python -c "
import json; d=json.load(open('$O/c5q.json')); print('$L', round(d['value']/1e6,3))" || tail -2 $O/c5q.err
done; done
