# GPU-box helper: FP32 kernel with its rare paths out of line (a: boundary steps; b: + pair fetch, plain staging).
O=gpurun_out
for L in a b; do TTC_LIB_PATH=tools/libttc_$L.so timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c5 or C5 or ffma or variants or edge" 2>&1 | tail -1; done
for r in 1 2; do for L in old a b; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config C5 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c5n.json 2>$O/c5n.err
python -c "
import json; d=json.load(open('$O/c5n.json')); print('$L', round(d['value']/1e6,3))" || tail -2 $O/c5n.err
done; done
