O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_reconstruct.py tests/test_gpu_guard.py -q -x 2>&1 | tail -1
for r in 1 2; do for L in old new; do
TTC_LIB_PATH=tools/libttc_$L.so timeout 300 python bench.py --config R1 --no-sub --no-cpu --no-e2e > $O/r1.json 2>$O/r1.err; python -c "
import json; d=json.load(open('$O/r1.json')); print('$L', round(d['value']/1e6,3), round(d['roofline']['frac'],3))"
done; done
