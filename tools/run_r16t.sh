# GPU-box helper: rank-16 kernel tests and the C2 bench line.
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c2 or C2 or rank16 or integer or tagged or determinism or virtual or variants" 2>&1 | tail -2
timeout 300 python bench.py --config C2 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/c2.json 2>&1; python -c "
import json; d=json.load(open('$O/c2.json')); print('C2', d['value'], d['roofline']['frac'])"
