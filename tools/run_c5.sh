O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_inner.py -q -x -k "c5 or C5 or ffma or variants or cost_ordered or virtual or integer or edge" > $O/c5_t.log 2>&1; echo "t rc=$?"; tail -3 $O/c5_t.log
CMD="python bench.py --config C5 --no-sub --no-cpu --no-e2e --steps 5 --warmup 3 --pairs ${C5PAIRS:-65536}"
timeout 300 $CMD > $O/c5.json 2>$O/c5.err; echo "b rc=$?"
python -c "
import json
d=json.load(open('$O/c5.json')); print('c5', d['value'], d['roofline']['frac'], d['roofline']['other']['frac'])
"
if [ "$1" = "ncu" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_ffma -s 2 -c 1 -o $O/c5_ffma -f $CMD > $O/ncu_c5.log 2>&1; echo "ncu rc=$?"; fi
