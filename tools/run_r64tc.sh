O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_inner.py -q -k "r64_tcgen05 or c4 or C4 or variants or cost_ordered or integer" > $O/r64tc_t2.log 2>&1; echo "t2 rc=$?"; tail -3 $O/r64tc_t2.log
CMD="python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 3 --warmup 3"
timeout 300 $CMD > $O/c4_tc.json 2>$O/c4_tc.err; echo "b1 rc=$?"
python -c "
import json
d=json.load(open('$O/c4_tc.json')); print('c4_tc', d['value'], d['roofline']['frac'], d['roofline']['other']['frac'])
"
bash tools/run_prof.sh
if [ "$1" = "ncu" ]; then timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_r64tc -s 2 -c 1 -o $O/c4_tc -f $CMD > $O/ncu_c4.log 2>&1; echo "ncu rc=$?"; fi
