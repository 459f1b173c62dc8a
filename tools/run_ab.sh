# usage: bash tools/run_ab.sh CONFIG libA libB  (alternating A/B bench runs of one config)
O=gpurun_out
for v in $2 $3 $2 $3; do
TTC_LIB_PATH=tools/libttc_$v.so timeout 300 python bench.py --config $1 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/ab_$v.json 2>&1
python -c "
import json
d=json.load(open('$O/ab_$v.json')); print('$v', d['value'], d['roofline']['frac'])
"
done
