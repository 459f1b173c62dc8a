# C5 throughput against the number of one-warp CTAs per SM (TTC_FFMA_PER_SM caps it)
O=gpurun_out
for r in 1 2; do for P in 7 6 5 4; do
TTC_FFMA_PER_SM=$P timeout 300 python bench.py --config C5 --no-sub --no-cpu --no-e2e --steps 5 --warmup 3 > $O/c5o.json 2>$O/c5o.err
python -c "
import json; d=json.load(open('$O/c5o.json')); print('per_sm $P', round(d['value']/1e6,3))"
done; done
