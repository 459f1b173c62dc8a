# GPU-box helper: C5 at 7 / 8 / 9 / 10 one-warp CTAs per SM (TTC_FFMA_PER_SM), TMA staging, two rounds.
O=gpurun_out
for r in 1 2; do for w in 8 9 10 7; do
TTC_FFMA_PER_SM=$w timeout 300 python bench.py --config C5 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/occ.json 2>$O/occ.err
python -c "
import json; d=json.load(open('$O/occ.json')); print('warps/SM $w', round(d['value']/1e6,3))" || tail -3 $O/occ.err
done; done
