# GPU-box helper: C4 as the main line (clock sampling during the timed region), three runs.
O=gpurun_out
for r in 1 2 3; do
timeout 300 python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 20 --warmup 3 > $O/c4c.json 2>$O/c4c.err
python -c "
import json; d=json.load(open('$O/c4c.json')); print(round(d['value']/1e6,4), d['clocks'], d.get('per_step_ms'))"
done
nvidia-smi --query-gpu=name,power.limit,clocks.max.sm,temperature.gpu --format=csv
