for p in 592 1024 1184 2048 2368 4096; do
python bench.py --config C3 --pairs $p --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > gpurun_out/c3w.json 2>&1
python -c "
import json; d=json.load(open('gpurun_out/c3w.json')); print($p, round(d['value']/1e6,3), round(d['roofline']['frac'],3), round(d['ms_per_step'],4))"
done
