mkdir -p gpurun_out
timeout 600 python bench.py --config A2 --steps 10 --warmup 3 --cpu-seconds 5 > gpurun_out/a2_bench.json 2> gpurun_out/a2_bench.err
CMD="python bench.py --config A2 --steps 2 --warmup 1 --no-cpu --no-e2e"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/a2_launches.csv $CMD > gpurun_out/a2_ncu.log 2>&1
echo done
