# GPU-box helper: per-kernel launch times of one A2 bench step (ncu launch list, gpu__time_duration only).
O=gpurun_out
CMD="python bench.py --config A2 --no-sub --no-cpu --no-e2e --steps 1 --warmup 1"
$CMD > $O/a2_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem --clock-control none --csv --log-file $O/a2_launches.csv $CMD > $O/a2_ncu.log 2>&1; echo "ncu rc=$?"
