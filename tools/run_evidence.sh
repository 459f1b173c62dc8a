# Round evidence: default bench line, reference arm, ncu launch list + one full capture of the top kernel.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > gpurun_out/ev_smi.csv 2>&1
timeout 600 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev_ref.json 2> gpurun_out/ev_ref.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/ev_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ev_launches.csv $CMD > gpurun_out/ev_ncu_launch.log 2>&1
CMD2="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD2 > gpurun_out/ev_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_r16 -s 1 -c 1 -o gpurun_out/ev_full_c2 $CMD2 > gpurun_out/ev_ncu_full.log 2>&1
echo done
