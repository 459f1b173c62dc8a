mkdir -p gpurun_out
CMD="python bench.py --config C5 --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD > gpurun_out/nc5_plain.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_ffma -s 1 -c 1 -o gpurun_out/c5_ffma $CMD > gpurun_out/nc5_ncu.log 2>&1
echo done
