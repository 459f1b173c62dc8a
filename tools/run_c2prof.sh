O=gpurun_out
CMD="python bench.py --config C2 --no-sub --no-cpu --no-e2e --steps 3 --warmup 3"
$CMD > $O/c2.json 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_r16 -s 2 -c 1 -o $O/c2_full -f $CMD > $O/ncu_c2.log 2>&1; echo "ncu rc=$?"
