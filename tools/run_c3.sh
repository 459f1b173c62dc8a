O=gpurun_out
CMD="python bench.py --config C3 --no-sub --no-cpu --no-e2e --steps 3 --warmup 3"
$CMD > $O/c3.json 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:contract -s 2 -c 1 -o $O/c3_full -f $CMD > $O/ncu_c3.log 2>&1; echo "ncu rc=$?"
