mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu34.log 2>&1
for r in 1 2; do
timeout 300 python bench.py --config C2 --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench34_$r.json 2> gpurun_out/bench34_$r.err
done
CMD2="python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e"
$CMD2 > gpurun_out/ev_plain2.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:inner_r16 -s 1 -c 1 -o gpurun_out/c2_r34 $CMD2 > gpurun_out/ncu34.log 2>&1
echo done
