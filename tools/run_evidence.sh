# Round evidence: GPU tests, smoke, default bench line (main C2 + C1/C3/C4/C5 sub-results), NEXT-row bench lines,
# reference arm, ncu launch list of the default main-line command, one full capture per hot kernel.
mkdir -p gpurun_out/ev
O=gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.max.mem,power.limit --format=csv > $O/smi.csv 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
timeout 900 python bench.py --example2 > $O/example2.json 2> $O/example2.err
for c in S1 R1 A2 A2ii; do
  timeout 600 python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/ref_default.json 2> $O/ref_default.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --no-sub"
$CMD > $O/plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv $CMD > $O/ncu_launch.log 2>&1
for kc in "C1 inner_small" "C2 inner_r16" "C3 contract" "C4 inner_r64tc" "C5 inner_ffma" "S1 splice" "R1 reconstruct" "A2 ttsvd_jacobi"; do
  set -- $kc
  CMD2="python bench.py --config $1 --steps 2 --warmup 1 --no-cpu --no-e2e --no-sub"
  $CMD2 > $O/plain_$1.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 -o $O/full_$1 -f $CMD2 > $O/ncu_full_$1.log 2>&1
done
echo done
