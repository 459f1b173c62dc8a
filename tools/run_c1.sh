# GPU-box helper: C1 graph latency with inner_small at 256 / default / 32 threads per CTA (TTC_SMALL_THREADS).
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_inner.py -q -x -k "c1 or C1 or edge or small or variants" 2>&1 | tail -1
for r in 1 2; do for t in 256 def 32 64; do
if [ "$t" = "def" ]; then unset TTC_SMALL_THREADS; else export TTC_SMALL_THREADS=$t; fi
timeout 300 python tools/c1_lat.py > $O/c1.json 2>$O/c1.err
echo "threads $t $(cat $O/c1.json)" || tail -3 $O/c1.err
done; done
