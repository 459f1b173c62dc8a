# GPU-box helper: TT-SVD / NEXT-row parity, then the A2 / A2ii bench lines and the Example 2 table.
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_reconstruct.py tests/test_gpu_splice.py -q -x > $O/a2fin_t.log 2>&1; echo "t rc=$?"; tail -1 $O/a2fin_t.log
timeout 300 python bench.py --config A2 > $O/bench_A2.json 2>$O/bench_A2.err; echo "A2 rc=$?"
timeout 300 python bench.py --config A2ii > $O/bench_A2ii.json 2>$O/bench_A2ii.err; echo "A2ii rc=$?"
timeout 600 python bench.py --example2 > $O/example2.json 2>$O/example2.err; echo "ex2 rc=$?"
