# GPU-box helper: the NEXT-row kernels' tests (TT-SVD, reconstruction, splice, contraction) repeated.
O=gpurun_out
for r in 1 2 3; do
timeout 900 python -m pytest tests/test_gpu_ttsvd.py tests/test_gpu_reconstruct.py tests/test_gpu_splice.py tests/test_gpu_contract.py -q -x -p no:cacheprovider > $O/stress2_$r.log 2>&1; echo "round $r rc=$? $(tail -1 $O/stress2_$r.log)"
done
