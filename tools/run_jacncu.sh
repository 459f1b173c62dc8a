# GPU-box helper: one ncu source-level capture of ttsvd_jacobi_kernel under the A2 bench.
O=gpurun_out
CMD="python bench.py --config A2 --no-sub --no-cpu --no-e2e --steps 1 --warmup 1"
$CMD > $O/a2p.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-ttsvd_jacobi} -s ${KSKIP:-1} -c 1 -o $O/jac -f $CMD > $O/jac_ncu.log 2>&1; echo "ncu rc=$?"
