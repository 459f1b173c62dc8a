# ncu capture of the workspace TT-SVD kernel on a 400 x 400 unfolding batch (8 tensors)
O=gpurun_out
cat > /tmp/ttsvd_one.py <<'PY'
import sys; sys.path.insert(0, ".")
import torch, paper_2109_00626_b200 as ttc
dims, B = (400, 400), 8
x = torch.randn(B * 160000, device="cuda")
for _ in range(2):
    T = ttc.ttc_tt_svd(x, dims, 0.0)
torch.cuda.synchronize()
PY
python /tmp/ttsvd_one.py && timeout 900 ncu --set full --clock-control none --import-source on -k regex:ttsvd_big -s 1 -c 1 -o $O/ttsvd_big -f python /tmp/ttsvd_one.py > $O/ncu_ttsvd.log 2>&1; echo "ncu rc=$?"
