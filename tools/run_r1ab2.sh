# GPU-box helper: reconstruction parity on tools/libttc_new.so (both layouts), then A/B of libttc_old vs libttc_new
# on R1 and A2, and the staged layout of the new build.
O=gpurun_out
TTC_LIB_PATH=tools/libttc_new.so timeout 900 python -m pytest tests/test_gpu_reconstruct.py tests/test_gpu_guard.py tests/test_gpu_ttsvd.py -q -x > $O/r1_t.log 2>&1; echo "t rc=$?"; tail -2 $O/r1_t.log
TTC_RECON_STAGED=1 TTC_LIB_PATH=tools/libttc_new.so timeout 900 python -m pytest tests/test_gpu_reconstruct.py -q -x > $O/r1_t2.log 2>&1; echo "t2 rc=$?"; tail -2 $O/r1_t2.log
bash tools/run_ab.sh R1 old new
TTC_RECON_STAGED=1 TTC_LIB_PATH=tools/libttc_new.so timeout 300 python bench.py --config R1 --no-sub --no-cpu --no-e2e --steps 10 --warmup 3 > $O/r1s.json 2>&1; python -c "
import json; d=json.load(open('$O/r1s.json')); print('new staged', d['value'], d['roofline']['frac'])"
bash tools/run_ab.sh A2 old new
