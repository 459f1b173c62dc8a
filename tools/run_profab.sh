# GPU-box helper for C4 kernel experiments: A/B of two builds of libttc.so copied into tools/ (see DESIGN §6 C4).
for v in old new; do echo "== $v"; TTC_LIB_PATH=tools/libttc_prof_$v.so timeout 120 python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 1 --warmup 0 2>&1 | grep "r64tc prof" | head -8; done
