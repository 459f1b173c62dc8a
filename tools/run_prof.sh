TTC_LIB_PATH=tools/libttc_prof.so timeout 120 python bench.py --config C4 --no-sub --no-cpu --no-e2e --steps 1 --warmup 0 2>&1 | grep "r64tc prof" | head -8
