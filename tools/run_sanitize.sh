# usage: bash tools/run_sanitize.sh memcheck|racecheck|synccheck  (one tool per gpurun call)
O=gpurun_out
timeout 120 python tools/sanitize_cases.py > $O/san_plain.log 2>&1 && echo plain ok && \
timeout 1500 compute-sanitizer --tool $1 --error-exitcode 9 --print-limit 50 python tools/sanitize_cases.py > $O/san_$1.log 2>&1; echo "sanitizer $1 rc=$?"; tail -15 $O/san_$1.log
