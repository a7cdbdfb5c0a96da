mkdir -p gpurun_out
timeout 600 python scripts/debug_small.py 0 240 > gpurun_out/debug_plain.log 2>&1
grep -B1 -A2 "MISMATCH\|Error" gpurun_out/debug_plain.log | head -20
LAST=$(grep "^case" gpurun_out/debug_plain.log | tail -1 | awk '{print $2}')
echo "last case $LAST"
timeout 600 compute-sanitizer --tool memcheck --show-backtrace device python scripts/debug_small.py $LAST 1 > gpurun_out/sanitizer.log 2>&1
grep -v "^=========     " gpurun_out/sanitizer.log | head -40
