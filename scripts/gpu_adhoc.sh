cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
RQA_PREFILTER=1 timeout 900 compute-sanitizer --tool initcheck --print-limit 20 --error-exitcode 9 python scripts/sanitize_cases.py 1200 > gpurun_out/sanitize_initcheck.txt 2>&1; echo initcheck rc=$?; tail -2 gpurun_out/sanitize_initcheck.txt
bash scripts/gpu_prof1.sh i5 C3 262146
