mkdir -p gpurun_out
timeout 900 python scripts/stripe_projection.py C3 > gpurun_out/proj.log 2>&1; tail -4 gpurun_out/proj.log
