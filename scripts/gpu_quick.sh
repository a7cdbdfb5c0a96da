mkdir -p gpurun_out
timeout 1200 python scripts/stripe_projection.py C5 > gpurun_out/proj_C5.log 2>&1; tail -3 gpurun_out/proj_C5.log | cut -c1-250
cp gpurun_out/stripe_projection.json gpurun_out/stripe_projection_C5.json
