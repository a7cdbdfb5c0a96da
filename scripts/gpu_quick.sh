mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -2 gpurun_out/q_all.log
timeout 300 python scripts/time_configs.py C3 2>&1 | tail -1
