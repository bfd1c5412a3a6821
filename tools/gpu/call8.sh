mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gputest.log 2>&1; tail -15 gpurun_out/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
