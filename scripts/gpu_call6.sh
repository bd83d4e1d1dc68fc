mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke6.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -x -q -m gpu --durations=8 > gpurun_out/gputests6.log 2>&1; echo tests=$?
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo bench=$?
